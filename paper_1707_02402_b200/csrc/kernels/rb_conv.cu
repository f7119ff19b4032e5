// rb_conv.cu — Tier-B IEP module bodies: residual conv blocks on 128×14×14
// feature maps as tcgen05/TMEM implicit-GEMM kernels (sm_100a).
//
// Module (north star; no reference implementation — SPEC.md:268-269):
//   unary  y = relu(x + conv3x3_2(relu(conv3x3_1(x) + b1)) + b2)
//   binary z = relu(conv1x1([x; y]) + b0), then the unary block on z.
// Executor semantics around it follow src/executor.cpp:117-166 (gather child
// k as operand k, apply, scatter to the member's slot); leaves alias the
// example's input map instead of being copied.
//
// Data layout:
//   * node values / inputs: fp32 "plane maps" [16 planes][196 px][8 ch]
//     (plane j = channels 8j..8j+7) — 100,352 B per node;
//   * per-step staging: fp16 planes over a packed position axis. Each image
//     occupies a 15×15 grid (225 positions; row 14 and column 14 are zero
//     pads shared with the next image / row), so a 3×3 tap (dh, dw) is the
//     row shift dh·15 + dw of the same array. Images of one call group are
//     contiguous; each group's segment starts on a TILE_M boundary so a CTA
//     tile never mixes weights. Plane j of position q lives at
//     ((j·PS) + GUARD + q) · 16 bytes.
//   * tensor-core operands use the K-major SWIZZLE_NONE canonical layout
//     (tc_common.cuh): the shared-memory activation window
//     [plane][position][8] is a valid operand starting at ANY position, so
//     all nine taps read the same window at different row offsets — the
//     im2col never materialises.
//
// Kernel (one CTA per SM, persistent over the step's tile list):
//   warp 0 — producer: bulk async copies (TMA engine) of the activation
//            window per 64-channel K chunk (TILE_M + 2·halo positions × 8
//            planes, double-buffered) and a ring of 16 KB weight stages
//            (one (chunk, tap) block each);
//   warp 1 — TMEM allocator + single-thread tcgen05.mma issuer:
//            D[128 out channels][256 positions] (M = 128, N = 256, K = 16),
//            A = weight stage, B = window at the tap's row shift;
//   warps 2-9 — epilogue: per-tile position table in shared memory, then
//            tcgen05.ld (lane = channel, 32 positions per load), bias, ReLU,
//            residual, pad masking, fp16 staging / fp32 node-value stores.
// Accumulators are double-buffered in TMEM (2 × 256 columns) so the epilogue
// of tile i overlaps the MMAs of tile i+1.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "dynbatch/dbk.h"
#include "tc_common.cuh"

namespace {

using namespace dbk;

constexpr int kC = 128;              // channels
constexpr int kPlanes = kC / 8;      // 16
constexpr int kImg = 225;            // 15 × 15 packed grid per image
constexpr int kPx = 196;             // 14 × 14
constexpr int kFmap = kPlanes * kPx * 8;  // 25,088 floats per node map
constexpr int kGuard = 32;           // zero positions before position 0
constexpr int kTileM = 256;          // positions per CTA tile (MMA N)
constexpr int kChunkPlanes = 8;      // K chunk = 64 input channels = 8 planes
constexpr int kBStage = 128 * 64 * 2;  // 16 KB: 128 out channels × K=64 fp16 weight block
constexpr int kASlots = 2;           // A window double-buffered per K chunk
constexpr int kEpiWarps = 8;         // two warps per TMEM lane quarter, 128 positions each
constexpr int kTableWarp = 2 + kEpiWarps;  // fills the per-tile position tables ahead of the epilogue
constexpr int kThreads = (kTableWarp + 1) * 32;

// K is streamed in 64-channel chunks: for each chunk the producer loads one
// A slot (8 planes × the position window) and then one 16 KB weight block
// per tap; the MMA warp consumes (chunk, tap) blocks in that order, so the
// next chunk's (or next tile's) window loads while the current one computes.
template <int KIND>
struct Cfg;
template <>
struct Cfg<0> {  // conv1x1 over [x; y] (256 → 128)
  static constexpr int kChunks = 4, kTaps = 1, kHalo = 0, kBStages = 6;
};
template <>
struct Cfg<1> {  // conv3x3 #1 (128 → 128)
  static constexpr int kChunks = 2, kTaps = 9, kHalo = 16, kBStages = 8;
};
template <>
struct Cfg<2> : Cfg<1> {};  // conv3x3 #2 + residual

template <int KIND>
constexpr int win() { return kTileM + 2 * Cfg<KIND>::kHalo; }
template <int KIND>
constexpr int a_slot_bytes() { return kChunkPlanes * win<KIND>() * 16; }


// Per-member epilogue metadata (schedule order), built once per forward by
// k_rb_memtab from the forwarding tables.
struct MemberEntry {
  const float* res;  // residual map of conv3x3 #2 (binary: own slot = z; unary: child / input)
  float* slot;       // the node's own fp32 plane map
  uint8_t* fwd;      // parent's fp16 operand image of this node (plane 0, position 0) or null
  int32_t keep32;    // conv3x3 #2 stores the fp32 value (a reader needs it)
  int32_t pad;
};

struct ConvParams {
  int32_t step;
  const int32_t* step_tile_begin;
  const int32_t* tile_group;
  const int32_t* tile_q0;
  const int32_t* group_fid;
  const int32_t* group_begin;
  const int32_t* seg_start;
  const MemberEntry* memtab;
  const __half* stage_in;
  __half* stage_out;
  int64_t ps;  // plane stride in positions
  const __half* const* wpack;
  const float* const* bias;
  int32_t debug;  // nonzero: the MMA thread accumulates its wait cycles in g_conv_dbg
};

// MMA-thread wait accounting per kernel kind: [waiting for a drained
// accumulator, for an A window, for a weight stage, total cycles of the MMA
// loop] (entries 12..23 are unused). Read/reset with dbk_rb_debug().
__device__ unsigned long long g_conv_dbg[6 * 4];

// Residual source of positions that are not real pixels (read, never used).
__device__ float4 g_zero_res[2 * kPlanes * kPx];

// Per-position epilogue table of one tile (built by the 256 epilogue threads,
// one position each, read warp-uniformly by the 8 epilogue warps).
struct PosEntry {
  const float* res;  // KIND 2: residual map + px·8 (plane 0, channel 0)
  float* dst;        // KIND 0/2: node plane map + px·8 (nullptr: no fp32 store)
  uint8_t* fwd;      // KIND 2: parent's fp16 operand image at this position (plane 0)
  int32_t valid;     // a real pixel of a real member
  int32_t pad;
};
constexpr int kTableBytes = 2 * kTileM * static_cast<int>(sizeof(PosEntry));  // double-buffered

template <int KIND>
constexpr int smem_bytes() {
  return kASlots * a_slot_bytes<KIND>() + Cfg<KIND>::kBStages * kBStage + kTableBytes + 256;
}

// Fills the table entries of positions lane + 32k (k = 0..7) of a tile from
// the per-member table: one independent 32-byte load per position, all
// issued before any entry is stored.
template <int KIND>
__device__ __forceinline__ void rb_fill_table(const ConvParams& P, PosEntry* tab, int32_t g, int32_t q0,
                                              int lane) {
  constexpr int kPer = kTileM / 32;
  const int32_t gb0 = P.group_begin[g];
  const int32_t rows = P.group_begin[g + 1] - gb0;
  const int32_t base = q0 - P.seg_start[g];
  MemberEntry me[kPer];
  int32_t rem[kPer], px[kPer];
  bool valid[kPer];
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int32_t local = base + lane + 32 * k;
    const int32_t img = local / kImg;
    rem[k] = local - img * kImg;
    const int32_t r = rem[k] / 15, c = rem[k] - r * 15;
    valid[k] = img < rows && r < 14 && c < 14;
    px[k] = r * 14 + c;
    if (KIND != 1 && valid[k]) me[k] = P.memtab[gb0 + img];
  }
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    PosEntry e{nullptr, nullptr, nullptr, valid[k] ? 1 : 0, 0};
    if (KIND != 1 && valid[k]) {
      float* slot = me[k].slot + px[k] * 8;
      if (KIND == 0) {
        e.dst = slot;  // fp32 z, the residual of the binary block
      } else {
        e.res = me[k].res + px[k] * 8;
        e.dst = me[k].keep32 ? slot : nullptr;
        e.fwd = me[k].fwd ? me[k].fwd + rem[k] * 16 : nullptr;
      }
    }
    tab[lane + 32 * k] = e;
  }
}

// 8×8 transpose across the 8 lanes of a plane group (three butterfly
// stages): in, lane e holds x[i] = D[channel 8g+e][position i]; out, lane e
// holds x[k] = D[channel 8g+k][position e].
__device__ __forceinline__ void transpose8(float* x, int e) {
#pragma unroll
  for (int s = 4; s >= 1; s >>= 1) {
    const bool up = (e & s) != 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (i & s) continue;
      const float send = up ? x[i] : x[i + s];
      const float recv = __shfl_xor_sync(0xffffffffu, send, s);
      x[i] = up ? recv : x[i];
      x[i + s] = up ? x[i + s] : recv;
    }
  }
}

// Epilogue of one tile for this warp: TMEM lanes = output channels
// 32·quarter + lane, columns = the tile's positions; the warp covers
// positions [128·half, 128·half + 128) in eight 16-column chunks. After the
// in-register transpose, lane (g = lane/8, e = lane%8) owns positions
// 8m + e (m = 0, 1) of each chunk with the 8 channels of plane 4·quarter + g,
// so every global access is a 16-byte vector (fp16 image: one, fp32 map:
// two) and a warp instruction covers 4 planes × 8 consecutive positions.
struct EpiLane {
  int quarter, half, e, plane;
  int64_t plane_off16;  // fp16 staging offset of this lane's plane
  int plane_off32;      // fp32 plane-map offset of this lane's plane
};

constexpr int kChunk = 16;                 // positions per epilogue chunk
constexpr int kChunks = 128 / kChunk;      // chunks per warp and tile
constexpr int kResAhead = 3;               // residual prefetch distance (chunks)

// Residual rows of chunk cb of a tile for this lane (2 positions × 8 ch).
// Unconditional loads (invalid positions read a zero record) followed by a
// warp sync, so ptxas issues them here instead of sinking them to the uses.
__device__ __forceinline__ void rb_load_res(const PosEntry* tab, const EpiLane& L, int cb, float4* r) {
  const float* zero = reinterpret_cast<const float*>(g_zero_res);
  const PosEntry* my = tab + L.half * 128 + cb * kChunk + L.e;
#pragma unroll
  for (int m = 0; m < kChunk / 8; ++m) {
    const PosEntry& pe = my[8 * m];
    const float4* rp = reinterpret_cast<const float4*>((pe.valid ? pe.res : zero) + L.plane_off32);
    r[2 * m] = __ldg(rp);
    r[2 * m + 1] = __ldg(rp + 1);
  }
  __syncwarp();
}

// One 16-position chunk: TMEM → transpose → bias (+ residual) → ReLU → stores.
template <int KIND>
__device__ __forceinline__ void rb_chunk(const ConvParams& P, const PosEntry* tab, const EpiLane& L,
                                         uint32_t taddr, const float* bias, int32_t q0, int cb,
                                         const float4* res) {
  float v[kChunk];
  tmem_ld16(taddr + cb * kChunk, v);
  const PosEntry* my = tab + L.half * 128 + cb * kChunk + L.e;
#pragma unroll
  for (int m = 0; m < kChunk / 8; ++m) {
    float* x = v + 8 * m;
    transpose8(x, L.e);
    const PosEntry& pe = my[8 * m];
    if constexpr (KIND == 2) {
      if (pe.valid) {
        const float4 r0 = res[2 * m], r1 = res[2 * m + 1];
        const float o[8] = {fmaxf(x[0] + bias[0] + r0.x, 0.f), fmaxf(x[1] + bias[1] + r0.y, 0.f),
                            fmaxf(x[2] + bias[2] + r0.z, 0.f), fmaxf(x[3] + bias[3] + r0.w, 0.f),
                            fmaxf(x[4] + bias[4] + r1.x, 0.f), fmaxf(x[5] + bias[5] + r1.y, 0.f),
                            fmaxf(x[6] + bias[6] + r1.z, 0.f), fmaxf(x[7] + bias[7] + r1.w, 0.f)};
        if (pe.dst) {
          float4* dp = reinterpret_cast<float4*>(pe.dst + L.plane_off32);
          dp[0] = make_float4(o[0], o[1], o[2], o[3]);
          dp[1] = make_float4(o[4], o[5], o[6], o[7]);
        }
        if (pe.fwd) {
          uint4 pk;
          pk.x = pack_f16x2(o[0], o[1]);
          pk.y = pack_f16x2(o[2], o[3]);
          pk.z = pack_f16x2(o[4], o[5]);
          pk.w = pack_f16x2(o[6], o[7]);
          *reinterpret_cast<uint4*>(pe.fwd + L.plane_off16) = pk;
        }
      }
    } else {
      float o[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) o[k] = pe.valid ? fmaxf(x[k] + bias[k], 0.f) : 0.f;
      uint4 pk;
      pk.x = pack_f16x2(o[0], o[1]);
      pk.y = pack_f16x2(o[2], o[3]);
      pk.z = pack_f16x2(o[4], o[5]);
      pk.w = pack_f16x2(o[6], o[7]);
      uint8_t* out16 = reinterpret_cast<uint8_t*>(P.stage_out) +
                       static_cast<int64_t>(kGuard + q0 + L.half * 128 + cb * kChunk + 8 * m + L.e) * 16 +
                       L.plane_off16;
      *reinterpret_cast<uint4*>(out16) = pk;
      if (KIND == 0 && pe.valid) {  // fp32 z, the residual of the binary block
        float4* dp = reinterpret_cast<float4*>(pe.dst + L.plane_off32);
        dp[0] = make_float4(o[0], o[1], o[2], o[3]);
        dp[1] = make_float4(o[4], o[5], o[6], o[7]);
      }
    }
  }
}

// Implicit-GEMM conv, operands swapped so every MMA is N = 256 wide:
// D[128 out channels][256 positions] += W[128][k16] · X[256 positions][k16]^T
// (A = the weight stage, B = the activation window at the tap's row shift).
// N = 128 MMAs are issue-bound once the per-tap commit / barrier traffic is
// added (tools/mma_rate.cu: 88–97 cycles vs 64 ideal); N = 256 MMAs run at
// the ideal 128 cycles with the same per-tap overhead.
template <int KIND>
__global__ void __launch_bounds__(kThreads, 1) k_rb_conv(const __grid_constant__ ConvParams P) {
  using K = Cfg<KIND>;
  constexpr int WIN = win<KIND>();
  constexpr uint32_t IDESC = idesc_f16_f32(128, kTileM);
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = smem + kASlots * a_slot_bytes<KIND>();
  PosEntry* tables = reinterpret_cast<PosEntry*>(sB + K::kBStages * kBStage);
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(tables) + kTableBytes);
  uint64_t* a_full = bars;
  uint64_t* a_empty = a_full + kASlots;
  uint64_t* b_full = a_empty + kASlots;
  uint64_t* b_empty = b_full + K::kBStages;
  uint64_t* acc_full = b_empty + K::kBStages;
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* tab_full = acc_empty + 2;
  uint64_t* tab_empty = tab_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tab_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kASlots; ++s) {
      mbar_init(a_full + s, 1);
      mbar_init(a_empty + s, 1);
    }
    for (int s = 0; s < K::kBStages; ++s) {
      mbar_init(b_full + s, 1);
      mbar_init(b_empty + s, 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(acc_full + s, 1);
      mbar_init(acc_empty + s, kEpiWarps * 32);
      mbar_init(tab_full + s, 32);
      mbar_init(tab_empty + s, kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int32_t t_begin = P.step_tile_begin[P.step];
  const int32_t n_tiles = P.step_tile_begin[P.step + 1] - t_begin;

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------ producer
      uint32_t ai = 0, bi = 0;
      for (int32_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const int32_t g = P.tile_group[t_begin + t];
        const int32_t q0 = P.tile_q0[t_begin + t];
        const uint8_t* w = reinterpret_cast<const uint8_t*>(P.wpack[P.group_fid[g]]);
        const uint8_t* src = reinterpret_cast<const uint8_t*>(P.stage_in) +
                             static_cast<int64_t>(kGuard + q0 - K::kHalo) * 16;
        for (int ch = 0; ch < K::kChunks; ++ch, ++ai) {
          const uint32_t sa = ai % kASlots, pa = (ai / kASlots) & 1;
          mbar_wait(a_empty + sa, pa ^ 1);
          mbar_expect_tx(a_full + sa, a_slot_bytes<KIND>());
          for (int j = 0; j < kChunkPlanes; ++j) {
            bulk_g2s(sA + sa * a_slot_bytes<KIND>() + j * WIN * 16,
                     src + static_cast<int64_t>(ch * kChunkPlanes + j) * P.ps * 16, WIN * 16, a_full + sa);
          }
          for (int tap = 0; tap < K::kTaps; ++tap, ++bi) {
            const uint32_t s = bi % K::kBStages, ph = (bi / K::kBStages) & 1;
            mbar_wait(b_empty + s, ph ^ 1);
            mbar_expect_tx(b_full + s, kBStage);
            bulk_g2s(sB + s * kBStage, w + static_cast<int64_t>(ch * K::kTaps + tap) * kBStage, kBStage,
                     b_full + s);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------------------------------- MMA issuer
      long long w_acc = 0, w_a = 0, w_b = 0;
      const long long t_start = clock64();
      uint32_t ai = 0, bi = 0;
      int it = 0;
      const uint32_t a_base = smem_u32(sA), b_base = smem_u32(sB);
      for (int32_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++it) {
        const int abuf = it & 1;
        long long c0 = clock64();
        mbar_wait(acc_empty + abuf, ((it >> 1) & 1) ^ 1);
        w_acc += clock64() - c0;
        tc_fence_after();
        for (int ch = 0; ch < K::kChunks; ++ch, ++ai) {
          const uint32_t sa = ai % kASlots, pa = (ai / kASlots) & 1;
          c0 = clock64();
          mbar_wait(a_full + sa, pa);
          w_a += clock64() - c0;
          tc_fence_after();
          const uint32_t a_slot = a_base + sa * a_slot_bytes<KIND>();
          for (int tap = 0; tap < K::kTaps; ++tap, ++bi) {
            const uint32_t s = bi % K::kBStages, ph = (bi / K::kBStages) & 1;
            c0 = clock64();
            mbar_wait(b_full + s, ph);
            w_b += clock64() - c0;
            tc_fence_after();
            const int shift = K::kTaps == 9 ? (tap / 3 - 1) * 15 + (tap % 3 - 1) : 0;
            const uint32_t xrow = static_cast<uint32_t>(K::kHalo + shift);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint64_t wd = smem_desc(b_base + s * kBStage + (2 * kk) * 2048, 2048, 128);
              const uint64_t xd = smem_desc(a_slot + ((2 * kk) * WIN + xrow) * 16, WIN * 16, 128);
              mma_bf16(tmem_base + abuf * kTileM, wd, xd, IDESC, (ch | tap | kk) != 0);
            }
            mma_commit(b_empty + s);
          }
          mma_commit(a_empty + sa);
        }
        mma_commit(acc_full + abuf);
      }
      if (P.debug) {
        atomicAdd(&g_conv_dbg[KIND * 4 + 0], static_cast<unsigned long long>(w_acc));
        atomicAdd(&g_conv_dbg[KIND * 4 + 1], static_cast<unsigned long long>(w_a));
        atomicAdd(&g_conv_dbg[KIND * 4 + 2], static_cast<unsigned long long>(w_b));
        atomicAdd(&g_conv_dbg[KIND * 4 + 3], static_cast<unsigned long long>(clock64() - t_start));
      }
    }
  } else if (warp == kTableWarp) {  // ------------------------ table filler
    int it = 0;
    for (int32_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++it) {
      const int buf = it & 1;
      const int32_t g = P.tile_group[t_begin + t];
      const int32_t q0 = P.tile_q0[t_begin + t];
      mbar_wait(tab_empty + buf, ((it >> 1) & 1) ^ 1);
      rb_fill_table<KIND>(P, tables + buf * kTileM, g, q0, lane);
      mbar_arrive(tab_full + buf);  // release: the entries are visible to the waiters
    }
  } else {  // ------------------------------------------------------ epilogue
    EpiLane L;
    L.quarter = warp & 3;
    L.half = (warp - 2) >> 2;
    L.e = lane & 7;
    L.plane = L.quarter * 4 + (lane >> 3);
    L.plane_off16 = static_cast<int64_t>(L.plane) * P.ps * 16;
    L.plane_off32 = L.plane * kPx * 8;
    const uint32_t lane_addr = (static_cast<uint32_t>(L.quarter * 32) << 16) + L.half * 128;
    // residual chunks are loaded kResAhead ahead, across tile boundaries
    // (ring of 4 buffers, so every index is a compile-time constant)
    float4 rbuf[4][kChunk / 4];
    int it = 0;
    int32_t t = blockIdx.x;
    if (KIND == 2 && t < n_tiles) {
      mbar_wait(tab_full + 0, 0);
#pragma unroll
      for (int c = 0; c < kResAhead; ++c) rb_load_res(tables, L, c, rbuf[c]);
    }
    for (; t < n_tiles; t += gridDim.x, ++it) {
      const int abuf = it & 1;
      const int32_t g = P.tile_group[t_begin + t];
      const int32_t q0 = P.tile_q0[t_begin + t];
      const PosEntry* tab = tables + abuf * kTileM;
      const float* bias_p = P.bias[P.group_fid[g]] + L.plane * 8;
      const float4 b_lo = __ldg(reinterpret_cast<const float4*>(bias_p));
      const float4 b_hi = __ldg(reinterpret_cast<const float4*>(bias_p + 4));
      const float bias[8] = {b_lo.x, b_lo.y, b_lo.z, b_lo.w, b_hi.x, b_hi.y, b_hi.z, b_hi.w};
      mbar_wait(tab_full + abuf, (it >> 1) & 1);
      mbar_wait(acc_full + abuf, (it >> 1) & 1);
      tc_fence_after();
      const uint32_t taddr = tmem_base + abuf * kTileM + lane_addr;
      const bool has_next = t + static_cast<int32_t>(gridDim.x) < n_tiles;
#pragma unroll
      for (int cb = 0; cb < kChunks; ++cb) {
        if (KIND == 2) {
          constexpr int A = kResAhead;
          if (cb + A < kChunks) {
            rb_load_res(tab, L, cb + A, rbuf[(cb + A) & 3]);
          } else if (has_next) {
            const int nb = (it + 1) & 1;
            if (cb + A == kChunks) mbar_wait(tab_full + nb, ((it + 1) >> 1) & 1);
            rb_load_res(tables + nb * kTileM, L, cb + A - kChunks, rbuf[(cb + A) & 3]);
          }
        }
        rb_chunk<KIND>(P, tab, L, taddr, bias, q0, cb, rbuf[cb & 3]);
      }
      tc_fence_before();
      mbar_arrive(acc_empty + abuf);
      __syncwarp();
      if (lane == 0) mbar_arrive(tab_empty + abuf);
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

// ----------------------------------------------------------------- plan
// Segment layout and tile lists for every step, from the group tables.
// seg_start[g] is relative to the step's position origin; tiles of step s
// occupy [step_tile_begin[s], step_tile_begin[s+1]).
__global__ void k_rb_plan(int32_t n_steps, const int32_t* __restrict__ sgb,
                          const int32_t* __restrict__ group_fid, const int32_t* __restrict__ group_begin,
                          const int32_t* __restrict__ arity_of, int32_t* __restrict__ seg_start,
                          int32_t* __restrict__ group_tile0, int32_t* __restrict__ group_bintile0,
                          int32_t* __restrict__ step_tile_begin, int32_t* __restrict__ step_bintile_begin,
                          int32_t* __restrict__ step_positions, int32_t tile_m) {
  // One thread per step computes its segment starts; tile prefixes over
  // steps are then accumulated serially (steps are few for improved schedules).
  for (int32_t s = threadIdx.x; s < n_steps; s += blockDim.x) {
    int32_t cursor = 0, tiles = 0, bintiles = 0;
    for (int32_t g = sgb[s]; g < sgb[s + 1]; ++g) {
      const int32_t rows = group_begin[g + 1] - group_begin[g];
      if (arity_of[group_fid[g]] == 0 || rows == 0) {
        seg_start[g] = -1;
        continue;
      }
      const int32_t nt = (rows * kImg + tile_m - 1) / tile_m;
      seg_start[g] = cursor;
      group_tile0[g] = tiles;
      group_bintile0[g] = arity_of[group_fid[g]] == 2 ? bintiles : -1;
      cursor += nt * tile_m;
      tiles += nt;
      if (arity_of[group_fid[g]] == 2) bintiles += nt;
    }
    step_positions[s] = cursor;
    step_tile_begin[s + 1] = tiles;
    step_bintile_begin[s + 1] = bintiles;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    step_tile_begin[0] = 0;
    step_bintile_begin[0] = 0;
    int32_t base = 0;
    for (int32_t s = 0; s < n_steps; ++s) {
      step_tile_begin[s + 1] += step_tile_begin[s];
      step_bintile_begin[s + 1] += step_bintile_begin[s];
      const int32_t n = step_positions[s];
      step_positions[s] = base;  // becomes the step's position origin
      base += n;
    }
    step_positions[n_steps] = base;
  }
  __syncthreads();
  // Every step owns its own staging range, so a result can be written
  // straight into the operand image of its parent's (later) step.
  for (int32_t s = threadIdx.x; s < n_steps; s += blockDim.x) {
    const int32_t base = step_positions[s];
    for (int32_t g = sgb[s]; g < sgb[s + 1]; ++g)
      if (seg_start[g] >= 0) seg_start[g] += base;
  }
}

// Forwarding table for conv3x3 #2 epilogues: for every expensive member,
// each child with a unique parent (fwd_ok) receives the absolute staging
// position of that parent's image and which buffer / planes it fills.
__global__ void k_rb_fwd_init(int64_t n, int32_t* __restrict__ fwd_pos, int32_t* __restrict__ fwd_slot) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) {
    fwd_pos[i] = -1;
    fwd_slot[i] = 1 << 8;  // keep the fp32 value (roots, shared children)
  }
}

__global__ void k_rb_fwd(int32_t n_steps, const int32_t* __restrict__ sgb, const int32_t* __restrict__ group_fid,
                         const int32_t* __restrict__ group_begin, const int32_t* __restrict__ arity_of,
                         const int32_t* __restrict__ seg_start, const int32_t* __restrict__ member_g,
                         const int32_t* __restrict__ child0, const int32_t* __restrict__ child1,
                         const int32_t* __restrict__ fwd_ok, int32_t* __restrict__ fwd_pos,
                         int32_t* __restrict__ fwd_slot) {
  const int32_t s = blockIdx.x;
  if (s >= n_steps) return;
  for (int32_t g = sgb[s]; g < sgb[s + 1]; ++g) {
    if (seg_start[g] < 0) continue;
    const int32_t arity = arity_of[group_fid[g]];
    const int32_t rows = group_begin[g + 1] - group_begin[g];
    for (int32_t i = threadIdx.x; i < rows; i += blockDim.x) {
      const int32_t node = member_g[group_begin[g] + i];
      for (int k = 0; k < arity; ++k) {
        const int32_t c = k == 0 ? child0[node] : child1[node];
        if (!fwd_ok[c]) continue;
        fwd_pos[c] = seg_start[g] + i * kImg;
        // unary parent: conv3x3 #2 of the parent reads the child's fp32 value
        // as its residual, so keep it; binary parents use their own z.
        fwd_slot[c] = (arity == 2 ? 1 : 0) | ((16 * k) << 1) | ((arity == 1 ? 1 : 0) << 8);
      }
    }
  }
}

__global__ void k_rb_memtab(int32_t n_steps, const int32_t* __restrict__ sgb,
                            const int32_t* __restrict__ group_fid, const int32_t* __restrict__ group_begin,
                            const int32_t* __restrict__ arity_of, const int32_t* __restrict__ seg_start,
                            const int32_t* __restrict__ member_g, const int32_t* __restrict__ fid,
                            const int32_t* __restrict__ child0, const int32_t* __restrict__ example,
                            const int32_t* __restrict__ fwd_pos, const int32_t* __restrict__ fwd_slot,
                            const float* inputs, float* values, uint8_t* stage_x, uint8_t* stage_cat,
                            int64_t ps, MemberEntry* __restrict__ memtab) {
  const int32_t s = blockIdx.x;
  if (s >= n_steps) return;
  for (int32_t g = sgb[s]; g < sgb[s + 1]; ++g) {
    if (seg_start[g] < 0) continue;
    const int32_t arity = arity_of[group_fid[g]];
    for (int32_t m = group_begin[g] + threadIdx.x; m < group_begin[g + 1]; m += blockDim.x) {
      const int32_t node = member_g[m];
      MemberEntry e;
      e.slot = values + static_cast<int64_t>(node) * kFmap;
      if (arity == 2) {
        e.res = e.slot;
      } else {
        const int32_t ch = child0[node];
        e.res = arity_of[fid[ch]] == 0 ? inputs + static_cast<int64_t>(example[ch]) * kFmap
                                       : values + static_cast<int64_t>(ch) * kFmap;
      }
      const int32_t sw = fwd_slot[node];
      const int32_t tgt = fwd_pos[node];
      e.keep32 = (sw >> 8) & 1;
      e.fwd = tgt >= 0 ? ((sw & 1) ? stage_cat : stage_x) + (static_cast<int64_t>((sw >> 1) & 31) * ps + kGuard + tgt) * 16
                       : nullptr;
      e.pad = 0;
      memtab[m] = e;
    }
  }
}

__global__ void k_rb_tiles(int32_t n_steps, const int32_t* __restrict__ sgb,
                           const int32_t* __restrict__ group_fid, const int32_t* __restrict__ group_begin,
                           const int32_t* __restrict__ arity_of, const int32_t* __restrict__ seg_start,
                           const int32_t* __restrict__ group_tile0, const int32_t* __restrict__ group_bintile0,
                           const int32_t* __restrict__ step_tile_begin,
                           const int32_t* __restrict__ step_bintile_begin, int32_t* __restrict__ tile_group,
                           int32_t* __restrict__ tile_q0, int32_t* __restrict__ bin_group,
                           int32_t* __restrict__ bin_q0, int32_t tile_m) {
  const int32_t s = blockIdx.x;
  if (s >= n_steps) return;
  for (int32_t g = sgb[s]; g < sgb[s + 1]; ++g) {
    if (seg_start[g] < 0) continue;
    const int32_t rows = group_begin[g + 1] - group_begin[g];
    const int32_t nt = (rows * kImg + tile_m - 1) / tile_m;
    for (int32_t i = threadIdx.x; i < nt; i += blockDim.x) {
      const int32_t ti = step_tile_begin[s] + group_tile0[g] + i;
      tile_group[ti] = g;
      tile_q0[ti] = seg_start[g] + i * tile_m;
      if (group_bintile0[g] >= 0) {
        const int32_t bi = step_bintile_begin[s] + group_bintile0[g] + i;
        bin_group[bi] = g;
        bin_q0[bi] = seg_start[g] + i * tile_m;
      }
    }
  }
}

// --------------------------------------------------------------- gather
// Packs the operand maps that were NOT forwarded by a child's conv3x3 #2
// epilogue — leaves (the example's input map) and children shared by
// several parents — into the member's fp16 staging image: unary → stage_x
// (16 planes), binary → stage_cat planes 16k.. (the channel concat of
// [x; y] is fused into the write). Only the 196 data positions are written;
// pads and alignment gaps were zeroed once at session creation.
__global__ void __launch_bounds__(256) k_rb_gather(
    int32_t step, const int32_t* __restrict__ sgb, const int32_t* __restrict__ group_fid,
    const int32_t* __restrict__ group_begin, const int32_t* __restrict__ seg_start,
    const int32_t* __restrict__ member_g, const int32_t* __restrict__ arity_of,
    const int32_t* __restrict__ fid, const int32_t* __restrict__ child0,
    const int32_t* __restrict__ child1, const int32_t* __restrict__ example,
    const int32_t* __restrict__ fwd_ok, const float* __restrict__ inputs,
    const float* __restrict__ values, uint8_t* __restrict__ stage_x, uint8_t* __restrict__ stage_cat,
    int64_t ps) {
  const int32_t g_lo = sgb[step], g_hi = sgb[step + 1];
  const int32_t m_lo = group_begin[g_lo], m_hi = group_begin[g_hi];
  for (int32_t m = m_lo + blockIdx.x; m < m_hi; m += gridDim.x) {
    int32_t g = g_lo;
    while (group_begin[g + 1] <= m) ++g;
    const int32_t arity = arity_of[group_fid[g]];
    if (arity == 0 || seg_start[g] < 0) continue;
    const int32_t node = member_g[m];
    const int32_t base = kGuard + seg_start[g] + (m - group_begin[g]) * kImg;
    uint8_t* dst = arity == 2 ? stage_cat : stage_x;
    for (int k = 0; k < arity; ++k) {
      const int32_t ch = k == 0 ? child0[node] : child1[node];
      if (fwd_ok[ch]) continue;  // written by the child's epilogue
      const float* src = arity_of[fid[ch]] == 0 ? inputs + static_cast<int64_t>(example[ch]) * kFmap
                                                : values + static_cast<int64_t>(ch) * kFmap;
      for (int idx = threadIdx.x; idx < kPlanes * kPx; idx += blockDim.x) {
        const int p = idx / kPx, px = idx - p * kPx;
        const int r = px / 14, c = px - r * 14;
        const float* sp = src + (p * kPx + px) * 8;
        const float4 lo = *reinterpret_cast<const float4*>(sp);
        const float4 hi = *reinterpret_cast<const float4*>(sp + 4);
        uint4 pk;
        pk.x = pack_f16x2(lo.x, lo.y);
        pk.y = pack_f16x2(lo.z, lo.w);
        pk.z = pack_f16x2(hi.x, hi.y);
        pk.w = pack_f16x2(hi.z, hi.w);
        *reinterpret_cast<uint4*>(dst + (static_cast<int64_t>(16 * k + p) * ps + base + r * 15 + c) * 16) = pk;
      }
    }
  }
}

// Layout conversions between reference rows (CHW: element c·196 + px) and
// plane maps ([16][196][8]); one block per (row, plane) transposes a
// 196 × 8 tile through shared memory so both sides stay coalesced.
__global__ void __launch_bounds__(256) k_chw_to_planes(const float* __restrict__ chw,
                                                       float* __restrict__ planes) {
  __shared__ float t[8][kPx + 1];
  const int64_t row = blockIdx.x / kPlanes;
  const int p = blockIdx.x % kPlanes;
  const float* src = chw + row * kFmap + p * 8 * kPx;
  for (int i = threadIdx.x; i < 8 * kPx; i += blockDim.x) t[i / kPx][i % kPx] = src[i];
  __syncthreads();
  float* dst = planes + row * kFmap + p * kPx * 8;
  for (int i = threadIdx.x; i < 8 * kPx; i += blockDim.x) dst[i] = t[i & 7][i >> 3];
}

__global__ void __launch_bounds__(256) k_roots_to_chw(const int32_t* __restrict__ root_g,
                                                      const int32_t* __restrict__ fid,
                                                      const int32_t* __restrict__ arity_of,
                                                      const int32_t* __restrict__ example,
                                                      const float* __restrict__ inputs,
                                                      const float* __restrict__ values,
                                                      float* __restrict__ chw) {
  __shared__ float t[8][kPx + 1];
  const int64_t e = blockIdx.x / kPlanes;
  const int p = blockIdx.x % kPlanes;
  const int32_t r = root_g[e];
  const float* map = arity_of[fid[r]] == 0 ? inputs + static_cast<int64_t>(example[r]) * kFmap
                                          : values + static_cast<int64_t>(r) * kFmap;
  const float* src = map + p * kPx * 8;
  for (int i = threadIdx.x; i < 8 * kPx; i += blockDim.x) t[i & 7][i >> 3] = src[i];
  __syncthreads();
  float* dst = chw + e * kFmap + p * 8 * kPx;
  for (int i = threadIdx.x; i < 8 * kPx; i += blockDim.x) dst[i] = t[i / kPx][i % kPx];
}

int32_t g_debug_flag = 0;

template <int KIND>
int launch_conv(const ConvParams& p, int num_sms, cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_rb_conv<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes<KIND>());
    configured = true;
  }
  k_rb_conv<KIND><<<num_sms, kThreads, smem_bytes<KIND>(), s>>>(p);
  return static_cast<int>(cudaGetLastError());
}

}  // namespace

extern "C" int dbk_rb_plan(int32_t n_steps, const int32_t* step_group_begin, const int32_t* group_fid,
                           const int32_t* group_begin, const int32_t* arity_of, int32_t* seg_start,
                           int32_t* group_tile0, int32_t* group_bintile0, int32_t* step_tile_begin,
                           int32_t* step_bintile_begin, int32_t* step_positions, int32_t* tile_group,
                           int32_t* tile_q0, int32_t* bin_group, int32_t* bin_q0, int64_t n_nodes,
                           const int32_t* member_g, const int32_t* child0, const int32_t* child1,
                           const int32_t* fwd_ok, int32_t* fwd_pos, int32_t* fwd_slot, int32_t tile_m,
                           void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (n_steps <= 0) return 0;
  k_rb_plan<<<1, 1024, 0, s>>>(n_steps, step_group_begin, group_fid, group_begin, arity_of, seg_start,
                               group_tile0, group_bintile0, step_tile_begin, step_bintile_begin,
                               step_positions, tile_m);
  k_rb_tiles<<<n_steps, 256, 0, s>>>(n_steps, step_group_begin, group_fid, group_begin, arity_of,
                                     seg_start, group_tile0, group_bintile0, step_tile_begin,
                                     step_bintile_begin, tile_group, tile_q0, bin_group, bin_q0, tile_m);
  k_rb_fwd_init<<<static_cast<unsigned>((n_nodes + 255) / 256), 256, 0, s>>>(n_nodes, fwd_pos, fwd_slot);
  k_rb_fwd<<<n_steps, 256, 0, s>>>(n_steps, step_group_begin, group_fid, group_begin, arity_of, seg_start,
                                   member_g, child0, child1, fwd_ok, fwd_pos, fwd_slot);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_rb_gather(int32_t step, const int32_t* step_group_begin, const int32_t* group_fid,
                             const int32_t* group_begin, const int32_t* seg_start, const int32_t* member_g,
                             const int32_t* arity_of, const int32_t* fid, const int32_t* child0,
                             const int32_t* child1, const int32_t* example, const int32_t* fwd_ok,
                             const float* inputs, const float* values, void* stage_x, void* stage_cat,
                             int64_t plane_stride, int32_t blocks, void* stream) {
  k_rb_gather<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      step, step_group_begin, group_fid, group_begin, seg_start, member_g, arity_of, fid, child0, child1,
      example, fwd_ok, inputs, values, static_cast<uint8_t*>(stage_x), static_cast<uint8_t*>(stage_cat),
      plane_stride);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_rb_memtab(int32_t n_steps, const int32_t* step_group_begin, const int32_t* group_fid,
                             const int32_t* group_begin, const int32_t* arity_of, const int32_t* seg_start,
                             const int32_t* member_g, const int32_t* fid, const int32_t* child0,
                             const int32_t* example, const int32_t* fwd_pos, const int32_t* fwd_slot,
                             const float* inputs, float* values, void* stage_x, void* stage_cat,
                             int64_t plane_stride, void* memtab, void* stream) {
  if (n_steps <= 0) return 0;
  k_rb_memtab<<<n_steps, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      n_steps, step_group_begin, group_fid, group_begin, arity_of, seg_start, member_g, fid, child0, example,
      fwd_pos, fwd_slot, inputs, values, static_cast<uint8_t*>(stage_x), static_cast<uint8_t*>(stage_cat),
      plane_stride, static_cast<MemberEntry*>(memtab));
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_rb_conv(int32_t kind, int32_t step, const int32_t* step_tile_begin,
                           const int32_t* tile_group, const int32_t* tile_q0, const int32_t* group_fid,
                           const int32_t* group_begin, const int32_t* seg_start, const void* memtab,
                           const void* stage_in, void* stage_out, int64_t plane_stride,
                           const void* const* wpack, const float* const* bias, int32_t num_sms,
                           void* stream) {
  ConvParams p{step,
               step_tile_begin,
               tile_group,
               tile_q0,
               group_fid,
               group_begin,
               seg_start,
               static_cast<const MemberEntry*>(memtab),
               static_cast<const __half*>(stage_in),
               static_cast<__half*>(stage_out),
               plane_stride,
               reinterpret_cast<const __half* const*>(wpack),
               bias,
               g_debug_flag};
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  switch (kind) {
    case 0: return launch_conv<0>(p, num_sms, s);
    case 1: return launch_conv<1>(p, num_sms, s);
    case 2: return launch_conv<2>(p, num_sms, s);
  }
  return static_cast<int>(cudaErrorInvalidValue);
}

extern "C" int dbk_rb_inputs_from_chw(int64_t rows, const float* chw, float* planes, void* stream) {
  const int64_t total = rows * kFmap;
  if (total <= 0) return 0;
  k_chw_to_planes<<<static_cast<unsigned>(rows * kPlanes), 256, 0, static_cast<cudaStream_t>(stream)>>>(chw,
                                                                                                     planes);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_rb_outputs_to_chw(int64_t b, const int32_t* root_g, const int32_t* fid,
                                     const int32_t* arity_of, const int32_t* example, const float* inputs,
                                     const float* values, float* chw, void* stream) {
  const int64_t total = b * kFmap;
  if (total <= 0) return 0;
  k_roots_to_chw<<<static_cast<unsigned>(b * kPlanes), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      root_g, fid, arity_of, example, inputs, values, chw);
  return static_cast<int>(cudaGetLastError());
}

// Copies (and optionally zeroes) the MMA-thread wait counters; enable != 0
// turns accounting on for subsequent launches.
extern "C" int dbk_rb_debug(unsigned long long* out, int32_t reset, int32_t enable) {
  g_debug_flag = enable;
  if (out) cudaMemcpyFromSymbol(out, g_conv_dbg, sizeof(unsigned long long) * 24);
  if (reset) {
    unsigned long long z[24] = {};
    cudaMemcpyToSymbol(g_conv_dbg, z, sizeof(z));
  }
  return static_cast<int>(cudaGetLastError());
}
