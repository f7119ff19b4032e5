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
//     (tc_common.cuh): the shared-memory A window [plane][position][8] is a
//     valid operand starting at ANY position, so all nine taps read the same
//     window at different row offsets — the im2col never materialises.
//
// Kernel (one CTA per SM, persistent over the step's tile list):
//   warp 0 — producer: bulk async copies (TMA engine) of the A window
//            (TILE_M + 32 positions × all input planes) and a ring of 32 KB
//            weight stages (one 3×3 tap, or one 128-channel half of the 1×1);
//   warp 1 — TMEM allocator + single-thread tcgen05.mma issuer
//            (M = 128 per accumulator, N = 128, K = 16 per instruction);
//   warps 2-5 — epilogue: tcgen05.ld of the fp32 accumulators, bias, ReLU,
//            residual, pad masking, fp16 staging / fp32 node-value stores.
// Accumulators are double-buffered in TMEM (2 × 256 columns) so the epilogue
// of tile i overlaps the MMAs of tile i+1.
#include <cuda_bf16.h>
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
constexpr int kTileM = 256;          // positions per CTA tile (2 accumulators)
constexpr int kChunkPlanes = 8;      // K chunk = 64 input channels = 8 planes
constexpr int kBStage = 128 * 64 * 2;  // 16 KB: N=128 × K=64 fp16 weight block
constexpr int kASlots = 2;           // A window double-buffered per K chunk
constexpr int kEpiWarps = 8;       // two warps per TMEM lane quarter, two column chunks each
constexpr int kThreads = 64 + kEpiWarps * 32;

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
template <int KIND>
constexpr int smem_bytes() {
  return kASlots * a_slot_bytes<KIND>() + Cfg<KIND>::kBStages * kBStage + 256;
}

struct ConvParams {
  int32_t step;
  const int32_t* step_tile_begin;
  const int32_t* tile_group;
  const int32_t* tile_q0;
  const int32_t* group_fid;
  const int32_t* group_begin;
  const int32_t* seg_start;
  const int32_t* member_g;
  const int32_t* arity_of;
  const int32_t* fid;
  const int32_t* child0;
  const int32_t* example;
  const __nv_bfloat16* stage_in;
  __nv_bfloat16* stage_out;
  int64_t ps;  // plane stride in positions
  const float* inputs;
  float* values;
  const __nv_bfloat16* const* wpack;
  const float* const* bias;
  // conv3x3 #2 only: forwarding of each result as the fp16 operand image of
  // its (unique) parent's call — fwd_pos[g] = absolute staging position of
  // the parent's image (-1: none), fwd_slot[g] = buffer (bit 0: 0 stage_x,
  // 1 stage_cat) | first plane << 1 | keep-fp32-value << 8.
  const int32_t* fwd_pos;
  const int32_t* fwd_slot;
  __nv_bfloat16* stage_x;
  __nv_bfloat16* stage_cat;
  int32_t debug;  // nonzero: the MMA thread accumulates its wait cycles in g_conv_dbg
};

// MMA-thread wait accounting per kernel kind (pair kinds at +3):
// [waiting for a drained accumulator, for an A window, for a weight stage,
// total cycles of the MMA loop]. Read/reset with dbk_rb_debug().
__device__ unsigned long long g_conv_dbg[6 * 4];

// Epilogue of one tile (256 positions = 2 TMEM accumulators) for this warp's
// lane quarter and two 32-column chunks.
template <int KIND>
__device__ __forceinline__ void rb_epilogue(const ConvParams& P, uint32_t tmem_base, int abuf, int32_t g,
                                            int32_t q0, int quarter, int cb0, int lane) {
      const int32_t f = P.group_fid[g];
      const int32_t gb0 = P.group_begin[g];
      const int32_t rows = P.group_begin[g + 1] - gb0;
      const int32_t seg = P.seg_start[g];
      const float* __restrict__ bias = P.bias[f];
      const bool binary = P.arity_of[f] == 2;
#pragma unroll 1
      for (int a = 0; a < kTileM / 128; ++a) {
        const int row = a * 128 + quarter * 32 + lane;
        const int32_t q = q0 + row;
        const int32_t local = q - seg;
        const int32_t img = local / kImg, rem = local - img * kImg;
        const int32_t r = rem / 15, c = rem - r * 15;
        const bool valid = img < rows && r < 14 && c < 14;
        const int32_t px = r * 14 + c;
        int32_t node = 0;
        const float* res = nullptr;
        float* dst32 = nullptr;
        if (valid && KIND != 1) {
          node = P.member_g[gb0 + img];
          dst32 = P.values + static_cast<int64_t>(node) * kFmap;
          if (KIND == 2) {
            if (binary) {
              res = dst32;  // z was parked in the node's own slot by conv1x1
            } else {
              const int32_t ch = P.child0[node];
              res = P.arity_of[P.fid[ch]] == 0 ? P.inputs + static_cast<int64_t>(P.example[ch]) * kFmap
                                               : P.values + static_cast<int64_t>(ch) * kFmap;
            }
          }
        }
        if constexpr (KIND == 2) {
          // Residual rows are fetched one 32-channel chunk ahead of the TMEM
          // loads so the epilogue keeps 8 independent 16-byte loads in flight
          // (the residual may alias the destination for binary modules, so
          // every chunk is fully loaded before any of its stores).
          const float* rbase = valid ? res + px * 8 : nullptr;
          float* dbase = valid ? dst32 + px * 8 : nullptr;
          // forwarding target: the parent's fp16 operand image (if unique parent)
          int32_t slot = 0;
          uint8_t* fbase = nullptr;
          if (valid) {
            const int32_t tgt = P.fwd_pos[node];
            slot = P.fwd_slot[node];
            if (tgt >= 0) {
              fbase = reinterpret_cast<uint8_t*>((slot & 1) ? P.stage_cat : P.stage_x) +
                      (static_cast<int64_t>((slot >> 1) & 31) * P.ps + kGuard + tgt + rem) * 16;
            }
          }
          const bool keep32 = (slot >> 8) & 1;
          float4 rcur[8], rnext[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) rcur[i] = rnext[i] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (valid) {
#pragma unroll
            for (int pp = 0; pp < 4; ++pp) {
              rcur[2 * pp] = *reinterpret_cast<const float4*>(rbase + (cb0 * 4 + pp) * kPx * 8);
              rcur[2 * pp + 1] = *reinterpret_cast<const float4*>(rbase + (cb0 * 4 + pp) * kPx * 8 + 4);
            }
          }
#pragma unroll
          for (int cbi = 0; cbi < 2; ++cbi) {
            const int cb = cb0 + cbi;
            float v[32];
            tmem_ld32(tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + abuf * 256 + a * 128 + cb * 32, v);
            if (valid && cbi == 0) {
#pragma unroll
              for (int pp = 0; pp < 4; ++pp) {
                const float* rp = rbase + ((cb + 1) * 4 + pp) * kPx * 8;
                rnext[2 * pp] = *reinterpret_cast<const float4*>(rp);
                rnext[2 * pp + 1] = *reinterpret_cast<const float4*>(rp + 4);
              }
            }
            if (valid) {
#pragma unroll
              for (int pp = 0; pp < 4; ++pp) {
                const int plane = cb * 4 + pp;
                const float4 b_lo = __ldg(reinterpret_cast<const float4*>(bias + plane * 8));
                const float4 b_hi = __ldg(reinterpret_cast<const float4*>(bias + plane * 8 + 4));
                const float4 r0 = rcur[2 * pp], r1 = rcur[2 * pp + 1];
                const float4 o0 = make_float4(fmaxf(v[pp * 8 + 0] + b_lo.x + r0.x, 0.f),
                                              fmaxf(v[pp * 8 + 1] + b_lo.y + r0.y, 0.f),
                                              fmaxf(v[pp * 8 + 2] + b_lo.z + r0.z, 0.f),
                                              fmaxf(v[pp * 8 + 3] + b_lo.w + r0.w, 0.f));
                const float4 o1 = make_float4(fmaxf(v[pp * 8 + 4] + b_hi.x + r1.x, 0.f),
                                              fmaxf(v[pp * 8 + 5] + b_hi.y + r1.y, 0.f),
                                              fmaxf(v[pp * 8 + 6] + b_hi.z + r1.z, 0.f),
                                              fmaxf(v[pp * 8 + 7] + b_hi.w + r1.w, 0.f));
                if (keep32) {
                  float* dp = dbase + plane * kPx * 8;
                  *reinterpret_cast<float4*>(dp) = o0;
                  *reinterpret_cast<float4*>(dp + 4) = o1;
                }
                if (fbase) {
                  uint4 pk;
                  pk.x = pack_f16x2(o0.x, o0.y);
                  pk.y = pack_f16x2(o0.z, o0.w);
                  pk.z = pack_f16x2(o1.x, o1.y);
                  pk.w = pack_f16x2(o1.z, o1.w);
                  *reinterpret_cast<uint4*>(fbase + static_cast<int64_t>(plane) * P.ps * 16) = pk;
                }
              }
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) rcur[i] = rnext[i];
          }
          continue;
        }
        uint8_t* out16 = reinterpret_cast<uint8_t*>(P.stage_out) + static_cast<int64_t>(kGuard + q) * 16;
#pragma unroll 1
        for (int cbi = 0; cbi < 2; ++cbi) {
          const int cb = cb0 + cbi;
          float v[32];
          tmem_ld32(tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + abuf * 256 + a * 128 + cb * 32, v);
#pragma unroll
          for (int pp = 0; pp < 4; ++pp) {
            const int plane = cb * 4 + pp;
            const float4 b_lo = __ldg(reinterpret_cast<const float4*>(bias + plane * 8));
            const float4 b_hi = __ldg(reinterpret_cast<const float4*>(bias + plane * 8 + 4));
            float o[8] = {v[pp * 8 + 0] + b_lo.x, v[pp * 8 + 1] + b_lo.y, v[pp * 8 + 2] + b_lo.z,
                          v[pp * 8 + 3] + b_lo.w, v[pp * 8 + 4] + b_hi.x, v[pp * 8 + 5] + b_hi.y,
                          v[pp * 8 + 6] + b_hi.z, v[pp * 8 + 7] + b_hi.w};
            if (KIND == 2) {
              if (valid) {
                const float* rp = res + (plane * kPx + px) * 8;
                const float4 r0 = *reinterpret_cast<const float4*>(rp);
                const float4 r1 = *reinterpret_cast<const float4*>(rp + 4);
                o[0] += r0.x; o[1] += r0.y; o[2] += r0.z; o[3] += r0.w;
                o[4] += r1.x; o[5] += r1.y; o[6] += r1.z; o[7] += r1.w;
#pragma unroll
                for (int i = 0; i < 8; ++i) o[i] = fmaxf(o[i], 0.0f);
                float* dp = dst32 + (plane * kPx + px) * 8;
                *reinterpret_cast<float4*>(dp) = make_float4(o[0], o[1], o[2], o[3]);
                *reinterpret_cast<float4*>(dp + 4) = make_float4(o[4], o[5], o[6], o[7]);
              }
            } else {
#pragma unroll
              for (int i = 0; i < 8; ++i) o[i] = valid ? fmaxf(o[i], 0.0f) : 0.0f;
              uint4 pk;
              pk.x = pack_f16x2(o[0], o[1]);
              pk.y = pack_f16x2(o[2], o[3]);
              pk.z = pack_f16x2(o[4], o[5]);
              pk.w = pack_f16x2(o[6], o[7]);
              *reinterpret_cast<uint4*>(out16 + static_cast<int64_t>(plane) * P.ps * 16) = pk;
              if (KIND == 0 && valid) {  // fp32 z for the residual of the block
                float* dp = dst32 + (plane * kPx + px) * 8;
                *reinterpret_cast<float4*>(dp) = make_float4(o[0], o[1], o[2], o[3]);
                *reinterpret_cast<float4*>(dp + 4) = make_float4(o[4], o[5], o[6], o[7]);
              }
            }
          }
        }
      }
}

template <int KIND>
__global__ void __launch_bounds__(kThreads, 1) k_rb_conv(const __grid_constant__ ConvParams P) {
  using K = Cfg<KIND>;
  constexpr int WIN = win<KIND>();
  constexpr uint32_t IDESC = idesc_f16_f32(128, 128);
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = smem + kASlots * a_slot_bytes<KIND>();
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + K::kBStages * kBStage);
  uint64_t* a_full = bars;
  uint64_t* a_empty = a_full + kASlots;
  uint64_t* b_full = a_empty + kASlots;
  uint64_t* b_empty = b_full + K::kBStages;
  uint64_t* acc_full = b_empty + K::kBStages;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

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
#pragma unroll
            for (int a = 0; a < kTileM / 128; ++a) {
#pragma unroll
              for (int kk = 0; kk < 4; ++kk) {
                const uint32_t arow = static_cast<uint32_t>(K::kHalo + shift + a * 128);
                const uint64_t ad = smem_desc(a_slot + ((2 * kk) * WIN + arow) * 16, WIN * 16, 128);
                const uint64_t bd = smem_desc(b_base + s * kBStage + (2 * kk) * 2048, 2048, 128);
                mma_bf16(tmem_base + abuf * 256 + a * 128, ad, bd, IDESC, (ch | tap | kk) != 0);
              }
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
  } else {  // ------------------------------------------------------ epilogue
    const int quarter = warp & 3;
    const int cb0 = ((warp - 2) >> 2) * 2;  // this warp's first 32-column chunk
    int it = 0;
    for (int32_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++it) {
      const int abuf = it & 1;
      const int32_t g = P.tile_group[t_begin + t];
      const int32_t q0 = P.tile_q0[t_begin + t];
      mbar_wait(acc_full + abuf, (it >> 1) & 1);
      tc_fence_after();
      rb_epilogue<KIND>(P, tmem_base, abuf, g, q0, quarter, cb0, lane);
      tc_fence_before();
      mbar_arrive(acc_empty + abuf);
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

// ------------------------------------------------------- CTA-pair kernel
// Cluster of two CTAs on one TPC computes a 512-position pair tile with
// tcgen05.mma.cta_group::2 (M = 256 = 128 rows from each CTA's window,
// N = 128): each CTA stages its own 256-position A window and HALF of every
// weight block (64 output channels), so per-SM shared-memory reads per MMA
// drop from 8 KB to 6 KB and weight traffic per SM halves. The even CTA
// issues the MMAs; the odd CTA relays its "data landed" events to the even
// CTA's barriers (remote mbarrier arrives), and commits multicast back to
// both CTAs' empty / accumulator-full barriers. Each CTA's epilogue reads the
// accumulator rows of its own positions from its own TMEM.
constexpr int kPairBStage = 64 * 64 * 2;  // 8 KB: N=64 (half) × K=64

template <int KIND>
struct PairCfg;
template <>
struct PairCfg<0> { static constexpr int kBStages = 8; };
template <>
struct PairCfg<1> { static constexpr int kBStages = 16; };
template <>
struct PairCfg<2> : PairCfg<1> {};

template <int KIND>
constexpr int pair_smem_bytes() {
  return kASlots * a_slot_bytes<KIND>() + PairCfg<KIND>::kBStages * kPairBStage + 512;
}

template <int KIND>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    k_rb_conv_pair(const __grid_constant__ ConvParams P) {
  using K = Cfg<KIND>;
  constexpr int NB = PairCfg<KIND>::kBStages;
  constexpr int WIN = win<KIND>();
  constexpr uint32_t IDESC = idesc_f16_f32(256, 128);
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = smem + kASlots * a_slot_bytes<KIND>();
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + NB * kPairBStage);
  uint64_t* a_full = bars;
  uint64_t* a_empty = a_full + kASlots;
  uint64_t* b_full = a_empty + kASlots;
  uint64_t* b_empty = b_full + NB;
  uint64_t* acc_full = b_empty + NB;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  if (threadIdx.x == 0) {
    const uint32_t full_count = leader ? 2 : 1;  // own copies + the peer's relay
    for (int s = 0; s < kASlots; ++s) {
      mbar_init(a_full + s, full_count);
      mbar_init(a_empty + s, 1);
    }
    for (int s = 0; s < NB; ++s) {
      mbar_init(b_full + s, full_count);
      mbar_init(b_empty + s, 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(acc_full + s, 1);
      mbar_init(acc_empty + s, 2 * kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair(tmem_slot, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int32_t t_begin = P.step_tile_begin[P.step];
  const int32_t n_tiles = P.step_tile_begin[P.step + 1] - t_begin;
  const int32_t pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------- producer (both CTAs)
      uint32_t ai = 0, bi = 0;
      for (int32_t t = pair; t < n_tiles; t += n_pairs) {
        const int32_t g = P.tile_group[t_begin + t];
        const int32_t q0 = P.tile_q0[t_begin + t] + static_cast<int32_t>(rank) * kTileM;
        const uint8_t* w = reinterpret_cast<const uint8_t*>(P.wpack[P.group_fid[g]]) + rank * kPairBStage;
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
            const uint32_t s = bi % NB, ph = (bi / NB) & 1;
            mbar_wait(b_empty + s, ph ^ 1);
            mbar_expect_tx(b_full + s, kPairBStage);
            bulk_g2s(sB + s * kPairBStage, w + static_cast<int64_t>(ch * K::kTaps + tap) * 2 * kPairBStage,
                     kPairBStage, b_full + s);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {  // ------------------- MMA issuer (even CTA)
      long long w_acc = 0, w_a = 0, w_b = 0;
      const long long t_start = clock64();
      uint32_t ai = 0, bi = 0;
      int it = 0;
      const uint32_t a_base = smem_u32(sA), b_base = smem_u32(sB);
      for (int32_t t = pair; t < n_tiles; t += n_pairs, ++it) {
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
            const uint32_t s = bi % NB, ph = (bi / NB) & 1;
            c0 = clock64();
            mbar_wait(b_full + s, ph);
            w_b += clock64() - c0;
            tc_fence_after();
            const int shift = K::kTaps == 9 ? (tap / 3 - 1) * 15 + (tap % 3 - 1) : 0;
#pragma unroll
            for (int a = 0; a < kTileM / 128; ++a) {
#pragma unroll
              for (int kk = 0; kk < 4; ++kk) {
                const uint32_t arow = static_cast<uint32_t>(K::kHalo + shift + a * 128);
                const uint64_t ad = smem_desc(a_slot + ((2 * kk) * WIN + arow) * 16, WIN * 16, 128);
                const uint64_t bd = smem_desc(b_base + s * kPairBStage + (2 * kk) * 1024, 1024, 128);
                mma_bf16_pair(tmem_base + abuf * 256 + a * 128, ad, bd, IDESC, (ch | tap | kk) != 0);
              }
            }
            mma_commit_pair(b_empty + s, 0x3);
          }
          mma_commit_pair(a_empty + sa, 0x3);
        }
        mma_commit_pair(acc_full + abuf, 0x3);
      }
      if (P.debug) {
        atomicAdd(&g_conv_dbg[12 + KIND * 4 + 0], static_cast<unsigned long long>(w_acc));
        atomicAdd(&g_conv_dbg[12 + KIND * 4 + 1], static_cast<unsigned long long>(w_a));
        atomicAdd(&g_conv_dbg[12 + KIND * 4 + 2], static_cast<unsigned long long>(w_b));
        atomicAdd(&g_conv_dbg[12 + KIND * 4 + 3], static_cast<unsigned long long>(clock64() - t_start));
      }
    } else if (lane == 0) {  // ---------------- relay (odd CTA): data landed
      uint32_t ai = 0, bi = 0;
      for (int32_t t = pair; t < n_tiles; t += n_pairs) {
        for (int ch = 0; ch < K::kChunks; ++ch, ++ai) {
          const uint32_t sa = ai % kASlots, pa = (ai / kASlots) & 1;
          mbar_wait(a_full + sa, pa);
          mbar_arrive_remote(a_full + sa, 0);
          for (int tap = 0; tap < K::kTaps; ++tap, ++bi) {
            const uint32_t s = bi % NB, ph = (bi / NB) & 1;
            mbar_wait(b_full + s, ph);
            mbar_arrive_remote(b_full + s, 0);
          }
        }
      }
    }
  } else {  // ---------------------------------------------- epilogue (both)
    const int quarter = warp & 3;
    const int cb0 = ((warp - 2) >> 2) * 2;
    int it = 0;
    for (int32_t t = pair; t < n_tiles; t += n_pairs, ++it) {
      const int abuf = it & 1;
      const int32_t g = P.tile_group[t_begin + t];
      const int32_t q0 = P.tile_q0[t_begin + t] + static_cast<int32_t>(rank) * kTileM;
      mbar_wait(acc_full + abuf, (it >> 1) & 1);
      tc_fence_after();
      rb_epilogue<KIND>(P, tmem_base, abuf, g, q0, quarter, cb0, lane);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (leader) mbar_arrive(acc_empty + abuf); else mbar_arrive_remote(acc_empty + abuf, 0);
      }
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, 512);
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

template <int KIND>
int launch_conv_pair(const ConvParams& p, int num_sms, cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_rb_conv_pair<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, pair_smem_bytes<KIND>());
    configured = true;
  }
  k_rb_conv_pair<KIND><<<(num_sms / 2) * 2, kThreads, pair_smem_bytes<KIND>(), s>>>(p);
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

extern "C" int dbk_rb_conv(int32_t kind, int32_t step, const int32_t* step_tile_begin,
                           const int32_t* tile_group, const int32_t* tile_q0, const int32_t* group_fid,
                           const int32_t* group_begin, const int32_t* seg_start, const int32_t* member_g,
                           const int32_t* arity_of, const int32_t* fid, const int32_t* child0,
                           const int32_t* example, const void* stage_in, void* stage_out,
                           int64_t plane_stride, const float* inputs, float* values,
                           const void* const* wpack, const float* const* bias, const int32_t* fwd_pos,
                           const int32_t* fwd_slot, void* stage_x, void* stage_cat, int32_t num_sms,
                           void* stream) {
  ConvParams p{step, step_tile_begin, tile_group, tile_q0, group_fid, group_begin, seg_start, member_g,
               arity_of, fid, child0, example, static_cast<const __nv_bfloat16*>(stage_in),
               static_cast<__nv_bfloat16*>(stage_out), plane_stride, inputs, values,
               reinterpret_cast<const __nv_bfloat16* const*>(wpack), bias, fwd_pos, fwd_slot,
               static_cast<__nv_bfloat16*>(stage_x), static_cast<__nv_bfloat16*>(stage_cat), g_debug_flag};
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  switch (kind) {
    case 0: return launch_conv<0>(p, num_sms, s);
    case 1: return launch_conv<1>(p, num_sms, s);
    case 2: return launch_conv<2>(p, num_sms, s);
    case 0 + 16: return launch_conv_pair<0>(p, num_sms, s);  // CTA-pair variants
    case 1 + 16: return launch_conv_pair<1>(p, num_sms, s);
    case 2 + 16: return launch_conv_pair<2>(p, num_sms, s);
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
