// bwd_conv.cu — data gradient of the IEP blocks' 3×3 convolutions as an
// implicit GEMM on the tensor cores (tcgen05, kind::tf32), for the training
// step's backward (iep_train.cpp).
//
//   dX[r] = Σ_t W_tᵀ · dA[r − s_t]      (s_t = 15·dh + dw: the tap's row shift)
//
// over the backward's padded-image rows (PI: per member 16 zero guard rows,
// the 225 positions of the packed 15×15 grid, 16 guard rows), so a tap is a
// row shift of one shared-memory window exactly as in the forward's conv
// (rb_conv.cu): no im2col, no col2im. dA is first packed into 32-channel
// chunk rows of 128 B with the forward's SWIZZLE_128B row swizzle
// (k_pack_sw128f), so every (tile, chunk) window is one bulk copy and the
// MMA descriptor may start at any row.
//
// Per tile of 256 PI rows of one call group: D[ci (M = 128)][rows (N = 256)]
// in TMEM, K = 9 taps × 128 co (tf32, 8 per MMA); A = the function's
// transposed tap weights (16 KB blocks [128 ci][32 co] fp32, SW128), B = the
// dA window at row offset 16 − s_t. The epilogue (8 warps, lane = channel,
// 8×8 transposes to row-major) writes every row of the group's members it
// covers: real positions get D, masked by mid > 0 (conv3x3 #2's gradient) or
// plus the residual dA (conv3x3 #1's); pads and guard rows get 0, so the
// output is again a valid PI operand.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>

#include "dynbatch/dbk.h"
#include "tc_common.cuh"

namespace {

using namespace dbk;

constexpr int kC = 128, kPI = 257, kPIG = 16, kHalo = 16;
constexpr int kTM = 256;                 // PI rows per tile (MMA N)
constexpr int kWin = kTM + 2 * kHalo;    // window rows
constexpr int kSlot = kWin * 128;        // 36 KB: one 32-channel chunk of the window
constexpr int kSlots = 4;
constexpr int kStage = 128 * 128;        // 16 KB weight block: 128 ci × 32 co fp32
constexpr int kStages = 4;
constexpr int kEpiWarps = 8;
constexpr int kThreads = (2 + kEpiWarps + 1) * 32;  // producer, MMA, epilogue × 8, weights
constexpr int kSmem = kSlots * kSlot + kStages * kStage + 256;

__device__ __forceinline__ int shift_of(int tap) { return (tap / 3 - 1) * 15 + (tap % 3 - 1); }

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

constexpr uint32_t idesc_tf32_f32(uint32_t M, uint32_t N) {
  return (1u << 4)            // D format: f32
         | (2u << 7)          // A format: tf32
         | (2u << 10)         // B format: tf32
         | ((N >> 3) << 17)   // N / 8
         | ((M >> 4) << 24);  // M / 16
}

// 8×8 transpose across the 8 lanes of a plane group (as rb_conv.cu).
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

// dA scale from |dA|max (bit pattern of a non-negative float): the largest
// power of two keeping it ≤ 2^14 (1 when dA is all zero).
__device__ __forceinline__ float grad_scale(const uint32_t* absmax_bits) {
  const float m = __uint_as_float(*absmax_bits);
  // the exponent is clamped so the scale and its inverse stay finite
  return m > 0.f && m < INFINITY ? exp2f(fminf(fmaxf(14.f - ceilf(log2f(m)), -100.f), 100.f)) : 1.f;
}

struct DgradParams {
  const uint8_t* src;   // packed dA: [4 chunks][rows_alloc][128 B], row 0 = PI row −lead
  int64_t rows_alloc;   // rows per chunk plane
  int32_t lead;         // zero rows before PI row 0
  int32_t n_tiles;
  const int32_t* tile_row0;  // first PI row of the tile (multiple of 8)
  const int32_t* tile_lo;    // the tile's group: PI rows [lo, hi) are written
  const int32_t* tile_hi;
  const int32_t* tile_fn;    // weight table index
  const uint8_t* const* wpack;  // per function: 9 taps × 4 chunks × 16 KB (tile_fn indexes it)
  const float* mask;    // PI [rows][128]: output ⊙ (mask > 0), or null
  const float* resid;   // PI [rows][128]: output + resid, or null
  float* out;           // PI [rows][128]
  const uint32_t* absmax;  // F16: |dA| max (float bits), the operand scale
  uint32_t* out_absmax;    // |out| max (float bits, atomicMax), or null
  const uint8_t* mask_h;   // the mask as packed fp16 rows (k_stage_to_pack), instead of `mask`, or null
};

// F16: dA packed to fp16 (64 channels per 128-byte row, 2 K chunks, scaled by
// absmax's power of two) with fp16 transposed weights, kind::f16; else fp32
// rows of 32 channels (4 chunks), kind::tf32.
template <bool F16>
__global__ void __launch_bounds__(kThreads, 1) k_tr_dgrad(const __grid_constant__ DgradParams P) {
  constexpr int kChunks = F16 ? 2 : 4;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;                      // window chunks
  uint8_t* sW = smem + kSlots * kSlot;     // weight blocks
  uint64_t* bars = reinterpret_cast<uint64_t*>(sW + kStages * kStage);
  uint64_t* a_full = bars;
  uint64_t* a_empty = a_full + kSlots;
  uint64_t* w_full = a_empty + kSlots;
  uint64_t* w_empty = w_full + kStages;
  uint64_t* acc_full = w_empty + kStages;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kSlots; ++s) {
      mbar_init(a_full + s, 1);
      mbar_init(a_empty + s, 1);
    }
    for (int s = 0; s < kStages; ++s) {
      mbar_init(w_full + s, 1);
      mbar_init(w_empty + s, 1);
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

  if (warp == 0) {
    if (lane == 0) {  // ---------------------------------------- dA windows
      uint32_t ai = 0;
      for (int32_t t = blockIdx.x; t < P.n_tiles; t += gridDim.x) {
        const int64_t r0 = P.lead + P.tile_row0[t] - kHalo;  // window's first packed row
        for (int c = 0; c < kChunks; ++c, ++ai) {
          const uint32_t s = ai % kSlots, par = (ai / kSlots) & 1;
          mbar_wait(a_empty + s, par ^ 1);
          mbar_expect_tx(a_full + s, kSlot);
          bulk_g2s(sA + s * kSlot, P.src + ((static_cast<int64_t>(c) * P.rows_alloc + r0) << 7), kSlot, a_full + s);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ------------------------------------------ MMA issuer
      constexpr uint32_t IDESC = F16 ? idesc_f16_f32(128, kTM) : idesc_tf32_f32(128, kTM);
      const uint32_t a_base = smem_u32(sA), w_base = smem_u32(sW);
      uint32_t ai = 0, wi = 0;
      int n = 0;
      for (int32_t t = blockIdx.x; t < P.n_tiles; t += gridDim.x, ++n) {
        const int abuf = n & 1;
        mbar_wait(acc_empty + abuf, ((n >> 1) & 1) ^ 1);
        tc_fence_after();
        uint32_t acc = 0;
        for (int c = 0; c < kChunks; ++c, ++ai) {
          const uint32_t sa = ai % kSlots;
          mbar_wait(a_full + sa, (ai / kSlots) & 1);
          tc_fence_after();
          for (int tap = 0; tap < 9; ++tap, ++wi) {
            const uint32_t sw = wi % kStages;
            mbar_wait(w_full + sw, (wi / kStages) & 1);
            tc_fence_after();
            const uint32_t row = static_cast<uint32_t>(kHalo - shift_of(tap));
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint64_t wd = smem_desc_sw128(w_base + sw * kStage + kk * 32);
              const uint64_t xd = smem_desc_sw128(a_base + sa * kSlot + row * 128 + kk * 32);
              if (F16) mma_bf16(tmem_base + abuf * kTM, wd, xd, IDESC, acc);
              else mma_tf32(tmem_base + abuf * kTM, wd, xd, IDESC, acc);
              acc = 1;
            }
            mma_commit(w_empty + sw);
          }
          mma_commit(a_empty + sa);
        }
        mma_commit(acc_full + abuf);
      }
    }
  } else if (warp == 2 + kEpiWarps) {
    if (lane == 0) {  // --------------------------------------- weight blocks
      uint32_t wi = 0;
      for (int32_t t = blockIdx.x; t < P.n_tiles; t += gridDim.x) {
        const uint8_t* w = P.wpack[P.tile_fn[t]];
        for (int c = 0; c < kChunks; ++c)
          for (int tap = 0; tap < 9; ++tap, ++wi) {
            const uint32_t s = wi % kStages, par = (wi / kStages) & 1;
            mbar_wait(w_empty + s, par ^ 1);
            mbar_expect_tx(w_full + s, kStage);
            bulk_g2s(sW + s * kStage, w + static_cast<int64_t>(tap * kChunks + c) * kStage, kStage, w_full + s);
          }
      }
    }
  } else {  // ---------------------------------------------------- epilogue
    const int quarter = warp & 3, half = (warp - 2) >> 2;
    const int g = lane >> 3, e = lane & 7;
    const int plane = quarter * 4 + g;  // 8 channels: ci = 8·plane + k
    const float inv = F16 ? 1.f / grad_scale(P.absmax) : 1.f;
    int n = 0;
    for (int32_t t = blockIdx.x; t < P.n_tiles; t += gridDim.x, ++n) {
      const int abuf = n & 1;
      mbar_wait(acc_full + abuf, (n >> 1) & 1);
      tc_fence_after();
      const int32_t row0 = P.tile_row0[t], lo = P.tile_lo[t], hi = P.tile_hi[t];
      const uint32_t taddr = tmem_base + abuf * kTM + (static_cast<uint32_t>(quarter * 32) << 16) + half * (kTM / 2);
      // the mask (mid) or residual rows of the next 16-position chunk are
      // loaded while this chunk is transposed and stored (they are the
      // epilogue's only reads; issued just before use they stall it)
      const float* aux = P.mask ? P.mask : P.resid;
      const bool is_mask = P.mask != nullptr || P.mask_h != nullptr;
      const bool packed_mask = P.mask_h != nullptr;
      auto row_of = [&](int cb, int m) { return row0 + half * (kTM / 2) + cb * 16 + 8 * m + e; };
      auto real_row = [&](int32_t r) {
        if (r < lo || r >= hi) return false;
        const int32_t p = r % kPI - kPIG;
        return p >= 0 && p < 225 && p / 15 < 14 && p % 15 < 14;
      };
      // raw 16-byte loads, converted only where used (a conversion right
      // after the load would wait for it and undo the prefetch)
      uint4 nxt[4];
      auto load_aux = [&](int cb) {
#pragma unroll
        for (int m = 0; m < 2; ++m) {
          const int32_t r = row_of(cb, m);
          nxt[2 * m] = nxt[2 * m + 1] = make_uint4(0, 0, 0, 0);
          if (packed_mask && real_row(r)) {  // 8 fp16 channels of plane `plane` in the packed row
            const int64_t pr = P.lead + r;
            nxt[2 * m] = __ldg(reinterpret_cast<const uint4*>(
                P.mask_h + (((static_cast<int64_t>(plane >> 3) * P.rows_alloc + pr) << 7) +
                            (((plane & 7) ^ static_cast<int>(pr & 7)) << 4))));
          } else if (aux && real_row(r)) {
            const uint4* a = reinterpret_cast<const uint4*>(aux + static_cast<int64_t>(r) * kC + plane * 8);
            nxt[2 * m] = __ldg(a);
            nxt[2 * m + 1] = __ldg(a + 1);
          }
        }
      };
      load_aux(0);
      float omax = 0.f;
#pragma unroll 1
      for (int cb = 0; cb < kTM / 2 / 16; ++cb) {
        uint4 cur[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) cur[i] = nxt[i];
        if (cb + 1 < kTM / 2 / 16) load_aux(cb + 1);
        float v[16];
        tmem_ld16(taddr + cb * 16, v);
#pragma unroll
        for (int m = 0; m < 2; ++m) {
          float* x = v + 8 * m;
          transpose8(x, e);
          if (F16) {
#pragma unroll
            for (int k = 0; k < 8; ++k) x[k] *= inv;
          }
          const int32_t r = row_of(cb, m);
          if (r < lo || r >= hi) continue;
          float au[8];
          if (packed_mask) {
            const __half2* h2 = reinterpret_cast<const __half2*>(&cur[2 * m]);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float2 f = __half22float2(h2[q]);
              au[2 * q] = f.x;
              au[2 * q + 1] = f.y;
            }
          } else {
            const float* f = reinterpret_cast<const float*>(&cur[2 * m]);
#pragma unroll
            for (int q = 0; q < 8; ++q) au[q] = f[q];  // cur[2m], cur[2m + 1] are adjacent
          }
          float o[8];
          if (real_row(r)) {
#pragma unroll
            for (int k = 0; k < 8; ++k) o[k] = is_mask ? (au[k] > 0.f ? x[k] : 0.f) : (aux ? x[k] + au[k] : x[k]);
          } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) o[k] = 0.f;
          }
          float4* dst = reinterpret_cast<float4*>(P.out + static_cast<int64_t>(r) * kC + plane * 8);
          dst[0] = make_float4(o[0], o[1], o[2], o[3]);
          dst[1] = make_float4(o[4], o[5], o[6], o[7]);
#pragma unroll
          for (int k = 0; k < 8; ++k) omax = fmaxf(omax, fabsf(o[k]));
        }
      }
      if (P.out_absmax) {  // the next gradient's fp16 scale
        for (int o = 16; o; o >>= 1) omax = fmaxf(omax, __shfl_xor_sync(0xffffffffu, omax, o));
        if (lane == 0 && omax > 0.f) atomicMax(P.out_absmax, __float_as_uint(omax));
      }
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

// PI rows [0, rows) fp32 [rows][128] → 4 chunk planes of 128-byte rows
// (32 channels each), 16-byte pieces XOR-swizzled by row; `lead` zero rows
// before PI row 0 and the rest of rows_alloc zero (halo reads past either end).
__global__ void k_pack_sw128f(int64_t rows, int64_t rows_alloc, int32_t lead, const float* __restrict__ pi,
                              uint8_t* __restrict__ out) {
  // the rows any window of this call reads: the lead, the PI rows, one
  // tile plus halo past the end (zeros)
  const int64_t used = min(rows_alloc, lead + rows + kWin);
  const int64_t total = 4 * used * 8;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int j = static_cast<int>(i & 7);         // 16-byte piece: channels 4j .. 4j + 3 of the chunk
    const int64_t q = i >> 3;
    const int c = static_cast<int>(q / used);
    const int64_t rr = q - static_cast<int64_t>(c) * used;  // packed row
    const int64_t r = rr - lead;                                   // PI row
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (r >= 0 && r < rows) v = *reinterpret_cast<const float4*>(pi + r * kC + c * 32 + 4 * j);
    *reinterpret_cast<float4*>(out + ((static_cast<int64_t>(c) * rows_alloc + rr) << 7) +
                               ((j ^ static_cast<int>(rr & 7)) << 4)) = v;
  }
}

// one thread per 16-byte piece: 9 taps × 4 chunks × 128 rows (ci) × 8 pieces
__global__ void k_pack_dgrad_w(const float* __restrict__ w, uint8_t* __restrict__ out) {
  constexpr int kChunks = 4;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 9 * kChunks * 128 * 8) return;
  const int j = i & 7, ci = (i >> 3) & 127, blk = i >> 10;  // blk = tap · 4 + chunk
  const int tap = blk / kChunks, c = blk % kChunks;
  const float* src = w + (static_cast<int64_t>(tap) * kC + ci) * kC + c * 32 + 4 * j;
  *reinterpret_cast<float4*>(out + static_cast<int64_t>(blk) * kStage + ci * 128 + ((j ^ (ci & 7)) << 4)) =
      *reinterpret_cast<const float4*>(src);
}

// fp16 version: 9 taps × 2 chunks of 64 co, row ci = 128 B of 8 pieces of 8 co.
__global__ void k_pack_dgrad_wh(const float* __restrict__ w, uint8_t* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 9 * 2 * 128 * 8) return;
  const int j = i & 7, ci = (i >> 3) & 127, blk = i >> 10;  // blk = tap · 2 + chunk
  const int tap = blk / 2, c = blk % 2;
  const float* src = w + (static_cast<int64_t>(tap) * kC + ci) * kC + c * 64 + 8 * j;
  uint4 h;
  h.x = pack_f16x2(src[0], src[1]);
  h.y = pack_f16x2(src[2], src[3]);
  h.z = pack_f16x2(src[4], src[5]);
  h.w = pack_f16x2(src[6], src[7]);
  *reinterpret_cast<uint4*>(out + static_cast<int64_t>(blk) * kStage + ci * 128 + ((j ^ (ci & 7)) << 4)) = h;
}


// ------------------------------------------------------------ weight gradient
// dW_t[ci][co] = Σ_r x[r + s_t][ci] · dA[r][co]. Both operands are read
// MN-major (a 128-byte row = one K index = 64 channels of M or N; the two
// 64-channel planes are the MN blocks, LBO apart; 8-row groups 1024 B apart),
// so a tap is again a row offset of the x window and nothing is expanded.
// MN-major operands exist for 16-bit formats only (a kind::tf32 MMA with
// MN-major operands produces zeros: tools/mn_major_test.cu), so x and dA are
// packed to fp16 (k_pack_sw128h), dA scaled by a power of two from its
// maximum (k_absmax) so the gradients sit in fp16's normal range. One work
// item = (call group, kernel row dr, K range): D[ci][3 × 128 co] in TMEM over
// 64-row K blocks (K = 16 per MMA); the epilogue adds D / scale into the
// function's fp32 gradient (input-major w[(t·C + ci)·C + co]) with vector
// atomics, straight from TMEM (lane = ci, columns = co: no transposes).
constexpr int kWB = 64;                     // K rows per block
constexpr int kXW = kWB + 16;               // x window rows (3 shifts + 8-row alignment)
constexpr int kWDa = 2 * kWB * 128;         // 16 KB: dA block, 2 planes
constexpr int kWX = 2 * kXW * 128;          // 20 KB: x window, 2 planes
constexpr int kWStage = kWDa + kWX;
constexpr int kWStages = 6;
constexpr int kWSmem = kWStages * kWStage + 256;

// MN-major SWIZZLE_128B descriptor: MN blocks of 128 B `lbo` bytes apart,
// K rows 128 B apart in 8-row groups of 1024 B.
__device__ __forceinline__ uint64_t smem_desc_mn128(uint32_t saddr, uint32_t lbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;  // LBO: next MN block
  d |= static_cast<uint64_t>(1024 >> 4) << 32;            // SBO: next 8 K rows
  d |= static_cast<uint64_t>(1) << 46;                    // descriptor version (sm_100)
  d |= static_cast<uint64_t>(2) << 61;                    // SWIZZLE_128B
  return d;
}

struct WgradParams {
  const uint8_t* x;      // packed fp16 activations (x or mid), k_pack_sw128h
  const uint8_t* da;     // packed fp16 dA, scaled
  const uint32_t* absmax;  // |dA| max (float bits): the scale
  int64_t rows_alloc;
  int32_t lead;
  int32_t n_items;
  int64_t stride;        // between the item table's four columns
  const int32_t* item;   // [4][stride]: k0, k1 (PI rows, multiples of 16), dr, function
  float* const* gw;      // per function: fp32 gradient, input-major [9·C][C]
};

__global__ void __launch_bounds__(kThreads, 1) k_tr_wgrad(const __grid_constant__ WgradParams P) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kWStages * kWStage);
  uint64_t* full = bars;
  uint64_t* empty = full + kWStages;
  uint64_t* acc_full = empty + kWStages;
  uint64_t* acc_empty = acc_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t n = P.n_items;
  const int32_t* k0s = P.item;
  const int32_t* k1s = P.item + P.stride;
  const int32_t* drs = P.item + 2 * P.stride;
  const int32_t* fns = P.item + 3 * P.stride;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kWStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, kEpiWarps * 32);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------ producer
      uint32_t bi = 0;
      for (int32_t it = blockIdx.x; it < n; it += gridDim.x) {
        const int32_t k0 = k0s[it], k1 = k1s[it], sh = 15 * (drs[it] - 1);
        for (int32_t kb = k0; kb < k1; kb += kWB, ++bi) {
          const uint32_t s = bi % kWStages;
          mbar_wait(empty + s, ((bi / kWStages) & 1) ^ 1);
          mbar_expect_tx(full + s, kWStage);
          uint8_t* st = smem + s * kWStage;
          const int64_t ws = ((kb + sh - 1) >> 3) << 3;  // x window start row (8-aligned)
          for (int c = 0; c < 2; ++c) {
            bulk_g2s(st + c * (kWB * 128), P.da + ((static_cast<int64_t>(c) * P.rows_alloc + P.lead + kb) << 7),
                     kWB * 128, full + s);
            bulk_g2s(st + kWDa + c * (kXW * 128),
                     P.x + ((static_cast<int64_t>(c) * P.rows_alloc + P.lead + ws) << 7), kXW * 128, full + s);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ------------------------------------------ MMA issuer
      constexpr uint32_t IDESC = idesc_f16_f32(128, 128) | (1u << 15) | (1u << 16);  // A, B MN-major
      const uint32_t base = smem_u32(smem);
      uint32_t bi = 0;
      int j = 0;
      for (int32_t it = blockIdx.x; it < n; it += gridDim.x, ++j) {
        const int32_t k0 = k0s[it], k1 = k1s[it], sh = 15 * (drs[it] - 1);
        mbar_wait(acc_empty, (j & 1) ^ 1);
        tc_fence_after();
        uint32_t acc = 0;
        for (int32_t kb = k0; kb < k1; kb += kWB, ++bi) {
          const uint32_t s = bi % kWStages;
          mbar_wait(full + s, (bi / kWStages) & 1);
          tc_fence_after();
          const uint32_t st = base + s * kWStage;
          const int32_t ws = ((kb + sh - 1) >> 3) << 3;
          const int32_t steps = min(kWB, k1 - kb) / 16;
          for (int kk = 0; kk < steps; ++kk) {
            const uint64_t bd = smem_desc_mn128(st + kk * 16 * 128, kWB * 128);
#pragma unroll
            for (int dc = 0; dc < 3; ++dc) {
              const uint32_t xr = static_cast<uint32_t>(kb + sh + dc - 1 + 16 * kk - ws);
              const uint64_t ad = smem_desc_mn128(st + kWDa + xr * 128, kXW * 128);
              mma_bf16(tmem_base + dc * 128, ad, bd, IDESC, acc);
            }
            acc = 1;
          }
          mma_commit(empty + s);
        }
        mma_commit(acc_full);
      }
    }
  } else if (warp >= 2 && warp < 2 + kEpiWarps) {  // -------------- epilogue
    const int quarter = warp & 3, half = (warp - 2) >> 2;
    const int ci = quarter * 32 + lane;
    const float inv = 1.f / grad_scale(P.absmax);
    int j = 0;
    for (int32_t it = blockIdx.x; it < n; it += gridDim.x, ++j) {
      mbar_wait(acc_full, j & 1);
      tc_fence_after();
      float* gw = P.gw[fns[it]];
      const int dr = drs[it];
      for (int cb = 0; cb < 6; ++cb) {  // this warp's 192 of the 384 columns, 32 at a time
        const int col = half * 192 + cb * 32;
        float v[32];
        tmem_ld32(tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + col, v);
        const int dc = col / 128, co = col % 128;
        float* dst = gw + (static_cast<int64_t>(3 * dr + dc) * kC + ci) * kC + co;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          atomicAdd(reinterpret_cast<float4*>(dst + 4 * q),
                    make_float4(v[4 * q] * inv, v[4 * q + 1] * inv, v[4 * q + 2] * inv, v[4 * q + 3] * inv));
      }
      tc_fence_before();
      mbar_arrive(acc_empty);
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

// PI rows fp32 [rows][128] → 2 planes of 128-byte rows (64 fp16 channels),
// 16-byte pieces XOR-swizzled by row, times the scale from `absmax` (null: 1);
// `lead` zero rows first, zeros up to one window past the end.
__global__ void k_pack_sw128h(int64_t rows, int64_t rows_alloc, int32_t lead, const float* __restrict__ pi,
                              const uint32_t* __restrict__ absmax, uint8_t* __restrict__ out) {
  const float sc = absmax ? grad_scale(absmax) : 1.f;
  const int64_t used = min(rows_alloc, lead + rows + kWin);
  const int64_t total = 2 * used * 8;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int j = static_cast<int>(i & 7);  // 16-byte piece: channels 8j .. 8j + 7 of the plane
    const int64_t q = i >> 3;
    const int c = static_cast<int>(q / used);
    const int64_t rr = q - static_cast<int64_t>(c) * used;
    const int64_t r = rr - lead;
    uint4 h = make_uint4(0, 0, 0, 0);
    if (r >= 0 && r < rows) {
      const float4 a = *reinterpret_cast<const float4*>(pi + r * kC + c * 64 + 8 * j);
      const float4 b = *reinterpret_cast<const float4*>(pi + r * kC + c * 64 + 8 * j + 4);
      h.x = pack_f16x2(a.x * sc, a.y * sc);
      h.y = pack_f16x2(a.z * sc, a.w * sc);
      h.z = pack_f16x2(b.x * sc, b.y * sc);
      h.w = pack_f16x2(b.z * sc, b.w * sc);
    }
    *reinterpret_cast<uint4*>(out + ((static_cast<int64_t>(c) * rows_alloc + rr) << 7) +
                              ((j ^ static_cast<int>(rr & 7)) << 4)) = h;
  }
}

// |x| max over n floats into *out (float bits, atomicMax; *out zeroed first).
__global__ void k_absmax(int64_t n, const float* __restrict__ x, uint32_t* __restrict__ out) {
  float m = 0.f;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n / 4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float4 v = reinterpret_cast<const float4*>(x)[i];
    m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
  }
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0.f) atomicMax(out, __float_as_uint(m));
}


// The forward's staged fp16 rows of n members (member k's image at staging
// row kGuard + srows[k], 64-channel chunk planes ps rows apart, row-swizzled)
// → the packed backward rows (PI order: 16 guard rows, 225 positions, 16
// guard rows per member; `lead` zero rows first, zeros one window past the
// end), the MN-major weight-gradient operand and the data gradient's mask
// with no fp32 round trip.
__global__ void k_stage_to_pack(int32_t n, const int64_t* __restrict__ srows, const uint8_t* __restrict__ hi,
                                int64_t ps, int64_t rows_alloc, int32_t lead, uint8_t* __restrict__ out) {
  const int64_t rows = static_cast<int64_t>(n) * kPI;
  const int64_t used = min(rows_alloc, lead + rows + kWin);
  const int64_t total = 2 * used * 8;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int j = static_cast<int>(i & 7);
    const int64_t q = i >> 3;
    const int c = static_cast<int>(q / used);
    const int64_t R = q - static_cast<int64_t>(c) * used;
    const int64_t r = R - lead;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (r >= 0 && r < rows) {
      const int32_t k = static_cast<int32_t>(r / kPI);
      const int p = static_cast<int>(r - static_cast<int64_t>(k) * kPI) - kPIG;
      if (p >= 0 && p < 225) {
        const int64_t srow = 32 + srows[k] + p;  // rb_conv.cu kGuard
        v = __ldg(reinterpret_cast<const uint4*>(hi + ((static_cast<int64_t>(c) * ps + srow) << 7) +
                                                  ((j ^ static_cast<int>(srow & 7)) << 4)));
      }
    }
    *reinterpret_cast<uint4*>(out + ((static_cast<int64_t>(c) * rows_alloc + R) << 7) +
                              ((j ^ static_cast<int>(R & 7)) << 4)) = v;
  }
}

// out[r − r0][c] = g[r][c] if the packed fp16 activation at (r, c) > 0, else
// 0, over PI rows [r0, r0 + n) (the binary blocks' z mask).
__global__ void k_mask_h(int64_t r0, int64_t n, const float* __restrict__ g, const uint8_t* __restrict__ packed,
                         int64_t rows_alloc, int32_t lead, float* __restrict__ out) {
  const int64_t total = n * 16;  // 8-channel planes
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int plane = static_cast<int>(i & 15);
    const int64_t r = r0 + (i >> 4);
    const int64_t pr = lead + r;
    const uint4 h = __ldg(reinterpret_cast<const uint4*>(packed + (((static_cast<int64_t>(plane >> 3) * rows_alloc + pr) << 7) +
                                                                   (((plane & 7) ^ static_cast<int>(pr & 7)) << 4))));
    const __half* z = reinterpret_cast<const __half*>(&h);
    const float4* gp = reinterpret_cast<const float4*>(g + r * kC + plane * 8);
    const float4 a = gp[0], b = gp[1];
    float4* op = reinterpret_cast<float4*>(out + (r - r0) * kC + plane * 8);
    op[0] = make_float4(__half2float(z[0]) > 0.f ? a.x : 0.f, __half2float(z[1]) > 0.f ? a.y : 0.f,
                        __half2float(z[2]) > 0.f ? a.z : 0.f, __half2float(z[3]) > 0.f ? a.w : 0.f);
    op[1] = make_float4(__half2float(z[4]) > 0.f ? b.x : 0.f, __half2float(z[5]) > 0.f ? b.y : 0.f,
                        __half2float(z[6]) > 0.f ? b.z : 0.f, __half2float(z[7]) > 0.f ? b.w : 0.f);
  }
}

}  // namespace

extern "C" int dbk_tr_pack_sw128f(int64_t rows, int64_t rows_alloc, int32_t lead, const float* pi, void* out,
                                  void* stream) {
  const int64_t total = 4 * std::min<int64_t>(rows_alloc, lead + rows + kWin) * 8;
  if (total <= 0) return 0;
  const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((total + 255) / 256, 148 * 16));
  k_pack_sw128f<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(rows, rows_alloc, lead, pi,
                                                                        static_cast<uint8_t*>(out));
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_tr_dgrad(const void* packed, int32_t f16, const uint32_t* absmax, int64_t rows_alloc,
                            int32_t lead, int32_t n_tiles, const int32_t* tile_row0, const int32_t* tile_lo,
                            const int32_t* tile_hi, const int32_t* tile_fn, const void* const* wpack, const float* mask,
                            const void* mask_h, const float* resid, float* out, uint32_t* out_absmax, int32_t sms,
                            void* stream) {
  if (n_tiles <= 0) return 0;
  static std::atomic<uint64_t> configured{0};  // per device, once
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (!(configured.load(std::memory_order_acquire) & bit)) {
    cudaFuncSetAttribute(k_tr_dgrad<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    cudaFuncSetAttribute(k_tr_dgrad<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    configured.fetch_or(bit, std::memory_order_release);
  }
  DgradParams p;
  p.src = static_cast<const uint8_t*>(packed);
  p.rows_alloc = rows_alloc;
  p.lead = lead;
  p.n_tiles = n_tiles;
  p.tile_row0 = tile_row0;
  p.tile_lo = tile_lo;
  p.tile_hi = tile_hi;
  p.tile_fn = tile_fn;
  p.wpack = reinterpret_cast<const uint8_t* const*>(wpack);
  p.mask = mask;
  p.resid = resid;
  p.out = out;
  p.absmax = absmax;
  p.out_absmax = out_absmax;
  p.mask_h = static_cast<const uint8_t*>(mask_h);
  const unsigned grid = static_cast<unsigned>(std::min(n_tiles, std::max(sms, 1)));
  if (f16) k_tr_dgrad<true><<<grid, kThreads, kSmem, static_cast<cudaStream_t>(stream)>>>(p);
  else k_tr_dgrad<false><<<grid, kThreads, kSmem, static_cast<cudaStream_t>(stream)>>>(p);
  return static_cast<int>(cudaGetLastError());
}

// Transposed tap weights of one function for k_tr_dgrad, from the
// input-major fp32 weights w[(tap·C + ci)·C + co] (= W_tap[co][ci]): block
// (tap, chunk c) row ci holds co = 32c .. 32c + 31, swizzled like the windows.
extern "C" int dbk_tr_pack_dgrad_weights(const float* w, void* out, void* stream) {
  k_pack_dgrad_w<<<9 * 4 * 128 * 8 / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      w, static_cast<uint8_t*>(out));
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_tr_pack_dgrad_weights_h(const float* w, void* out, void* stream) {
  k_pack_dgrad_wh<<<9 * 2 * 128 * 8 / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      w, static_cast<uint8_t*>(out));
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_tr_pack_sw128h(int64_t rows, int64_t rows_alloc, int32_t lead, const float* pi,
                                  const uint32_t* absmax, void* out, void* stream) {
  const int64_t total = 2 * std::min<int64_t>(rows_alloc, lead + rows + kWin) * 8;
  if (total <= 0) return 0;
  const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((total + 255) / 256, 148 * 16));
  k_pack_sw128h<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(rows, rows_alloc, lead, pi, absmax,
                                                                        static_cast<uint8_t*>(out));
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_tr_absmax(int64_t n, const float* x, uint32_t* out, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaMemsetAsync(out, 0, sizeof(uint32_t), s);
  if (n <= 0) return static_cast<int>(cudaGetLastError());
  const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((n / 4 + 255) / 256, 148 * 8));
  k_absmax<<<std::max(blocks, 1u), 256, 0, s>>>(n, x, out);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_tr_wgrad(const void* x_packed, const void* da_packed, const uint32_t* absmax, int64_t rows_alloc,
                            int32_t lead, int32_t n_items, const int32_t* items, int64_t item_stride, float* const* gw,
                            int32_t sms, void* stream) {
  if (n_items <= 0) return 0;
  static std::atomic<uint64_t> configured{0};  // per device, once
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (!(configured.load(std::memory_order_acquire) & bit)) {
    cudaFuncSetAttribute(k_tr_wgrad, cudaFuncAttributeMaxDynamicSharedMemorySize, kWSmem);
    configured.fetch_or(bit, std::memory_order_release);
  }
  WgradParams p;
  p.x = static_cast<const uint8_t*>(x_packed);
  p.da = static_cast<const uint8_t*>(da_packed);
  p.absmax = absmax;
  p.rows_alloc = rows_alloc;
  p.lead = lead;
  p.n_items = n_items;
  p.stride = item_stride;
  p.item = items;
  p.gw = gw;
  k_tr_wgrad<<<static_cast<unsigned>(std::min(n_items, std::max(sms, 1))), kThreads, kWSmem,
               static_cast<cudaStream_t>(stream)>>>(p);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_tr_stage_to_pack(int32_t n, const int64_t* srows, const void* hi, int64_t plane_stride,
                                    int64_t rows_alloc, int32_t lead, void* out, void* stream) {
  const int64_t total = 2 * std::min<int64_t>(rows_alloc, lead + static_cast<int64_t>(n) * kPI + kWin) * 8;
  if (total <= 0) return 0;
  const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((total + 255) / 256, 148 * 16));
  k_stage_to_pack<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      n, srows, static_cast<const uint8_t*>(hi), plane_stride, rows_alloc, lead, static_cast<uint8_t*>(out));
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_tr_mask_h(int64_t r0, int64_t n, const float* g, const void* packed, int64_t rows_alloc,
                             int32_t lead, float* out, void* stream) {
  if (n <= 0) return 0;
  const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((n * 16 + 255) / 256, 148 * 16));
  k_mask_h<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(r0, n, g, static_cast<const uint8_t*>(packed),
                                                                  rows_alloc, lead, out);
  return static_cast<int>(cudaGetLastError());
}
