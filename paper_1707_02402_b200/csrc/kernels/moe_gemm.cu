// moe_gemm.cu — tensor-core MoE experts: dispatch → grouped GEMM1+ReLU
// → grouped GEMM2 → slot-order combine (sm_100a, tcgen05/TMEM).
//
// Operand format (fmt): DBK_FMT_F16 (fp16 operands, H and Y; the precise
// mode, ≤ 1e-3 max-norm vs the fp64 reference) or DBK_FMT_BF16 (bf16; wider
// range, ≈4e-3). Both run tcgen05.mma kind::f16 at the same rate with fp32
// accumulation; only the idesc A/B format bits and the packing differ.
//
// Reference semantics: ExpertSet::apply (src/moe.cpp:98-145) on each
// occupied expert's stacked rows, staged at token·k + slot (:244-251),
// combined per token in slot order (:254-264). Routing (ids, weights, the
// stable per-expert item order and offsets) comes from moe.cu / sched.cu and
// is bit-identical to the reference; the arithmetic here is 16-bit operands
// with fp32 accumulation.
//
// Layout: rows of expert e occupy a 128-aligned padded range starting at
// pstart[e]. Activations are stored pre-tiled, so each pipeline stage is one
// bulk copy of a contiguous 16 KB block per (row block rb, K chunk kc):
//  * GEMM1's A (the dispatched x rows) in the K-major SWIZZLE_128B layout:
//    row r's 64 elements are the 128-byte line r, 16-byte piece j at slot
//    j ^ (r & 7) — a dispatched row is written as whole lines;
//  * GEMM2's A (H, written by GEMM1's epilogue) in the K-major SWIZZLE_NONE
//    layout [8 k-groups][128 rows][8 elements].
// Weights are pre-tiled SWIZZLE_NONE per (N tile, K chunk): [8][256 n][8].
// Padding rows of A and H are never initialised: their GEMM rows are never
// read (the combine reads valid rows only; the EP GEMM2 skips them).
#include <atomic>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "dynbatch/dbk.h"
#include "tc_common.cuh"

namespace {

using namespace dbk;

// Two fp32 values → one 32-bit pair of 16-bit operands (round to nearest).
template <bool F16>
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  return F16 ? pack_f16x2(lo, hi) : pack_bf16x2(lo, hi);
}
template <bool F16>
__device__ __forceinline__ float2 unpack2(uint32_t v) {
  if constexpr (F16) {
    return __half22float2(*reinterpret_cast<const __half2*>(&v));
  } else {
    return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v));
  }
}

constexpr int kBM = 128;         // rows per tile
constexpr int kBN = 256;         // output columns per tile
constexpr int kBK = 64;          // K chunk
constexpr int kABytes = kBM * kBK * 2;   // 16 KB
constexpr int kBBytes = kBN * kBK * 2;   // 32 KB
constexpr int kPairRows = 2 * kBM;  // experts are padded to whole 256-row tile pairs
constexpr int kBHalf = kBBytes / 2;  // 16 KB: this CTA's 128 of the 256 output columns
constexpr int kStages = 6;
constexpr int kEpiWarps = 8;
constexpr int kThreads = 64 + kEpiWarps * 32;
constexpr int kSmem = kStages * (kABytes + kBHalf) + 256;

// Padded starts and the (expert, row block) tile list: one thread per
// expert, a block-wide scan of the row blocks (single block, n ≤ 1024 × k).
__global__ void __launch_bounds__(1024) k_moe_layout(int32_t n, const int32_t* __restrict__ offsets,
                                                     int32_t* __restrict__ pstart, int32_t* __restrict__ tile_expert,
                                                     int32_t* __restrict__ tile_rb, int32_t* __restrict__ n_tiles) {
  __shared__ int32_t wsum[32];
  __shared__ int32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int32_t base = 0; base < n; base += blockDim.x) {
    const int32_t e = base + static_cast<int32_t>(threadIdx.x);
    const int32_t nb = e < n ? (offsets[e + 1] - offsets[e] + kPairRows - 1) / kPairRows * 2 : 0;
    int32_t x = nb;  // inclusive warp scan, then across warps
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int32_t w = lane < static_cast<int>(blockDim.x >> 5) ? wsum[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      wsum[lane] = w;
    }
    __syncthreads();
    const int32_t first = carry + (warp > 0 ? wsum[warp - 1] : 0) + x - nb;  // exclusive prefix (row blocks)
    if (e < n) {
      pstart[e] = first * kBM;
      for (int32_t b = 0; b < nb; ++b) {
        tile_expert[first + b] = e;
        tile_rb[first + b] = first + b;
      }
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = first + nb;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    pstart[n] = carry * kBM;
    *n_tiles = carry;
  }
}

// Padded row of every item: the item at sorted position pos belongs to
// expert e = ids[item] and sits at row pstart[e] + (pos − offsets[e]).
__global__ void k_moe_item_rows(int64_t items, const int32_t* __restrict__ order, const int32_t* __restrict__ ids,
                                const int32_t* __restrict__ offsets, const int32_t* __restrict__ pstart,
                                int32_t* __restrict__ row_of_item) {
  for (int64_t pos = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; pos < items;
       pos += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t item = order[pos];
    const int32_t e = ids[item];
    row_of_item[item] = pstart[e] + static_cast<int32_t>(pos) - offsets[e];
  }
}

// Byte offset of 16-byte piece j (elements 8j..8j+7 of K chunk kc) of padded
// row `row` in the SWIZZLE_128B tiled A.
__device__ __forceinline__ int64_t a_sw128_off(int32_t row, int32_t kchunks, int32_t kc, int32_t j) {
  const int32_t rb = row / kBM, rr = row % kBM;
  return (static_cast<int64_t>(rb) * kchunks + kc) * kABytes + rr * 128 + ((j ^ (rr & 7)) << 4);
}

// Token-major dispatch: one warp per token reads its fp32 row once
// (coalesced) and writes the 16-bit row into each of its k items' padded rows,
// whole 128-byte lines (lane group g = lane / 8 covers K chunk 4·it + g,
// lane e = lane % 8 its 16-byte piece e).
template <bool F16>
__global__ void k_moe_dispatch(int64_t T, int32_t k, int32_t d, const float* __restrict__ x,
                               const int32_t* __restrict__ row_of_item, uint8_t* __restrict__ A) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  const int32_t kchunks = d / kBK;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x >> 5) + (threadIdx.x >> 5); t < T; t += warps) {
    const float* src = x + t * d;
    int32_t rows[8];
#pragma unroll
    for (int s = 0; s < 8; ++s) rows[s] = s < k ? row_of_item[t * k + s] : 0;
    // four 1 KB rounds of the row in flight before any is written
    for (int32_t it0 = 0; it0 * 256 < d; it0 += 4) {
      float4 a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int32_t col = (it0 + u) * 256 + lane * 8;
        if (col < d) {
          a[u] = __ldg(reinterpret_cast<const float4*>(src + col));
          b[u] = __ldg(reinterpret_cast<const float4*>(src + col + 4));
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int32_t col = (it0 + u) * 256 + lane * 8;
        if (col >= d) break;
        uint4 pk;
        pk.x = pack2<F16>(a[u].x, a[u].y);
        pk.y = pack2<F16>(a[u].z, a[u].w);
        pk.z = pack2<F16>(b[u].x, b[u].y);
        pk.w = pack2<F16>(b[u].z, b[u].w);
        const int32_t kc = col / kBK, j = (col % kBK) / 8;
#pragma unroll
        for (int s = 0; s < 8; ++s)
          if (s < k) *reinterpret_cast<uint4*>(A + a_sw128_off(rows[s], kchunks, kc, j)) = pk;
      }
    }
  }
}

struct GemmParams {
  int32_t n_experts;
  int32_t K;                    // reduction length (multiple of 64)
  int32_t N;                    // output columns (multiple of 256)
  const int32_t* n_tiles;       // device scalar: row tiles
  const int32_t* tile_expert;
  const int32_t* tile_rb;
  const uint8_t* A;             // tiled activations [rb][K/64][16 KB]
  const uint8_t* const* W;      // per expert tiled weights [N/256][K/64][32 KB]
  uint8_t* H;                   // EPI 0: tiled 16-bit output [rb][N/64][16 KB]
  uint16_t* Y;                  // EPI 1: 16-bit row-major [row][N]
  int32_t tile_begin, tile_end;  // row-tile range (tile_end < 0: up to *n_tiles)
  const int32_t* out_row;        // EPI 1 / 2: Y row of padded row r = out_row[r] (< 0: skip); null = r
  const float* const* bias;      // per expert fp32 [N] added before the epilogue's activation; null = none
  float* Yf;                     // EPI 2: fp32 row-major [row][N]
};

// Grouped GEMM over (row-tile pair, N tile) units on CTA pairs
// (tcgen05.mma.cta_group::2): M = 256 rows, 128 from each CTA's A tile of
// one expert, N = 256 columns, each CTA staging half of the weight tile, so
// per SM the A + B bytes per MMA fall from 12 KB to 8 KB and the weight
// reads from L2 halve. The even CTA issues the MMAs. The odd CTA relays its
// "stage landed" events to the even CTA's barriers, and the commits arrive in
// both CTAs. Each CTA's epilogue drains its own 128 accumulator lanes.
// EPI 0 = ReLU → tiled H (GEMM2's A); EPI 1 = 16-bit rows; EPI 2 = fp32
// rows (the IEP classifier's logits). An optional per-expert bias is added
// first. F16: fp16 operands and outputs, else bf16.
template <int EPI, bool F16>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    k_moe_gemm(const __grid_constant__ GemmParams P) {
  constexpr uint32_t IDESC = F16 ? idesc_f16_f32(2 * kBM, kBN) : idesc_bf16_f32(2 * kBM, kBN);
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = smem + kStages * kABytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + kStages * kBHalf);
  uint64_t* full = bars;
  uint64_t* empty = full + kStages;
  uint64_t* acc_full = empty + kStages;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full + s, leader ? 2 : 1);  // own copies (+ the peer's relay on the leader)
      mbar_init(empty + s, 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(acc_full + s, 1);
      mbar_init(acc_empty + s, 2 * kEpiWarps);  // every epilogue warp of both CTAs
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair(tmem_slot, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int32_t n_nt = P.N / kBN, n_kc = P.K / kBK;
  // units: (row-tile pair, N tile); tile ranges are whole pairs
  const int32_t u_first = P.tile_begin / 2 * n_nt;
  const int32_t u_end = (P.tile_end < 0 ? *P.n_tiles : P.tile_end) / 2 * n_nt;
  const int32_t pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;

  if (warp == 0) {
    if (lane == 0) {  // producer (both CTAs): own A tile + own half of the weight tile
      uint32_t si = 0;
      for (int32_t u = u_first + pair; u < u_end; u += n_pairs) {
        const int32_t rt = 2 * (u / n_nt) + static_cast<int32_t>(rank), nt = u % n_nt;
        const int32_t e = P.tile_expert[rt], rb = P.tile_rb[rt];
        const uint8_t* a = P.A + static_cast<int64_t>(rb) * n_kc * kABytes;
        const uint8_t* w = P.W[e] + static_cast<int64_t>(nt) * n_kc * kBBytes + rank * kBHalf;
        for (int32_t kc = 0; kc < n_kc; ++kc, ++si) {
          const uint32_t s = si % kStages, ph = (si / kStages) & 1;
          mbar_wait(empty + s, ph ^ 1);
          mbar_expect_tx(full + s, kABytes + kBHalf);
          bulk_g2s(sA + s * kABytes, a + static_cast<int64_t>(kc) * kABytes, kABytes, full + s);
          bulk_g2s(sB + s * kBHalf, w + static_cast<int64_t>(kc) * kBBytes, kBHalf, full + s);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {  // MMA issuer (even CTA)
      uint32_t si = 0;
      int it = 0;
      const uint32_t a_base = smem_u32(sA), b_base = smem_u32(sB);
      for (int32_t u = u_first + pair; u < u_end; u += n_pairs, ++it) {
        const int abuf = it & 1;
        mbar_wait(acc_empty + abuf, ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        for (int32_t kc = 0; kc < n_kc; ++kc, ++si) {
          const uint32_t s = si % kStages, ph = (si / kStages) & 1;
          mbar_wait(full + s, ph);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk) {
            const uint64_t ad = EPI == 0 ? smem_desc_sw128(a_base + s * kABytes + kk * 32)
                                         : smem_desc(a_base + s * kABytes + (2 * kk) * kBM * 16, kBM * 16, 128);
            const uint64_t bd = smem_desc(b_base + s * kBHalf + (2 * kk) * 128 * 16, 128 * 16, 128);
            mma_bf16_pair(tmem_base + abuf * kBN, ad, bd, IDESC, (kc | kk) != 0);
          }
          mma_commit_pair(empty + s, 0x3);
        }
        mma_commit_pair(acc_full + abuf, 0x3);
      }
    } else if (lane == 0) {  // relay (odd CTA): its stage landed
      uint32_t si = 0;
      for (int32_t u = u_first + pair; u < u_end; u += n_pairs)
        for (int32_t kc = 0; kc < n_kc; ++kc, ++si) {
          const uint32_t s = si % kStages, ph = (si / kStages) & 1;
          mbar_wait(full + s, ph);
          mbar_arrive_remote_relaxed(full + s, 0);
        }
    }
  } else {  // epilogue: 8 warps, two per TMEM lane quarter, 128 columns each
    const int quarter = warp & 3;
    const int col0 = ((warp - 2) >> 2) * (kBN / 2);
    int it = 0;
    for (int32_t u = u_first + pair; u < u_end; u += n_pairs, ++it) {
      const int abuf = it & 1;
      const int32_t rt = 2 * (u / n_nt) + static_cast<int32_t>(rank), nt = u % n_nt;
      const int32_t rb = P.tile_rb[rt];
      const float* bias = P.bias ? P.bias[P.tile_expert[rt]] : nullptr;
      mbar_wait(acc_full + abuf, (it >> 1) & 1);
      tc_fence_after();
      const int32_t rr = quarter * 32 + lane;
      const int64_t row = static_cast<int64_t>(rb) * kBM + rr;
#pragma unroll 1
      for (int c = 0; c < kBN / 2; c += 32) {
        float v[32];
        tmem_ld32(tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + abuf * kBN + col0 + c, v);
        const int32_t n0 = nt * kBN + col0 + c;  // global output column of v[0]
        if (bias) {
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float4 b4 = __ldg(reinterpret_cast<const float4*>(bias + n0) + q);
            v[4 * q] += b4.x;
            v[4 * q + 1] += b4.y;
            v[4 * q + 2] += b4.z;
            v[4 * q + 3] += b4.w;
          }
        }
        if (EPI == 0) {
          const int32_t n_kc_out = P.N / kBK;
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            const int32_t col = n0 + g * 8;
            uint4 pk;
            pk.x = pack2<F16>(fmaxf(v[g * 8 + 0], 0.f), fmaxf(v[g * 8 + 1], 0.f));
            pk.y = pack2<F16>(fmaxf(v[g * 8 + 2], 0.f), fmaxf(v[g * 8 + 3], 0.f));
            pk.z = pack2<F16>(fmaxf(v[g * 8 + 4], 0.f), fmaxf(v[g * 8 + 5], 0.f));
            pk.w = pack2<F16>(fmaxf(v[g * 8 + 6], 0.f), fmaxf(v[g * 8 + 7], 0.f));
            uint8_t* blk = P.H + (static_cast<int64_t>(rb) * n_kc_out + col / kBK) * kABytes;
            *reinterpret_cast<uint4*>(blk + (((col % kBK) / 8) * kBM + rr) * 16) = pk;
          }
        } else if (EPI == 2) {
          const int64_t orow = P.out_row ? P.out_row[row] : row;
          if (orow < 0) continue;
          float4* dst = reinterpret_cast<float4*>(P.Yf + orow * P.N + n0);
#pragma unroll
          for (int q = 0; q < 8; ++q) dst[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        } else {
          const int64_t orow = P.out_row ? P.out_row[row] : row;
          if (orow < 0) continue;  // padding row (EP: no receive row)
          uint16_t* dst = P.Y + orow * P.N + n0;
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            uint4 pk;
            pk.x = pack2<F16>(v[g * 8 + 0], v[g * 8 + 1]);
            pk.y = pack2<F16>(v[g * 8 + 2], v[g * 8 + 3]);
            pk.z = pack2<F16>(v[g * 8 + 4], v[g * 8 + 5]);
            pk.w = pack2<F16>(v[g * 8 + 6], v[g * 8 + 7]);
            *reinterpret_cast<uint4*>(dst + g * 8) = pk;
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (leader) mbar_arrive(acc_empty + abuf);
        else mbar_arrive_remote_relaxed(acc_empty + abuf, 0);
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

// out[t] = Σ_slot w[t·k + slot] · Y[row_of_item[t·k + slot]] in slot order.
template <bool F16>
__global__ void k_moe_combine_f32(int64_t T, int32_t k, int32_t d, const double* __restrict__ w,
                                  const int32_t* __restrict__ row_of_item, const uint16_t* __restrict__ Y,
                                  float* __restrict__ out) {
  const int64_t t = blockIdx.x;
  if (t >= T) return;
  for (int32_t j = threadIdx.x * 8; j < d; j += blockDim.x * 8) {
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int32_t s = 0; s < k; ++s) {
      const float ws = static_cast<float>(w[t * k + s]);
      const uint4 raw = *reinterpret_cast<const uint4*>(Y + static_cast<int64_t>(row_of_item[t * k + s]) * d + j);
      const uint32_t* y2 = reinterpret_cast<const uint32_t*>(&raw);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 f = unpack2<F16>(y2[q]);
        acc[2 * q] = fmaf(ws, f.x, acc[2 * q]);
        acc[2 * q + 1] = fmaf(ws, f.y, acc[2 * q + 1]);
      }
    }
    *reinterpret_cast<float4*>(out + t * d + j) = make_float4(acc[0], acc[1], acc[2], acc[3]);
    *reinterpret_cast<float4*>(out + t * d + j + 4) = make_float4(acc[4], acc[5], acc[6], acc[7]);
  }
}

template <int EPI, bool F16>
int launch_gemm(const GemmParams& p, int sms, cudaStream_t s) {
  static std::atomic<uint64_t> configured{0};  // per device (the attribute is), once, from any thread
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (!(configured.load(std::memory_order_acquire) & bit)) {
    cudaFuncSetAttribute(k_moe_gemm<EPI, F16>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    configured.fetch_or(bit, std::memory_order_release);
  }
  k_moe_gemm<EPI, F16><<<sms / 2 * 2, kThreads, kSmem, s>>>(p);  // CTA pairs
  return static_cast<int>(cudaGetLastError());
}

}  // namespace

extern "C" int dbk_moe_tc_layout(int32_t n, const int32_t* offsets, int32_t* pstart, int32_t* tile_expert,
                                   int32_t* tile_rb, int32_t* n_tiles, void* stream) {
  k_moe_layout<<<1, 1024, 0, static_cast<cudaStream_t>(stream)>>>(n, offsets, pstart, tile_expert, tile_rb, n_tiles);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_moe_tc_dispatch(int32_t fmt, int64_t T, int32_t k, int32_t d, const int32_t* order,
                                   const int32_t* ids, const int32_t* offsets, const int32_t* pstart, const float* x,
                                   void* A, int32_t* row_of_item, int32_t blocks, void* stream) {
  if (T <= 0) return 0;
  if (k > 8 || d % 256 != 0) return static_cast<int>(cudaErrorInvalidValue);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  k_moe_item_rows<<<blocks, 256, 0, s>>>(T * k, order, ids, offsets, pstart, row_of_item);
  if (fmt == DBK_FMT_F16) k_moe_dispatch<true><<<blocks, 256, 0, s>>>(T, k, d, x, row_of_item, static_cast<uint8_t*>(A));
  else k_moe_dispatch<false><<<blocks, 256, 0, s>>>(T, k, d, x, row_of_item, static_cast<uint8_t*>(A));
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_moe_tc_gemm(int32_t fmt, int32_t epi, int32_t n, int32_t K, int32_t N, const int32_t* n_tiles,
                                 const int32_t* tile_expert, const int32_t* tile_rb, const void* A,
                                 const void* const* W, void* H, void* Y, int32_t tile_begin, int32_t tile_end,
                                 const int32_t* out_row, int32_t sms, void* stream) {
  return dbk_tc_gemm_bias(fmt, epi, n, K, N, n_tiles, tile_expert, tile_rb, A, W, nullptr, H, Y, tile_begin,
                          tile_end, out_row, sms, stream);
}

extern "C" int dbk_tc_gemm_bias(int32_t fmt, int32_t epi, int32_t n, int32_t K, int32_t N, const int32_t* n_tiles,
                                const int32_t* tile_expert, const int32_t* tile_rb, const void* A,
                                const void* const* W, const float* const* bias, void* H, void* Y,
                                int32_t tile_begin, int32_t tile_end, const int32_t* out_row, int32_t sms,
                                void* stream) {
  if (K % kBK != 0 || N % kBN != 0 || epi < 0 || epi > 2) return static_cast<int>(cudaErrorInvalidValue);
  GemmParams p{n, K, N, n_tiles, tile_expert, tile_rb, static_cast<const uint8_t*>(A),
               reinterpret_cast<const uint8_t* const*>(W), static_cast<uint8_t*>(H),
               static_cast<uint16_t*>(Y), tile_begin, tile_end, out_row, bias, static_cast<float*>(Y)};
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (fmt == DBK_FMT_F16) {
    if (epi == 0) return launch_gemm<0, true>(p, sms, s);
    return epi == 1 ? launch_gemm<1, true>(p, sms, s) : launch_gemm<2, true>(p, sms, s);
  }
  if (epi == 0) return launch_gemm<0, false>(p, sms, s);
  return epi == 1 ? launch_gemm<1, false>(p, sms, s) : launch_gemm<2, false>(p, sms, s);
}

extern "C" int dbk_moe_tc_combine(int32_t fmt, int64_t T, int32_t k, int32_t d, const double* weights,
                                  const int32_t* row_of_item, const void* Y, float* out, void* stream) {
  if (T <= 0) return 0;
  const uint16_t* y = static_cast<const uint16_t*>(Y);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (fmt == DBK_FMT_F16) k_moe_combine_f32<true><<<static_cast<unsigned>(T), 128, 0, s>>>(T, k, d, weights, row_of_item, y, out);
  else k_moe_combine_f32<false><<<static_cast<unsigned>(T), 128, 0, s>>>(T, k, d, weights, row_of_item, y, out);
  return static_cast<int>(cudaGetLastError());
}

// ----------------------------------------------------- expert parallel
// Expert-parallel MoE: tokens are sharded T/G per rank and
// experts n/G per rank (contiguous). A rank's items, stably sorted by expert
// in (token, slot) order, are therefore already grouped by destination rank.
namespace {

// Rows per global expert of this rank's sorted items (the send counts of
// the exchange: destination q's experts are the block [q·E, (q+1)·E)).
__global__ void k_moe_ep_counts(int32_t n, const int32_t* __restrict__ offsets, int32_t* __restrict__ counts) {
  for (int32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x)
    counts[e] = offsets[e + 1] - offsets[e];
}

// pos_of_item[order[i]] = i: an item's row in the sorted send buffer.
__global__ void k_moe_ep_positions(int64_t items, const int32_t* __restrict__ order,
                                   int32_t* __restrict__ pos_of_item) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < items;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    pos_of_item[order[i]] = static_cast<int32_t>(i);
}

// send[pos_of_item[t·k + s]] = fp16/bf16(x[t]): one warp per token reads its fp32
// row once and writes its k 16-bit rows (row-contiguous, coalesced).
template <bool F16>
__global__ void k_moe_ep_pack(int64_t T, int32_t k, int32_t d, const int32_t* __restrict__ pos_of_item,
                              const float* __restrict__ x, uint16_t* __restrict__ send) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x >> 5) + (threadIdx.x >> 5); t < T; t += warps) {
    const float* src = x + t * d;
    int32_t pos[8];
#pragma unroll
    for (int s = 0; s < 8; ++s) pos[s] = s < k ? pos_of_item[t * k + s] : 0;
    for (int32_t j = lane * 8; j < d; j += 256) {
      const float4 a = __ldg(reinterpret_cast<const float4*>(src + j));
      const float4 b = __ldg(reinterpret_cast<const float4*>(src + j + 4));
      uint4 pk;
      pk.x = pack2<F16>(a.x, a.y);
      pk.y = pack2<F16>(a.z, a.w);
      pk.z = pack2<F16>(b.x, b.y);
      pk.w = pack2<F16>(b.z, b.w);
#pragma unroll
      for (int s = 0; s < 8; ++s)
        if (s < k) *reinterpret_cast<uint4*>(send + static_cast<int64_t>(pos[s]) * d + j) = pk;
    }
  }
}

// Block-wide exclusive scan of one value per thread (all threads call);
// *total = the block's sum.
__device__ __forceinline__ int32_t block_excl_scan(int32_t v, int32_t* total, int32_t* wsum) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int32_t x = v;
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int32_t w = lane < nw ? wsum[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    wsum[lane] = w;
  }
  __syncthreads();
  const int32_t excl = (warp > 0 ? wsum[warp - 1] : 0) + x - v;
  *total = wsum[nw - 1];
  __syncthreads();
  return excl;
}

// Receiver layout from the count matrix cnt[G][E] (rows source r sent for
// local expert e; the receive buffer holds source blocks in rank order, each
// expert-major), one 1024-thread block: per (expert, source) the receive row
// of its first row (src_row[e·G + r]) and its offset within the expert
// (cum[e·(G+1) + r]); per-expert padded starts and the tile list, as
// k_moe_layout.
__global__ void __launch_bounds__(1024) k_moe_ep_layout(int32_t G, int32_t E, const int32_t* __restrict__ cnt,
                                                        int32_t* __restrict__ pstart,
                                                        int32_t* __restrict__ tile_expert,
                                                        int32_t* __restrict__ tile_rb, int32_t* __restrict__ n_tiles,
                                                        int32_t* __restrict__ src_row, int32_t* __restrict__ cum) {
  __shared__ int32_t wsum[32];
  int32_t base = 0;  // receive row where source r's block starts
  for (int32_t r = 0; r < G; ++r) {
    int32_t carry = 0;
    for (int32_t e0 = 0; e0 < E; e0 += blockDim.x) {
      const int32_t e = e0 + static_cast<int32_t>(threadIdx.x);
      int32_t total;
      const int32_t excl = block_excl_scan(e < E ? cnt[r * E + e] : 0, &total, wsum);
      if (e < E) src_row[e * G + r] = base + carry + excl;
      carry += total;
    }
    base += carry;
  }
  int32_t carry = 0;  // row blocks so far
  for (int32_t e0 = 0; e0 < E; e0 += blockDim.x) {
    const int32_t e = e0 + static_cast<int32_t>(threadIdx.x);
    int32_t tot = 0;
    if (e < E) {
      for (int32_t r = 0; r < G; ++r) {
        cum[e * (G + 1) + r] = tot;
        tot += cnt[r * E + e];
      }
      cum[e * (G + 1) + G] = tot;
    }
    const int32_t nb = (tot + kPairRows - 1) / kPairRows * 2;
    int32_t total;
    const int32_t first = carry + block_excl_scan(nb, &total, wsum);
    if (e < E) {
      pstart[e] = first * kBM;
      for (int32_t b = 0; b < nb; ++b) {
        tile_expert[first + b] = e;
        tile_rb[first + b] = first + b;
      }
    }
    carry += total;
  }
  if (threadIdx.x == 0) {
    pstart[E] = carry * kBM;
    *n_tiles = carry;
  }
}

// Received rows → the SWIZZLE_128B tiled A operand (one warp per padded
// row, whole 128-byte lines), expert e's rows in source-rank order = the
// reference's (token, slot) order for that expert. recv_of_row[padded row]
// = receive-buffer row (−1 for padding, whose A rows are left unwritten).
__global__ void k_moe_ep_scatter(int32_t G, int32_t d, const int32_t* __restrict__ pstart,
                                 const int32_t* __restrict__ tile_expert, const int32_t* __restrict__ src_row,
                                 const int32_t* __restrict__ cum, int32_t E,
                                 const uint16_t* __restrict__ recv, uint8_t* __restrict__ A,
                                 int32_t* __restrict__ recv_of_row, int32_t row_begin, int32_t row_end) {
  const int32_t total_rows = row_end < 0 ? pstart[E] : row_end;
  const int32_t kchunks = d / kBK;
  const int lane = threadIdx.x & 31;
  const int32_t warps = gridDim.x * (blockDim.x >> 5);
  for (int32_t row = row_begin + blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < total_rows;
       row += warps) {
    const int32_t e = tile_expert[row / kBM];
    const int32_t local = row - pstart[e];
    const int32_t* ce = cum + e * (G + 1);
    int32_t src = -1;
    if (local < ce[G]) {
      int32_t r = 0;
      while (local >= ce[r + 1]) ++r;
      src = src_row[e * G + r] + (local - ce[r]);
    }
    if (lane == 0) recv_of_row[row] = src;
    if (src < 0) continue;
    const uint4* s4 = reinterpret_cast<const uint4*>(recv + static_cast<int64_t>(src) * d);
    for (int32_t gi = lane; gi < d / 8; gi += 32)
      *reinterpret_cast<uint4*>(A + a_sw128_off(row, kchunks, gi >> 3, gi & 7)) = __ldg(s4 + gi);
  }
}

}  // namespace

extern "C" int dbk_moe_ep_pack(int32_t fmt, int64_t items, int32_t k, int32_t d, const int32_t* order, const float* x,
                               void* send, int32_t* pos_of_item, int32_t blocks, void* stream) {
  if (items <= 0) return 0;
  if (k > 8 || d % 8 != 0) return static_cast<int>(cudaErrorInvalidValue);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  k_moe_ep_positions<<<blocks, 256, 0, s>>>(items, order, pos_of_item);
  if (fmt == DBK_FMT_F16) k_moe_ep_pack<true><<<blocks, 256, 0, s>>>(items / k, k, d, pos_of_item, x, static_cast<uint16_t*>(send));
  else k_moe_ep_pack<false><<<blocks, 256, 0, s>>>(items / k, k, d, pos_of_item, x, static_cast<uint16_t*>(send));
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_moe_ep_counts(int32_t n, const int32_t* offsets, int32_t* counts, void* stream) {
  k_moe_ep_counts<<<(n + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(n, offsets, counts);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_moe_ep_layout(int32_t G, int32_t E, const int32_t* cnt, int32_t* pstart, int32_t* tile_expert,
                                 int32_t* tile_rb, int32_t* n_tiles, int32_t* src_row, int32_t* cum,
                                 void* stream) {
  k_moe_ep_layout<<<1, 1024, 0, static_cast<cudaStream_t>(stream)>>>(G, E, cnt, pstart, tile_expert, tile_rb,
                                                                    n_tiles, src_row, cum);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_moe_ep_scatter(int32_t G, int32_t E, int32_t d, const int32_t* pstart,
                                  const int32_t* tile_expert, const int32_t* src_row, const int32_t* cum,
                                  const void* recv, void* A, int32_t* recv_of_row, int32_t row_begin,
                                  int32_t row_end, int32_t blocks, void* stream) {
  k_moe_ep_scatter<<<blocks, kBM, 0, static_cast<cudaStream_t>(stream)>>>(
      G, d, pstart, tile_expert, src_row, cum, E, static_cast<const uint16_t*>(recv),
      static_cast<uint8_t*>(A), recv_of_row, row_begin, row_end);
  return static_cast<int>(cudaGetLastError());
}

