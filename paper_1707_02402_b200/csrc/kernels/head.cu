// head.cu — the IEP classifier head on the root outputs (
// the reference stops at the root feature maps, so this follows
// the IEP classifier of Johnson et al. that PAPER.md:75 measures):
//   proj   = relu(conv1x1(root, 128 → P) + bp)          [196 px × P]
//   pooled = maxpool2x2(proj)                           [49 px × P]
//   hidden = relu(FC(flatten(pooled), 49·P → F) + b1)   flatten pixel-major: q·P + c
//   logits = FC(hidden, F → A) + b2
// The three contractions run on the grouped tcgen05 GEMM (moe_gemm.cu,
// dbk_tc_gemm_bias) as one group; the kernels here only move operands:
//   * k_head_pack: each root's fp32 plane map → fp16 rows (program·196 + px)
//     of the SWIZZLE_128B K-major tiled A ([row block][2 K chunks][16 KB]);
//   * k_head_pool: the projection's tiled output H ([rb][P/64][8][128][8]) →
//     2×2 max → fp16 rows (program) of the SW128 tiled A of the first FC.
// Both move 16-byte vectors only (HBM-bound).
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "dynbatch/dbk.h"
#include "tc_common.cuh"

namespace {

using namespace dbk;

constexpr int kPlanes = 16, kPx = 196, kFmap = kPlanes * kPx * 8;
constexpr int kBM = 128, kBK = 64, kABytes = kBM * kBK * 2;

// Byte offset of 16-byte piece j (elements 8j..8j+7 of K chunk kc) of row
// `row` in a SWIZZLE_128B tiled operand with `kchunks` K chunks per row block.
__device__ __forceinline__ int64_t sw128_off(int64_t row, int32_t kchunks, int32_t kc, int32_t j) {
  const int64_t rb = row / kBM;
  const int32_t rr = static_cast<int32_t>(row % kBM);
  return (rb * kchunks + kc) * kABytes + rr * 128 + ((j ^ (rr & 7)) << 4);
}

// One thread per (root row px, plane p): the plane's 8 fp32 channels → one
// 16-byte fp16 piece. The root is the example's input map for a leaf root.
__global__ void __launch_bounds__(256) k_head_pack(int64_t b, const int32_t* __restrict__ root_g,
                                                   const int32_t* __restrict__ fid,
                                                   const int32_t* __restrict__ arity_of,
                                                   const int32_t* __restrict__ example,
                                                   const float* __restrict__ inputs,
                                                   const float* __restrict__ values, uint8_t* __restrict__ A) {
  const int64_t total = b * kPx * kPlanes;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int p = static_cast<int>(i % kPlanes);
    const int64_t row = i / kPlanes;  // program · 196 + px
    const int64_t e = row / kPx;
    const int px = static_cast<int>(row % kPx);
    const int32_t r = root_g[e];
    const float* map = arity_of[fid[r]] == 0 ? inputs + static_cast<int64_t>(example[r]) * kFmap
                                            : values + static_cast<int64_t>(r) * kFmap;
    const float4* src = reinterpret_cast<const float4*>(map + (static_cast<int64_t>(p) * kPx + px) * 8);
    const float4 a = __ldg(src), c = __ldg(src + 1);
    uint4 pk;
    pk.x = pack_f16x2(a.x, a.y);
    pk.y = pack_f16x2(a.z, a.w);
    pk.z = pack_f16x2(c.x, c.y);
    pk.w = pack_f16x2(c.z, c.w);
    *reinterpret_cast<uint4*>(A + sw128_off(row, 2, p >> 3, p & 7)) = pk;
  }
}

// One thread per (program, pooled pixel q, 8-channel group g): the max of the
// four projected pixels (ReLU outputs, fp16) → the first FC's A at K index
// q·P + 8g.
__global__ void __launch_bounds__(256) k_head_pool(int64_t b, int32_t P, const uint8_t* __restrict__ H,
                                                   uint8_t* __restrict__ A) {
  const int32_t groups = P / 8, h_kchunks = P / kBK, a_kchunks = 49 * P / kBK;
  const int64_t total = b * 49 * groups;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t g = static_cast<int32_t>(i % groups);
    const int64_t eq = i / groups;
    const int32_t q = static_cast<int32_t>(eq % 49);
    const int64_t e = eq / 49;
    const int ph = q / 7, pw = q % 7;
    __half2 m[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int64_t row = e * kPx + (2 * ph + (t >> 1)) * 14 + 2 * pw + (t & 1);
      // H block (row block, K chunk) = [8 k-groups][128 rows][8 elements]
      const int64_t off = ((row / kBM) * h_kchunks + g / 8) * kABytes + ((g % 8) * kBM + row % kBM) * 16;
      const uint4 v = *reinterpret_cast<const uint4*>(H + off);
      const __half2* h = reinterpret_cast<const __half2*>(&v);
      if (t == 0) {
#pragma unroll
        for (int j = 0; j < 4; ++j) m[j] = h[j];
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) m[j] = __hmax2(m[j], h[j]);
      }
    }
    const int32_t k = q * P + 8 * g;
    *reinterpret_cast<uint4*>(A + sw128_off(e, a_kchunks, k / kBK, (k % kBK) / 8)) =
        *reinterpret_cast<const uint4*>(m);
  }
}

}  // namespace

extern "C" int dbk_head_pack(int64_t b, const int32_t* root_g, const int32_t* fid, const int32_t* arity_of,
                             const int32_t* example, const float* inputs, const float* values, void* A,
                             void* stream) {
  if (b <= 0) return 0;
  const int64_t total = b * kPx * kPlanes;
  const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((total + 255) / 256, 148 * 16));
  k_head_pack<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(b, root_g, fid, arity_of, example, inputs,
                                                                      values, static_cast<uint8_t*>(A));
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_head_pool(int64_t b, int32_t P, const void* H, void* A, void* stream) {
  if (b <= 0) return 0;
  if (P % kBK != 0) return static_cast<int>(cudaErrorInvalidValue);
  const int64_t total = b * 49 * (P / 8);
  const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((total + 255) / 256, 148 * 16));
  k_head_pool<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(b, P, static_cast<const uint8_t*>(H),
                                                                      static_cast<uint8_t*>(A));
  return static_cast<int>(cudaGetLastError());
}
