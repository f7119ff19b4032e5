// Probe of MN-major SWIZZLE_128B operands for tcgen05.mma (kind::f16 and
// kind::tf32): D[m][n] = Σ_k A[k][m]·B[k][n], operands written to shared
// memory in the canonical MN-major layout (K rows of 128 B, 8-row groups 1024
// B apart = SBO, MN blocks LBO apart, 16-byte pieces XOR-swizzled by row).
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 --expt-relaxed-constexpr \
//        -I paper_1707_02402_b200/csrc/kernels tools/mn_major_test.cu -o /tmp/mn && /tmp/mn
#include <cuda_fp16.h>
#include <cstdio>
#include <vector>
#include <cmath>
#include "tc_common.cuh"
using namespace dbk;

template <bool TF32>
__global__ void k_probe(const float* A, const float* B, float* D, int K, uint32_t lbo_mode_swap) {
  // A, B: [K][128] fp32 in global; D: [128][128]
  extern __shared__ __align__(1024) uint8_t sm[];
  constexpr int esz = TF32 ? 4 : 2, per_row = 128 / esz, blocks = 128 / per_row;
  const int kgroups = K / 8;
  const int blk_bytes = kgroups * 1024;            // one MN block: K rows
  uint8_t* sa = sm;
  uint8_t* sb = sm + blocks * blk_bytes;
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  // fill
  for (int i = threadIdx.x; i < K * 128; i += blockDim.x) {
    const int k = i / 128, m = i % 128;
    const int b = m / per_row, w = m % per_row;  // block, element within the 128-B row
    const int piece = (w * esz) / 16, inpiece = (w * esz) % 16;
    const int off = b * blk_bytes + (k / 8) * 1024 + (k % 8) * 128 + ((piece ^ (k % 8)) << 4) + inpiece;
    if (TF32) { *reinterpret_cast<float*>(sa + off) = A[i]; *reinterpret_cast<float*>(sb + off) = B[i]; }
    else { *reinterpret_cast<__half*>(sa + off) = __float2half(A[i]); *reinterpret_cast<__half*>(sb + off) = __float2half(B[i]); }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (threadIdx.x < 32) tmem_alloc(&tslot, 128);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    auto desc = [&](uint32_t addr) {
      uint64_t d = 0;
      d |= static_cast<uint64_t>((addr >> 4) & 0x3FFF);
      const uint32_t lbo = lbo_mode_swap ? 1024 : blk_bytes, sbo = lbo_mode_swap ? blk_bytes : 1024;
      d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
      d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
      d |= static_cast<uint64_t>(1) << 46;
      d |= static_cast<uint64_t>(2) << 61;
      return d;
    };
    const uint32_t fmt = TF32 ? 2u : 0u;
    const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | (1u << 15) | (1u << 16) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
    const int kstep = TF32 ? 8 : 16;
    for (int k = 0; k < K; k += kstep) {
      const uint32_t ao = smem_u32(sa) + (k / 8) * 1024, bo = smem_u32(sb) + (k / 8) * 1024;
      if (TF32)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                     ::"r"(tmem), "l"(desc(ao)), "l"(desc(bo)), "r"(idesc), "r"(k > 0 ? 1 : 0));
      else
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                     ::"r"(tmem), "l"(desc(ao)), "l"(desc(bo)), "r"(idesc), "r"(k > 0 ? 1 : 0));
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  if (threadIdx.x < 128) {
    const int w = threadIdx.x / 32;
    for (int c = 0; c < 128; c += 32) {
      float v[32];
      tmem_ld32(tmem + (static_cast<uint32_t>(w * 32) << 16) + c, v);
      for (int j = 0; j < 32; ++j) D[threadIdx.x * 128 + c + j] = v[j];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 128);
}

int main() {
  const int K = 32;
  std::vector<float> A(K * 128), B(K * 128), D(128 * 128);
  for (int i = 0; i < K * 128; ++i) { A[i] = ((i * 37) % 17 - 8) / 8.0f; B[i] = ((i * 11) % 13 - 6) / 8.0f; }
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  for (int tf = 0; tf < 2; ++tf)
    for (int swap = 0; swap < 2; ++swap) {
      cudaMemset(dD, 0, D.size() * 4);
      const int smem = 2 * 128 * K * (tf ? 4 : 2) + 1024;
      if (tf) { cudaFuncSetAttribute(k_probe<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); k_probe<true><<<1, 128, smem>>>(dA, dB, dD, K, swap); }
      else { cudaFuncSetAttribute(k_probe<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); k_probe<false><<<1, 128, smem>>>(dA, dB, dD, K, swap); }
      const cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
      double err = 0, ref_max = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 128; ++n) {
          double r = 0;
          for (int k = 0; k < K; ++k) r += A[k * 128 + m] * B[k * 128 + n];
          err = std::fmax(err, std::fabs(r - D[m * 128 + n]));
          ref_max = std::fmax(ref_max, std::fabs(r));
        }
      std::printf("%s swap=%d: %s  max err %.3e (ref max %.3e)  D[0]=%.4f D[129]=%.4f\n", tf ? "tf32" : "f16 ", swap,
                  cudaGetErrorString(e), err, ref_max, D[0], D[129]);
    }
  return 0;
}
