// sw128_test.cu — does a K-major SWIZZLE_128B UMMA descriptor work at
// arbitrary row starts (the conv tap shift) and K offsets within the swizzle
// atom? Data is stored swizzled by ABSOLUTE smem row (chunk j of row r at
// (j ^ (r & 7)) · 16), regions 1024-byte aligned. D = A · B[s : s+256]ᵀ,
// M = 128, N = 256, K = 64 (4 MMAs of K = 16). Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I../paper_1707_02402_b200/csrc/kernels sw128_test.cu
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <vector>
#include "tc_common.cuh"

using namespace dbk;

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr, uint32_t base_off) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(1) << 16;                 // LBO (unused for swizzled K-major)
  d |= static_cast<uint64_t>(1024 >> 4) << 32;         // SBO: 8 rows × 128 B
  d |= static_cast<uint64_t>(1) << 46;                 // version
  d |= static_cast<uint64_t>(base_off & 7) << 49;      // base offset
  d |= static_cast<uint64_t>(2) << 61;                 // SWIZZLE_128B
  return d;
}

constexpr int BR = 320;  // B rows available

__global__ void k_test(const __half* A, const __half* B, float* D, int shift, int mode) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;               // 128 × 128 B
  uint8_t* sB = smem + 16384;       // BR × 128 B
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  for (int i = tid; i < 128 * 64; i += blockDim.x) {
    const int m = i / 64, k = i % 64, c = k / 8, e = k % 8;
    reinterpret_cast<__half*>(sA + m * 128 + ((c ^ (m & 7)) * 16))[e] = A[i];
  }
  for (int i = tid; i < BR * 64; i += blockDim.x) {
    const int r = i / 64, k = i % 64, c = k / 8, e = k % 8;
    reinterpret_cast<__half*>(sB + r * 128 + ((c ^ (r & 7)) * 16))[e] = B[i];
  }
  if (tid == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc(&slot, 256);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (tid == 0) {
    const uint32_t idesc = idesc_f16_f32(128, 256);
    for (int kk = 0; kk < 4; ++kk) {
      const uint32_t aaddr = smem_u32(sA) + kk * 32;
      const uint32_t baddr = smem_u32(sB) + shift * 128 + kk * 32;
      const uint32_t boa = mode ? ((aaddr >> 7) & 7) : 0;
      const uint32_t bob = mode ? ((baddr >> 7) & 7) : 0;
      mma_bf16(tmem, desc_sw128(aaddr, boa), desc_sw128(baddr, bob), idesc, kk > 0);
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  for (int cb = 0; cb < 8; ++cb) {
    float v[32];
    tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + cb * 32, v);
    for (int j = 0; j < 32; ++j) D[(warp * 32 + lane) * 256 + cb * 32 + j] = v[j];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 256); }
}

int main() {
  std::vector<__half> hA(128 * 64), hB(BR * 64);
  std::vector<float> fA(128 * 64), fB(BR * 64);
  for (int i = 0; i < 128 * 64; ++i) { fA[i] = (float)((i * 7 + 3) % 11 - 5); hA[i] = __float2half(fA[i]); }
  for (int i = 0; i < BR * 64; ++i) { fB[i] = (float)((i * 5 + 1) % 13 - 6); hB[i] = __float2half(fB[i]); }
  __half *dA, *dB; float* dD;
  cudaMalloc(&dA, hA.size() * 2); cudaMalloc(&dB, hB.size() * 2); cudaMalloc(&dD, 128 * 256 * 4);
  cudaMemcpy(dA, hA.data(), hA.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), hB.size() * 2, cudaMemcpyHostToDevice);
  const int smem = 16384 + BR * 128;
  cudaFuncSetAttribute(k_test, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int shifts[] = {0, 1, 3, 7, 8, 15, 16, 17, 31, 32, 47, 64};
  std::vector<float> hD(128 * 256);
  for (int mode = 0; mode < 2; ++mode) {
    for (int s : shifts) {
      cudaMemset(dD, 0, 128 * 256 * 4);
      k_test<<<1, 128, smem>>>(dA, dB, dD, s, mode);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(hD.data(), dD, hD.size() * 4, cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 256; ++n) {
          float ref = 0;
          for (int k = 0; k < 64; ++k) ref += fA[m * 64 + k] * fB[(s + n) * 64 + k];
          if (hD[m * 256 + n] != ref) ++bad;
        }
      printf("mode=%d (base_offset %s) shift=%2d err=%d mismatches=%d\n", mode, mode ? "=(addr>>7)&7" : "=0", s,
             (int)e, bad);
    }
  }
  return 0;
}
