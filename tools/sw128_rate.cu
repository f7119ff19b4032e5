// sw128_rate.cu — microbenchmark: tcgen05.mma (M=128, N=256, K=16, kind::f16)
// rate when the B (window) descriptor starts at a row that is not a multiple
// of the 8-row SWIZZLE_128B atom, as the conv taps do (row shifts of ±1, ±14,
// ±15, ±16 on a 15-wide packed grid). One CTA per SM, operands resident in
// shared memory, one commit per tap (4 MMAs) as in k_rb_step. Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_1707_02402_b200/csrc/kernels sw128_rate.cu
#include <cstdio>
#include <string>
#include <cuda_runtime.h>
#include "tc_common.cuh"

using namespace dbk;

__global__ void __launch_bounds__(128, 1) k_rate(long long* out, int taps_total, int mode, int n_cols) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, cbar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 200 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&cbar, 1); fence_barrier_init(); }
  if (warp == 1) tmem_alloc(&slot, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = n_cols == 256 ? idesc_f16_f32(128, 256) : idesc_f16_f32(128, 128);
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 64 * 1024);
    const int shifts[9] = {-16, -15, -14, -1, 0, 1, 14, 15, 16};
    long long t0 = clock64();
    for (int t = 0; t < taps_total; ++t) {
      int row;
      if (mode < 0) row = 16 + shifts[t % 9];      // the conv's 9 taps (halo 16)
      else row = mode;                              // a fixed start row
      const uint32_t abase = a + (t & 3) * 16384;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t wd = smem_desc_sw128(abase + kk * 32);
        const uint64_t xd = smem_desc_sw128(b + row * 128 + kk * 32);
        mma_bf16(tmem + (t & 1) * 0, wd, xd, idesc, (t | kk) != 0);
      }
      mma_commit(&cbar);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  long long* d; cudaMalloc(&d, sizeof(long long) * 256);
  cudaFuncSetAttribute(k_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int taps = 9 * 512;
  for (int n : {256, 128}) {
    for (int mode = -1; mode <= 17; ++mode) {
      k_rate<<<148, 128, 200 * 1024>>>(d, taps, mode, n);
      k_rate<<<148, 128, 200 * 1024>>>(d, taps, mode, n);
      cudaError_t err = cudaDeviceSynchronize();
      long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      long long mx = 0; double avg = 0;
      for (int i = 0; i < 148; ++i) { mx = h[i] > mx ? h[i] : mx; avg += h[i] / 148.0; }
      printf("N=%d start row %-9s err=%d cycles/mma avg %7.1f max %7.1f (ideal %d)\n", n,
             mode < 0 ? "9-tap" : std::to_string(mode).c_str(), (int)err, avg / (taps * 4.0), mx / (taps * 4.0), n / 2);
    }
  }
  return 0;
}
