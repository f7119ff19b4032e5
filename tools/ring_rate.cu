// ring_rate.cu — microbenchmark of the k_rb_step issue structure without
// memory traffic: a weight-stage ring of S slots between a "weight warp"
// (waits b_empty, arrives b_full; no copy) and the single-thread MMA issuer
// (waits b_full, 4 × tcgen05.mma M=128 N=256 K=16, commits b_empty), tiles of
// 18 stages alternating two TMEM accumulators (commit acc_full; an epilogue
// warp waits acc_full and arrives acc_empty). Prints cycles per MMA and the
// issuer's b_full wait per stage. Variants: mode 0 = as the kernel; 1 = no
// weight warp (issuer never waits for stages); 2 = the weight warp arrives
// as 0 without the tcgen05 fence after the wait; 3 = stages pre-completed
// (one barrier per use) with the fence; 4 = the same without the fence;
// 5/6 = pre-completed waits without clock reads (6: + fence); 7 = commits
// only; 8 = clock reads only.
#include <cstdio>
#include <cuda_runtime.h>
#include "tc_common.cuh"

using namespace dbk;

template <int S>
__global__ void __launch_bounds__(128, 1) k_ring(long long* out, int tiles, int mode) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t b_full[S], b_empty[S], acc_full[2], acc_empty[2];
  uint64_t* pre = reinterpret_cast<uint64_t*>(smem + 128 * 1024);  // modes 3/4: one pre-completed barrier per stage use
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 200 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&b_full[s], 1); mbar_init(&b_empty[s], 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(&acc_full[s], 1); mbar_init(&acc_empty[s], 1); }
    if (mode >= 3) for (int i = 0; i < tiles * 18; ++i) { mbar_init(&pre[i], 1); mbar_arrive(&pre[i]); }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&slot, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  constexpr int kStages = 18;
  const int total = tiles * kStages;
  if (warp == 1 && lane == 0) {  // issuer
    const uint32_t idesc = idesc_f16_f32(128, 256);
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 64 * 1024);
    long long wait = 0;
    const long long t0 = clock64();
    int bi = 0;
    for (int n = 0; n < tiles; ++n) {
      const int abuf = n & 1;
      mbar_wait(&acc_empty[abuf], ((n >> 1) & 1) ^ 1);
      tc_fence_after();
      for (int t = 0; t < kStages; ++t, ++bi) {
        const int s = bi % S;
        if (mode == 0 || mode == 2) {
          const long long c0 = clock64();
          mbar_wait(&b_full[s], (bi / S) & 1);
          wait += clock64() - c0;
          if (mode == 0) tc_fence_after();
        } else if (mode == 3 || mode == 4) {
          const long long c0 = clock64();
          mbar_wait(&pre[bi], 0);
          wait += clock64() - c0;
          if (mode == 3) tc_fence_after();
        } else if (mode == 5 || mode == 6) {  // wait on a pre-completed barrier, no clock reads
          mbar_wait(&pre[bi], 0);
          if (mode == 6) tc_fence_after();
        } else if (mode == 8) {  // clock reads only
          const long long c0 = clock64();
          wait += clock64() - c0;
        }
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t wd = smem_desc_sw128(a + s * 16384 % 65536 + kk * 32);
          const uint64_t xd = smem_desc_sw128(b + (16 + (t % 3) - 1) * 128 + kk * 32);
          mma_bf16(tmem + abuf * 256, wd, xd, idesc, (t | kk) != 0);
        }
        if (mode == 0 || mode == 2) mma_commit(&b_empty[s]);
        else if (mode >= 3 && mode <= 7) mma_commit(&b_empty[0]);  // same commit traffic, nobody waits
      }
      mma_commit(&acc_full[abuf]);
    }
    const long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
    out[256 + blockIdx.x] = wait;
  } else if (warp == 2 && lane == 0 && (mode == 0 || mode == 2)) {  // weight warp
    for (int bi = 0; bi < total; ++bi) {
      const int s = bi % S;
      mbar_wait(&b_empty[s], ((bi / S) & 1) ^ 1);
      mbar_arrive(&b_full[s]);
    }
  } else if (warp == 3 && lane == 0) {  // epilogue stand-in
    for (int n = 0; n < tiles; ++n) {
      const int abuf = n & 1;
      mbar_wait(&acc_full[abuf], (n >> 1) & 1);
      tc_fence_after();
      mbar_arrive(&acc_empty[abuf]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int S>
void run(int mode, int grid = 148) {
  long long* d; cudaMalloc(&d, sizeof(long long) * 512);
  auto k = k_ring<S>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int tiles = 200;
  k<<<grid, 128, 200 * 1024>>>(d, tiles, mode);
  k<<<grid, 128, 200 * 1024>>>(d, tiles, mode);
  cudaError_t err = cudaDeviceSynchronize();
  long long h[512]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double cyc = 0, w = 0;
  for (int i = 0; i < grid; ++i) { cyc += h[i] / grid; w += h[256 + i] / grid; }
  const double mmas = tiles * 18.0 * 4;
  printf("grid=%3d S=%d mode=%d err=%d cycles/mma %.1f (ideal 128)  b_full wait per stage %.1f\n", S, mode, (int)err,
         cyc / mmas, w / (tiles * 18.0));
  cudaFree(d);
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  for (int g : {148, 16, 2, 148}) {
    run<4>(1, g);
    run<4>(0, g);
    run<4>(5, g);
    run<4>(7, g);
    run<4>(8, g);
  }
  return 0;
}
