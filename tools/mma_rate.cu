// mma_rate.cu — microbenchmark: tcgen05.mma issue rate per shape/mode on one
// SM (operands from shared memory, no loads). Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_1707_02402_b200/csrc/kernels mma_rate.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "tc_common.cuh"

using namespace dbk;

template <int M, int N, bool PAIR>
__global__ void __launch_bounds__(128, 1) k_rate(long long* out, int iters, uint32_t lbo_a, uint32_t lbo_b, const uint8_t* gsrc, int copy_kb, int a_step, int commit_every, int ld_warps) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint64_t cbar;
  __shared__ uint64_t dbar;
  __shared__ uint64_t cbar2;
  const bool wait_too = copy_kb < 0;
  __shared__ volatile int done;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&cbar, 1); mbar_init(&dbar, 1); mbar_init(&cbar2, 1); mbar_arrive(&cbar2); done = 0; fence_barrier_init(); }
  if (warp == 1) { if (PAIR) tmem_alloc_pair(&slot, 512); else tmem_alloc(&slot, 512); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  if (PAIR) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const bool leader = !PAIR || cluster_rank() == 0;
  if (threadIdx.x == 0 && leader) {
    const uint32_t idesc = idesc_bf16_f32(PAIR ? 2 * M : M, N);
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 48 * 1024);
    long long t0 = clock64();
    // like the conv issue loop: per "tap" 8 MMAs (2 accumulators × 4 k16)
    // at compile-time offsets from a per-tap base, then optional commit/wait
    const bool commit = commit_every != 0;
    for (int j = 0; j < iters / 8; ++j) {
      const int tap = j % 9;
      const uint32_t abase = a + tap * a_step;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t ad = smem_desc(abase + 2 * kk * lbo_a + h * 32, lbo_a, 128);
          const uint64_t bd = smem_desc(b + 2 * kk * lbo_b, lbo_b, 128);
          if (PAIR) mma_bf16_pair(tmem + h * 128, ad, bd, idesc, (j | kk) != 0);
          else mma_bf16(tmem + h * 128, ad, bd, idesc, (j | kk) != 0);
        }
      }
      if (commit) {
        if (PAIR) mma_commit_pair(&dbar, 0x3); else mma_commit(&dbar);
        if (wait_too) { mbar_wait(&cbar2, 0); tc_fence_after(); }
      }
    }
    if (PAIR) mma_commit_pair(&bar, 0x3); else mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
    done = 1;
  } else if (warp >= 2 && warp - 2 < ld_warps) {  // concurrent TMEM reads (epilogue-like)
    float acc = 0.f;
    const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
    while (!done) {
      float v[32];
      for (int c = 256; c < 512; c += 32) {
        tmem_ld32(tmem + lane_base + c, v);
        for (int j = 0; j < 32; ++j) acc += v[j];
      }
    }
    if (acc == 12345.f) out[blockIdx.x + 128] = 1;
  } else if (threadIdx.x == 64 && copy_kb > 0) {  // concurrent bulk copies into smem
    uint32_t ph = 0;
    while (!done) {
      mbar_expect_tx(&cbar, copy_kb * 1024);
      bulk_g2s(smem + 96 * 1024, gsrc + (blockIdx.x % 8) * 65536, copy_kb * 1024, &cbar);
      mbar_wait(&cbar, ph);
      ph ^= 1;
    }
  } else if (PAIR && threadIdx.x == 0) {
    mbar_wait(&bar, 0);
    out[blockIdx.x] = 0;
    done = 1;
  }
  tc_fence_before();
  if (PAIR) cluster_sync(); else __syncthreads();
  if (warp == 1) { tc_fence_after(); if (PAIR) tmem_dealloc_pair(tmem, 512); else tmem_dealloc(tmem, 512); }
}

template <int M, int N, bool PAIR>
void run(const char* name, int blocks, int copy_kb = 0, int a_step = 32, int lbo_a = M * 16, int commit_every = 0, int ld_warps = 0) {
  static uint8_t* gsrc = nullptr;
  if (!gsrc) { cudaMalloc(&gsrc, 1 << 20); cudaMemset(gsrc, 0, 1 << 20); }
  long long* d; cudaMalloc(&d, sizeof(long long) * 256);
  const int iters = 4096;
  auto k = k_rate<M, N, PAIR>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(blocks); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = 200 * 1024;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = PAIR ? 2 : 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaLaunchKernelEx(&cfg, k, d, iters, (uint32_t)lbo_a, (uint32_t)(N * 16), (const uint8_t*)gsrc, copy_kb, a_step, commit_every, ld_warps);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, k, d, iters, (uint32_t)lbo_a, (uint32_t)(N * 16), (const uint8_t*)gsrc, copy_kb, a_step, commit_every, ld_warps);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long h[256]; cudaMemcpy(h, d, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
  long long mx = 0; for (int i = 0; i < blocks; ++i) mx = h[i] > mx ? h[i] : mx;
  const double flop_per = 2.0 * (PAIR ? 2 * M : M) * N * 16;
  const double sms = blocks;
  printf("%-28s copy=%dKB err=%d cycles/mma=%7.1f  per-SM flop/cycle=%7.1f  chip TFLOP/s=%7.1f\n", name, (int)err,
         copy_kb, (double)mx / iters, flop_per * iters / mx / (PAIR ? 2 : 1),
         flop_per * iters * (PAIR ? blocks / 2 : blocks) / (ms * 1e-3) / 1e12);
  cudaFree(d);
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  run<128, 128, false>("M128 N128 K16 (1 CTA)", 148);
  run<128, 128, false>("tmem ld 1 warp", 148, 0, 16, 4608, 0, 1);
  run<128, 128, false>("tmem ld 2 warps", 148, 0, 16, 4608, 0, 2);
  run<128, 128, true>("pair tmem ld 2 warps", 148, 0, 16, 4608, 0, 2);
  run<128, 256, false>("N256 tmem ld 2 warps", 148, 0, 16, 4608, 0, 2);
  run<128, 128, false>("commit/8", 148, 0, 16, 4608, 8);
  run<128, 128, false>("commit/8 + wait", 148, -1, 16, 4608, 8);
  run<128, 128, false>("commit/4 + wait", 148, -1, 16, 4608, 4);
  run<128, 128, true>("pair commit/8", 148, 0, 16, 4608, 8);
  run<128, 128, true>("pair commit/8 + wait", 148, -1, 16, 4608, 8);
  run<128, 256, false>("N256 commit/4 + wait", 148, -1, 16, 4608, 4);
  run<128, 128, false>("M128N128 A step 0", 148, 0, 0);
  run<128, 128, false>("M128N128 A step 16B", 148, 0, 16);
  run<128, 128, false>("M128N128 A step 128B", 148, 0, 128);
  run<128, 128, false>("M128N128 A 16B lbo4608", 148, 0, 16, 4608);
  run<128, 128, false>("M128N128 A 128B lbo4608", 148, 0, 128, 4608);
  run<128, 128, true>("pair A step 16B lbo4608", 148, 0, 16, 4608);
  run<128, 128, true>("pair A step 128B lbo4608", 148, 0, 128, 4608);
  run<128, 128, false>("M128N128 16B lbo4608 +cp32", 148, 32, 16, 4608);
  run<128, 128, true>("pair 16B lbo4608 +cp32", 148, 32, 16, 4608);
  run<128, 128, false>("M128 N128 +copy16KB", 148, 16);
  run<128, 128, false>("M128 N128 +copy64KB", 148, 64);
  run<128, 256, false>("M128 N256 +copy64KB", 148, 64);
  run<128, 128, true>("M256 N128 pair +copy64KB", 148, 64);
  run<128, 256, false>("M128 N256 K16 (1 CTA)", 148);
  run<64, 128, false>("M64 N128 K16 (1 CTA)", 148);
  run<128, 128, true>("M256 N128 K16 (pair)", 148);
  run<128, 256, true>("M256 N256 K16 (pair)", 148);
  return 0;
}
