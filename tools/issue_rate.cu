// issue_rate.cu — microbenchmark: how much per-MMA issue work the single
// tcgen05.mma thread can afford at M=128, N=256, K=16 (128 cycles ideal).
// mode 0: constant descriptors (no arithmetic between MMAs);
// mode 1: descriptors rebuilt per MMA with smem_desc_sw128 (as k_rb_step);
// mode 2: precomputed base descriptors + 64-bit adds;
// mode 3: mode 2 + per-stage commit + wait on a pre-completed barrier;
// mode 4: mode 0 + per-stage commit only; 5-7: accumulator placement.
#include <cstdio>
#include <cuda_runtime.h>
#include "tc_common.cuh"

using namespace dbk;

__global__ void __launch_bounds__(128, 1) k_issue(long long* out, int stages, int mode) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, cb, acc_full[2], acc_empty[2], rb_full[8], rb_empty[8];
  __shared__ uint32_t slot;
  uint64_t* pre = reinterpret_cast<uint64_t*>(smem + 160 * 1024);
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&cb, 1);
    for (int i = 0; i < 2; ++i) { mbar_init(&acc_full[i], 1); mbar_init(&acc_empty[i], 1); }
    for (int i = 0; i < 8; ++i) { mbar_init(&rb_full[i], 1); mbar_init(&rb_empty[i], 1); }
    for (int i = 0; i < stages; ++i) { mbar_init(&pre[i], 1); mbar_arrive(&pre[i]); }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&slot, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 32) {
    const uint32_t idesc = idesc_f16_f32(128, 256);
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 64 * 1024);
    const uint64_t wd0 = smem_desc_sw128(a), xd0 = smem_desc_sw128(b);
    const long long t0 = clock64();
    if (mode == 0 || mode == 4) {
      for (int t = 0; t < stages; ++t) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) mma_bf16(tmem, wd0, xd0, idesc, 1);
        if (mode == 4) mma_commit(&cb);
      }
    } else if (mode >= 11) {
      // 11: a real S=4 stage ring fed by a second warp (waits rb_empty, arrives
      // rb_full), no clock reads; 12: S=8; 13: S=4 with the tcgen05 fence
      const int S = mode == 12 ? 8 : 4;
      for (int t = 0; t < stages; ++t) {
        const int s = t % S;
        mbar_wait(&rb_full[s], (t / S) & 1);
        if (mode == 13) tc_fence_after();
        const uint64_t wd = wd0 + static_cast<uint64_t>((t & 3) * (16384 >> 4));
        const uint64_t xd = xd0 + static_cast<uint64_t>((15 + t % 3) * (128 >> 4));
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) mma_bf16(tmem, wd + 2 * kk, xd + 2 * kk, idesc, 1);
        mma_commit(&rb_empty[s]);
      }
    } else if (mode >= 8) {
      // 8: two accumulators, 18 stages per tile, acc_empty wait + acc_full
      // commit per tile (an epilogue thread hands the buffers back); 9: as 8
      // without the tcgen05 fence after the wait; 10: commit only, no waits
      for (int n = 0; n < stages / 18; ++n) {
        const int abuf = n & 1;
        if (mode != 10) {
          mbar_wait(&acc_empty[abuf], ((n >> 1) & 1) ^ 1);
          if (mode == 8) tc_fence_after();
        }
        for (int t = 0; t < 18; ++t) {
          const int s = t & 3, row = 15 + (t % 3);
          const uint64_t wd = wd0 + static_cast<uint64_t>(s * (16384 >> 4));
          const uint64_t xd = xd0 + static_cast<uint64_t>(row * (128 >> 4));
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) mma_bf16(tmem + abuf * 256, wd + 2 * kk, xd + 2 * kk, idesc, (t | kk) != 0);
        }
        mma_commit(&acc_full[abuf]);
      }
    } else if (mode >= 5) {
      // 5: alternate two accumulators every 18 stages; 6: columns 256-511 only;
      // 7: mode 5 with accumulate = 0 on each tile's first MMA
      for (int t = 0; t < stages; ++t) {
        const int s = t & 3, row = 15 + (t % 3);
        const uint32_t d = mode == 6 ? tmem + 256 : tmem + ((t / 18) & 1) * 256;
        const uint64_t wd = wd0 + static_cast<uint64_t>(s * (16384 >> 4));
        const uint64_t xd = xd0 + static_cast<uint64_t>(row * (128 >> 4));
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_bf16(d, wd + 2 * kk, xd + 2 * kk, idesc, mode == 7 ? ((t % 18) | kk) != 0 : 1);
      }
    } else if (mode == 1) {
      for (int t = 0; t < stages; ++t) {
        const int s = t & 3, row = 15 + (t % 3);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t wd = smem_desc_sw128(a + s * 16384 + kk * 32);
          const uint64_t xd = smem_desc_sw128(b + row * 128 + kk * 32);
          mma_bf16(tmem, wd, xd, idesc, 1);
        }
      }
    } else {
      for (int t = 0; t < stages; ++t) {
        const int s = t & 3, row = 15 + (t % 3);
        if (mode == 3) {
          mbar_wait(&pre[t], 0);
          tc_fence_after();
        }
        const uint64_t wd = wd0 + static_cast<uint64_t>(s * (16384 >> 4));
        const uint64_t xd = xd0 + static_cast<uint64_t>(row * (128 >> 4));
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) mma_bf16(tmem, wd + 2 * kk, xd + 2 * kk, idesc, 1);
        if (mode == 3) mma_commit(&cb);
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    out[blockIdx.x] = clock64() - t0;
  } else if (threadIdx.x == 64 && mode >= 11) {  // weight-stage feeder
    const int S = mode == 12 ? 8 : 4;
    for (int t = 0; t < stages; ++t) {
      const int s = t % S;
      mbar_wait(&rb_empty[s], ((t / S) & 1) ^ 1);
      mbar_arrive(&rb_full[s]);
    }
  } else if (threadIdx.x == 64 && (mode == 8 || mode == 9)) {  // epilogue stand-in
    for (int n = 0; n < stages / 18; ++n) {
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

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  long long* d; cudaMalloc(&d, sizeof(long long) * 256);
  cudaFuncSetAttribute(k_issue, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int stages = 3600;
  for (int rep = 0; rep < 2; ++rep)
    for (int mode = 0; mode <= 13; ++mode) {
      k_issue<<<148, 128, 200 * 1024>>>(d, stages, mode);
      k_issue<<<148, 128, 200 * 1024>>>(d, stages, mode);
      const cudaError_t err = cudaDeviceSynchronize();
      long long h[148];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double cyc = 0;
      for (int i = 0; i < 148; ++i) cyc += h[i] / 148.0;
      printf("mode %d err %d: cycles per MMA %.1f (ideal 128)\n", mode, static_cast<int>(err), cyc / (stages * 4.0));
    }
  return 0;
}
