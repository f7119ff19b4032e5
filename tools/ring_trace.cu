// ring_trace.cu — timeline of the weight-stage handshake (see ring_rate.cu):
// per stage, the issuer's clock before its b_full wait, after it, and after
// its commit; the weight warp's clock when it observed b_empty (the MMAs of
// the stage S uses back completed) and when it arrived on b_full. One CTA per
// SM; CTA 0's trace of stages 100..163 is printed. Args: S, MMAs per stage.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "tc_common.cuh"

using namespace dbk;

constexpr int kMaxS = 8;
constexpr int kT0 = 100, kTN = 64;

__global__ void __launch_bounds__(128, 1) k_ring(long long* out, int stages, int S, int per) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t b_full[kMaxS], b_empty[kMaxS], done;
  __shared__ uint32_t slot;
  __shared__ long long tr[5][kTN];
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kMaxS; ++s) { mbar_init(&b_full[s], 1); mbar_init(&b_empty[s], 1); }
    mbar_init(&done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&slot, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 1 && lane == 0) {
    const uint32_t idesc = idesc_f16_f32(128, 256);
    const uint64_t wd0 = smem_desc_sw128(smem_u32(smem)), xd0 = smem_desc_sw128(smem_u32(smem + 64 * 1024));
    const long long t0 = clock64();
    for (int t = 0; t < stages; ++t) {
      const int s = t % S;
      const long long c0 = clock64();
      mbar_wait(&b_full[s], (t / S) & 1);
      const long long c1 = clock64();
      tc_fence_after();
      for (int k = 0; k < per; ++k) mma_bf16(tmem, wd0 + 2 * (k & 3), xd0 + 2 * (k & 3), idesc, (t | k) != 0);
      mma_commit(&b_empty[s]);
      const long long c2 = clock64();
      if (t >= kT0 && t < kT0 + kTN) { tr[0][t - kT0] = c0; tr[1][t - kT0] = c1; tr[2][t - kT0] = c2; }
    }
    mma_commit(&done);
    mbar_wait(&done, 0);
    out[blockIdx.x] = clock64() - t0;
  } else if (warp == 2 && lane == 0) {
    for (int t = 0; t < stages; ++t) {
      const int s = t % S;
      mbar_wait(&b_empty[s], ((t / S) & 1) ^ 1);
      const long long c3 = clock64();
      mbar_arrive(&b_full[s]);
      if (t >= kT0 && t < kT0 + kTN) { tr[3][t - kT0] = c3; tr[4][t - kT0] = clock64(); }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x < kTN)
    for (int r = 0; r < 5; ++r) out[256 + r * kTN + threadIdx.x] = tr[r][threadIdx.x];
  if (warp == 1) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

int main(int argc, char** argv) {
  const int S = argc > 1 ? atoi(argv[1]) : 4, per = argc > 2 ? atoi(argv[2]) : 4;
  long long* d; cudaMalloc(&d, sizeof(long long) * 1024);
  cudaFuncSetAttribute(k_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int stages = 2000;
  k_ring<<<148, 128, 200 * 1024>>>(d, stages, S, per);
  k_ring<<<148, 128, 200 * 1024>>>(d, stages, S, per);
  const cudaError_t err = cudaDeviceSynchronize();
  long long h[1024];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double cyc = 0;
  for (int i = 0; i < 148; ++i) cyc += h[i] / 148.0;
  printf("S=%d per=%d err=%d cycles per MMA %.1f (ideal 128)\n", S, per, (int)err, cyc / (stages * per));
  const long long* tr = h + 256;
  const long long base = tr[0];
  printf(" t | wait_start wait_end commit_done | empty_seen(t) full_arrive(t) | wait  issue->empty_seen\n");
  for (int i = 0; i < 24; ++i)
    printf("%2d | %8lld %8lld %8lld | %8lld %8lld | %5lld %6lld\n", i, tr[i] - base, tr[64 + i] - base,
           tr[128 + i] - base, tr[192 + i] - base, tr[256 + i] - base, tr[64 + i] - tr[i],
           (i + S < 64) ? tr[192 + i + S] - tr[128 + i] : -1);
  return 0;
}
