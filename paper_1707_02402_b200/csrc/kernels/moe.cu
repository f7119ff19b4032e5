// moe.cu — sparsely-gated MoE layer kernels (gate, fp64 experts, combine).
//
//   top_k_gate .......... src/moe.cpp:36-69   → k_topk (one warp per token)
//   ExpertSet::apply .... src/moe.cpp:98-145  → k_expert_fp64_{hidden,out}
//   batched staging ..... src/moe.cpp:244-251 → rows land at token·k + slot
//   combine ............. src/moe.cpp:254-264 → k_combine_fp64
// The dispatch (group_by_function, src/schedule.cpp:166-169) is the stable
// bucket sort in sched.cu keyed by expert id over (token, slot) order. All
// fp64 arithmetic follows the reference's ascending fused multiply-add
// order, so batched outputs equal the reference's bit for bit up to the
// last-ulp behaviour of exp() in the gate.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "dynbatch/dbk.h"

namespace {


// Rank order of the reference: higher score first, lower id on ties; `==`
// on doubles makes -0.0 tie with +0.0.
__device__ __forceinline__ bool ranks_before(double va, int ia, double vb, int ib) {
  return va > vb || (va == vb && ia < ib);
}

template <int kLocal>
__global__ void __launch_bounds__(256, kLocal == 4 ? 4 : 2) k_topk(int64_t T, int32_t n, int32_t k, const double* __restrict__ scores,
                       int32_t* __restrict__ ids, double* __restrict__ weights,
                       int32_t* __restrict__ err) {
  extern __shared__ double sel_v[];  // [warps][k]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x >> 5) + warp;
  if (t >= T) return;
  const double* row = scores + t * n;
  double* my_sel = sel_v + static_cast<int64_t>(warp) * k;
  double thr_v = INFINITY;
  int thr_i = -1;  // items must rank strictly after (thr_v, thr_i)
  int32_t taken = 0;
  bool first = true;
  while (taken < k) {
    double lv[kLocal];
    int li[kLocal];
#pragma unroll
    for (int q = 0; q < kLocal; ++q) { lv[q] = -INFINITY; li[q] = 0x7fffffff; }
    bool bad = false;
    auto consider = [&](double v, int j) {
      bad |= !isfinite(v);
      if (thr_i >= 0 && !ranks_before(thr_v, thr_i, v, j)) return;
      if (!ranks_before(v, j, lv[kLocal - 1], li[kLocal - 1])) return;
      // insertion into the lane's sorted candidate list
      double cv = v;
      int ci = j;
#pragma unroll
      for (int q = 0; q < kLocal; ++q) {
        if (ranks_before(cv, ci, lv[q], li[q])) {
          const double tv = lv[q];
          const int ti = li[q];
          lv[q] = cv; li[q] = ci; cv = tv; ci = ti;
        }
      }
    };
    if ((n & 1) == 0) {
      // 16-byte loads, 512 contiguous bytes per warp and round; the next
      // round's loads are issued before this round is ranked
      const double2* row2 = reinterpret_cast<const double2*>(row);
      const int32_t n2 = n >> 1;
      double2 nx[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int32_t j2 = lane + 32 * u;
        nx[u] = j2 < n2 ? __ldg(row2 + j2) : make_double2(-INFINITY, -INFINITY);
      }
      for (int32_t b2 = 0; b2 < n2; b2 += 128) {
        double2 c[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) c[u] = nx[u];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int32_t j2 = b2 + 128 + lane + 32 * u;
          nx[u] = j2 < n2 ? __ldg(row2 + j2) : make_double2(-INFINITY, -INFINITY);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int32_t j2 = b2 + lane + 32 * u;
          if (j2 < n2) {
            consider(c[u].x, 2 * j2);
            consider(c[u].y, 2 * j2 + 1);
          }
        }
      }
    } else {
      for (int32_t j = lane; j < n; j += 32) consider(__ldg(row + j), j);
    }
    // Non-finite scores are rejected before any result is written
    // (src/moe.cpp:41); the first pass reads every score.
    if (first && __any_sync(0xffffffffu, bad)) {
      if (lane == 0) atomicCAS(err, 0, 9);
      return;
    }
    first = false;
    const int32_t rounds = min(kLocal, k - taken);
    int head = 0;
    for (int32_t r = 0; r < rounds; ++r) {
      double bv = head < kLocal ? lv[0] : -INFINITY;
      int bi = head < kLocal ? li[0] : 0x7fffffff;
      int owner = lane;
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        const int oo = __shfl_xor_sync(0xffffffffu, owner, o);
        if (ranks_before(ov, oi, bv, bi)) { bv = ov; bi = oi; owner = oo; }
      }
      if (lane == owner) {  // pop the winner's head
#pragma unroll
        for (int q = 0; q < kLocal - 1; ++q) { lv[q] = lv[q + 1]; li[q] = li[q + 1]; }
        lv[kLocal - 1] = -INFINITY;
        li[kLocal - 1] = 0x7fffffff;
        ++head;
      }
      if (lane == 0) {
        ids[t * k + taken + r] = bi;
        my_sel[taken + r] = bv;
      }
      thr_v = bv;
      thr_i = bi;
    }
    taken += rounds;
  }
  __syncwarp();
  // weight_r = exp(s_r − s_0) / Σ_{j<k} exp(s_j − s_0), the denominator
  // summed in rank order as the reference does; the exps run in parallel
  // (lane r holds rank r, chunks of 32 for k > 32).
  const double top = my_sel[0];
  double denom = 0.0;
  for (int32_t base = 0; base < k; base += 32) {
    const double e = base + lane < k ? exp(my_sel[base + lane] - top) : 0.0;
    const int32_t m = min(32, k - base);
    for (int32_t r = 0; r < m; ++r) denom += __shfl_sync(0xffffffffu, e, r);
  }
  for (int32_t r = lane; r < k; r += 32) weights[t * k + r] = exp(my_sel[r] - top) / denom;
}

// Small gates (n ≤ 128 even, k ≤ 8): one thread per token, reading its own
// score row with 16-byte loads (eight in flight per 16-score chunk) and
// keeping its top-k in registers in the reference's rank order; the weights
// use the denominator summed in rank order. Non-finite scores are rejected
// before anything is written (src/moe.cpp:41).
template <int K>
__global__ void __launch_bounds__(64) k_topk_small(int64_t T, int32_t n, const double* __restrict__ scores,
                                                    int32_t* __restrict__ ids, double* __restrict__ weights,
                                                    int32_t* __restrict__ err) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const bool live = t < T;
  const double2* row = reinterpret_cast<const double2*>(scores + (live ? t : 0) * n);
  double tv[K];
  int ti[K];
#pragma unroll
  for (int q = 0; q < K; ++q) { tv[q] = -INFINITY; ti[q] = 0x7fffffff; }
  bool bad = false;
  // 128-byte rounds, the next round's loads issued before this one is ranked
  double2 nx[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) nx[u] = 2 * u < n ? __ldg(row + u) : make_double2(-INFINITY, -INFINITY);
  for (int32_t j0 = 0; j0 < n; j0 += 16) {
    double2 c[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) c[u] = nx[u];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      nx[u] = j0 + 16 + 2 * u < n ? __ldg(row + (j0 + 16) / 2 + u) : make_double2(-INFINITY, -INFINITY);
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int32_t j = j0 + u;
      if (j >= n) break;
      double cv = (u & 1) ? c[u >> 1].y : c[u >> 1].x;
      bad |= !isfinite(cv);
      int ci = j;
      if (!ranks_before(cv, ci, tv[K - 1], ti[K - 1])) continue;
#pragma unroll
      for (int q = 0; q < K; ++q) {
        if (ranks_before(cv, ci, tv[q], ti[q])) {
          const double sv = tv[q];
          const int si = ti[q];
          tv[q] = cv; ti[q] = ci; cv = sv; ci = si;
        }
      }
    }
  }
  if (__syncthreads_or(live && bad)) {
    if (threadIdx.x == 0) atomicCAS(err, 0, 9);
    return;
  }
  if (!live) return;
  double e[K], denom = 0.0;
#pragma unroll
  for (int q = 0; q < K; ++q) {
    e[q] = exp(tv[q] - tv[0]);
    denom += e[q];
  }
#pragma unroll
  for (int q = 0; q < K; ++q) {
    ids[t * K + q] = ti[q];
    weights[t * K + q] = e[q] / denom;
  }
}

constexpr int kRows = 8;

// Tiles of up to kRows rows of one expert; tile_begin[e] = Σ_{<e} ceil(rows/kRows).
__global__ void k_tile_offsets(int32_t n, const int32_t* __restrict__ offsets,
                               int32_t* __restrict__ tile_begin) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int32_t acc = 0;
  for (int32_t e = 0; e < n; ++e) {
    tile_begin[e] = acc;
    acc += (offsets[e + 1] - offsets[e] + kRows - 1) / kRows;
  }
  tile_begin[n] = acc;
}

__device__ __forceinline__ int32_t find_expert(int32_t n, const int32_t* tile_begin, int32_t t) {
  int32_t lo = 0, hi = n;  // largest e with tile_begin[e] <= t and non-empty
  while (hi - lo > 1) {
    const int32_t mid = (lo + hi) >> 1;
    if (tile_begin[mid] <= t) lo = mid; else hi = mid;
  }
  while (lo + 1 <= n && tile_begin[lo + 1] <= t) ++lo;
  return lo;
}

// h = relu(x · W1) for kRows rows of one expert: acc_j = Σ_i fma(x_i, W1[i][j]).
__global__ void __launch_bounds__(128) k_expert_hidden(
    int32_t n, int32_t k, int32_t d, int32_t h, const int32_t* __restrict__ order,
    const int32_t* __restrict__ offsets, const int32_t* __restrict__ tile_begin,
    const double* __restrict__ x, const double* const* __restrict__ w1,
    double* __restrict__ hidden) {
  extern __shared__ double xs[];  // [kRows][d]
  const int32_t total = tile_begin[n];
  for (int32_t t = blockIdx.x; t < total; t += gridDim.x) {
    const int32_t e = find_expert(n, tile_begin, t);
    const int32_t r0 = offsets[e] + (t - tile_begin[e]) * kRows;
    const int32_t rows = min(kRows, offsets[e + 1] - r0);
    __syncthreads();
    for (int32_t r = 0; r < rows; ++r) {
      const double* src = x + static_cast<int64_t>(order[r0 + r] / k) * d;
      for (int32_t i = threadIdx.x; i < d; i += blockDim.x) xs[r * d + i] = src[i];
    }
    __syncthreads();
    const double* __restrict__ w = w1[e];
    for (int32_t j = threadIdx.x; j < h; j += blockDim.x) {
      double acc[kRows];
#pragma unroll
      for (int r = 0; r < kRows; ++r) acc[r] = 0.0;
      for (int32_t i = 0; i < d; ++i) {
        const double wij = w[static_cast<int64_t>(i) * h + j];
#pragma unroll
        for (int r = 0; r < kRows; ++r) acc[r] = __fma_rn(xs[(r < rows ? r : 0) * d + i], wij, acc[r]);
      }
      for (int r = 0; r < rows; ++r) hidden[static_cast<int64_t>(r0 + r) * h + j] = acc[r] > 0.0 ? acc[r] : 0.0;
    }
  }
}

// y = h · W2, written to staged[token·k + slot].
__global__ void __launch_bounds__(128) k_expert_out(
    int32_t n, int32_t d, int32_t h, const int32_t* __restrict__ order,
    const int32_t* __restrict__ offsets, const int32_t* __restrict__ tile_begin,
    const double* const* __restrict__ w2, const double* __restrict__ hidden,
    double* __restrict__ staged) {
  extern __shared__ double hs[];  // [kRows][h]
  const int32_t total = tile_begin[n];
  for (int32_t t = blockIdx.x; t < total; t += gridDim.x) {
    const int32_t e = find_expert(n, tile_begin, t);
    const int32_t r0 = offsets[e] + (t - tile_begin[e]) * kRows;
    const int32_t rows = min(kRows, offsets[e + 1] - r0);
    __syncthreads();
    for (int32_t r = 0; r < rows; ++r)
      for (int32_t i = threadIdx.x; i < h; i += blockDim.x)
        hs[r * h + i] = hidden[static_cast<int64_t>(r0 + r) * h + i];
    __syncthreads();
    const double* __restrict__ w = w2[e];
    for (int32_t j = threadIdx.x; j < d; j += blockDim.x) {
      double acc[kRows];
#pragma unroll
      for (int r = 0; r < kRows; ++r) acc[r] = 0.0;
      for (int32_t i = 0; i < h; ++i) {
        const double wij = w[static_cast<int64_t>(i) * d + j];
#pragma unroll
        for (int r = 0; r < kRows; ++r) acc[r] = __fma_rn(hs[(r < rows ? r : 0) * h + i], wij, acc[r]);
      }
      for (int r = 0; r < rows; ++r) staged[static_cast<int64_t>(order[r0 + r]) * d + j] = acc[r];
    }
  }
}

__global__ void k_combine_fp64(int64_t T, int32_t k, int32_t d, const double* __restrict__ w,
                               const double* __restrict__ staged, double* __restrict__ out) {
  const int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (idx >= T * d) return;
  const int64_t t = idx / d, j = idx % d;
  double acc = 0.0;
  for (int32_t s = 0; s < k; ++s) acc = __fma_rn(w[t * k + s], staged[(t * k + s) * d + j], acc);
  out[idx] = acc;
}

}  // namespace

template <int K>
int launch_topk_small(int64_t T, int32_t n, const double* scores, int32_t* ids, double* weights, int32_t* err,
                      cudaStream_t s) {
  k_topk_small<K><<<static_cast<unsigned>((T + 63) / 64), 64, 0, s>>>(T, n, scores, ids, weights, err);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_moe_topk(int64_t T, int32_t n, int32_t k, const double* scores, int32_t* ids,
                            double* weights, int32_t* err, void* stream) {
  if (T <= 0) return 0;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (n <= 128 && n % 2 == 0 && k <= n) {
    switch (k) {
      case 1: return launch_topk_small<1>(T, n, scores, ids, weights, err, st);
      case 2: return launch_topk_small<2>(T, n, scores, ids, weights, err, st);
      case 3: return launch_topk_small<3>(T, n, scores, ids, weights, err, st);
      case 4: return launch_topk_small<4>(T, n, scores, ids, weights, err, st);
      case 8: return launch_topk_small<8>(T, n, scores, ids, weights, err, st);
      default: break;
    }
  }
  const int warps = 8;
  const size_t smem = sizeof(double) * static_cast<size_t>(warps) * k;
  const unsigned blocks = static_cast<unsigned>((T + warps - 1) / warps);
  // per-lane candidate lists: 4 deep when k ≤ 4 (shorter insertion chains,
  // fewer registers), else 8 deep with further passes for k > 8
  if (k <= 4) {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(k_topk<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    k_topk<4><<<blocks, warps * 32, smem, st>>>(T, n, k, scores, ids, weights, err);
  } else {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(k_topk<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    k_topk<8><<<blocks, warps * 32, smem, st>>>(T, n, k, scores, ids, weights, err);
  }
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_moe_expert_fp64(int64_t T, int32_t n, int32_t k, int32_t d, int32_t h,
                                   const int32_t* order, const int32_t* offsets,
                                   const double* x, const double* const* w1,
                                   const double* const* w2, double* hidden, double* staged,
                                   int32_t* tile_scratch, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (T <= 0) return 0;
  k_tile_offsets<<<1, 32, 0, s>>>(n, offsets, tile_scratch);
  const size_t s1 = sizeof(double) * kRows * static_cast<size_t>(d);
  const size_t s2 = sizeof(double) * kRows * static_cast<size_t>(h);
  if (s1 > 227 * 1024 || s2 > 227 * 1024) return static_cast<int>(cudaErrorInvalidValue);
  cudaFuncSetAttribute(k_expert_hidden, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(s1));
  cudaFuncSetAttribute(k_expert_out, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(s2));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int blocks = sms * 8;
  k_expert_hidden<<<blocks, 128, s1, s>>>(n, k, d, h, order, offsets, tile_scratch, x, w1, hidden);
  k_expert_out<<<blocks, 128, s2, s>>>(n, d, h, order, offsets, tile_scratch, w2, hidden, staged);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_moe_combine_fp64(int64_t T, int32_t k, int32_t d, const double* weights,
                                    const double* staged, double* out, void* stream) {
  if (T <= 0) return 0;
  const int64_t total = T * d;
  k_combine_fp64<<<static_cast<unsigned>((total + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      T, k, d, weights, staged, out);
  return static_cast<int>(cudaGetLastError());
}
