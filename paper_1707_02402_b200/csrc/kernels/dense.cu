// dense.cu — Tier-A module body on device: the reference's dense fp64 layer.
//
// One launch per schedule step runs every call group of the step
// (execute(), src/executor.cpp:117-166): leaf groups fetch the example's
// input row (:126-137); expensive groups gather child k of each member as
// operand k (:139-151) straight from the node-value slab, apply
//   out[j] = relu(bias[j] + Σ_k Σ_i x_k[i] · W[(k·W + i)·W + j])
// with the reference's ascending fused-multiply-add chain per output
// (src/modules.cpp:83-105 as compiled with FMA contraction), and scatter the
// row back to the member's slot (:161-163). Per-output accumulation order is
// identical whatever the grouping, so results are bit-identical to the
// reference CPU path. Presence words reproduce ValueStore's checks
// (src/executor.cpp:48-70): a missing child → MissingOperand, a second write
// → SingleAssignmentViolation, non-finite output → NonFiniteValue.
#include <cuda_runtime.h>
#include <stdint.h>

#include "dynbatch/dbk.h"

namespace {

constexpr int kRows = 8;  // members per block tile: weights are read once per 8 rows

enum : int32_t { kErrMissing = 7, kErrNonFinite = 9, kErrDouble = 14 };

__device__ __forceinline__ void set_err(int32_t* err, int32_t code) { atomicCAS(err, 0, code); }

__global__ void __launch_bounds__(128) k_dense_step(
    int32_t step, int32_t W, const int32_t* __restrict__ step_group_begin,
    const int32_t* __restrict__ group_fid, const int32_t* __restrict__ group_begin,
    const int32_t* __restrict__ member_g, const int32_t* __restrict__ arity_of,
    const int32_t* __restrict__ child_off, const int32_t* __restrict__ child_list,
    const int32_t* __restrict__ example, const double* __restrict__ inputs,
    double* __restrict__ values, int32_t* __restrict__ present,
    const double* const* __restrict__ weights, const double* const* __restrict__ biases,
    int32_t* __restrict__ err) {
  extern __shared__ double xs[];  // [kRows][max_arity * W]
  __shared__ int32_t s_node[kRows];
  __shared__ int32_t s_ok[kRows];
  const int32_t g_lo = step_group_begin[step], g_hi = step_group_begin[step + 1];
  // Tiles: each group contributes ceil(rows / kRows) tiles.
  int32_t total_tiles = 0;
  for (int32_t g = g_lo; g < g_hi; ++g) total_tiles += (group_begin[g + 1] - group_begin[g] + kRows - 1) / kRows;
  for (int32_t t = blockIdx.x; t < total_tiles; t += gridDim.x) {
    int32_t g = g_lo, acc_tiles = 0;
    for (;; ++g) {
      const int32_t nt = (group_begin[g + 1] - group_begin[g] + kRows - 1) / kRows;
      if (t < acc_tiles + nt) break;
      acc_tiles += nt;
    }
    const int32_t m0 = group_begin[g] + (t - acc_tiles) * kRows;
    const int32_t rows = min(kRows, group_begin[g + 1] - m0);
    const int32_t f = group_fid[g];
    const int32_t a = arity_of[f];
    const int32_t xw = a * W;
    __syncthreads();
    if (threadIdx.x < kRows) {
      int32_t ok = 0, node = -1;
      if (static_cast<int32_t>(threadIdx.x) < rows) {
        node = member_g[m0 + threadIdx.x];
        ok = 1;
        for (int32_t c = child_off[node]; c < child_off[node + 1]; ++c) {
          if (atomicAdd(&present[child_list[c]], 0) == 0) {
            set_err(err, kErrMissing);
            ok = 0;
          }
        }
        if (atomicOr(&present[node], 2) != 0) {  // claim; 2 = being written
          set_err(err, kErrDouble);
          ok = 0;
        }
      }
      s_node[threadIdx.x] = node;
      s_ok[threadIdx.x] = ok;
    }
    __syncthreads();
    if (a == 0) {  // leaf fetch: copy inputs[example]
      for (int32_t r = 0; r < rows; ++r) {
        if (!s_ok[r]) continue;
        const int32_t node = s_node[r];
        const double* src = inputs + static_cast<int64_t>(example[node]) * W;
        double* dst = values + static_cast<int64_t>(node) * W;
        for (int32_t j = threadIdx.x; j < W; j += blockDim.x) dst[j] = src[j];
      }
    } else {
      // Stage the operand rows (children in operand order) in shared memory.
      for (int32_t r = 0; r < rows; ++r) {
        if (!s_ok[r]) continue;
        const int32_t node = s_node[r];
        for (int32_t k = 0; k < a; ++k) {
          const double* src = values + static_cast<int64_t>(child_list[child_off[node] + k]) * W;
          for (int32_t i = threadIdx.x; i < W; i += blockDim.x) xs[r * xw + k * W + i] = src[i];
        }
      }
      __syncthreads();
      const double* __restrict__ w = weights[f];
      const double* __restrict__ bias = biases[f];
      for (int32_t j = threadIdx.x; j < W; j += blockDim.x) {
        double acc[kRows];
#pragma unroll
        for (int r = 0; r < kRows; ++r) acc[r] = bias[j];
        for (int32_t i = 0; i < xw; ++i) {
          const double wij = w[static_cast<int64_t>(i) * W + j];
#pragma unroll
          for (int r = 0; r < kRows; ++r) acc[r] = __fma_rn(xs[r * xw + i], wij, acc[r]);
        }
        for (int r = 0; r < rows; ++r) {
          if (!s_ok[r]) continue;
          const double v = acc[r] > 0.0 ? acc[r] : 0.0;
          if (!isfinite(v)) set_err(err, kErrNonFinite);
          values[static_cast<int64_t>(s_node[r]) * W + j] = v;
        }
      }
    }
    __syncthreads();
    if (threadIdx.x < kRows && s_ok[threadIdx.x]) {
      __threadfence();
      atomicExch(&present[s_node[threadIdx.x]], 1);
    }
  }
}

// apply_module on stacked operand rows (src/modules.cpp:52-108): x is
// [rows][a·W] (operand k of row r at x[r·a·W + k·W]), out[r][j] =
// relu(bias[j] + Σ_i x[r][i] · w[i·W + j]), the same fma chain per output
// as k_dense_step (so a row gives the same bits alone or batched).
__global__ void __launch_bounds__(128) k_dense_apply(int64_t rows, int32_t xw, int32_t W,
                                                     const double* __restrict__ x, const double* __restrict__ w,
                                                     const double* __restrict__ bias, double* __restrict__ out) {
  extern __shared__ double xs[];  // [kRows][xw]
  for (int64_t r0 = static_cast<int64_t>(blockIdx.x) * kRows; r0 < rows;
       r0 += static_cast<int64_t>(gridDim.x) * kRows) {
    const int32_t n = static_cast<int32_t>(rows - r0 < kRows ? rows - r0 : kRows);
    __syncthreads();
    for (int32_t i = threadIdx.x; i < n * xw; i += blockDim.x) xs[i] = x[r0 * xw + i];
    __syncthreads();
    for (int32_t j = threadIdx.x; j < W; j += blockDim.x) {
      double acc[kRows];
#pragma unroll
      for (int r = 0; r < kRows; ++r) acc[r] = bias[j];
      for (int32_t i = 0; i < xw; ++i) {
        const double wij = w[static_cast<int64_t>(i) * W + j];
#pragma unroll
        for (int r = 0; r < kRows; ++r) acc[r] = __fma_rn(xs[(r < n ? r : 0) * xw + i], wij, acc[r]);
      }
      for (int r = 0; r < n; ++r) out[(r0 + r) * W + j] = acc[r] > 0.0 ? acc[r] : 0.0;
    }
  }
}

__global__ void k_dense_roots(int64_t b, int32_t W, const int32_t* __restrict__ root_g,
                              const int32_t* __restrict__ present, const double* __restrict__ values,
                              double* __restrict__ out, int32_t* __restrict__ err) {
  const int64_t e = blockIdx.x;
  if (e >= b) return;
  const int32_t r = root_g[e];
  if (present[r] != 1) {
    if (threadIdx.x == 0) set_err(err, kErrMissing);
    return;
  }
  for (int32_t j = threadIdx.x; j < W; j += blockDim.x) out[e * W + j] = values[static_cast<int64_t>(r) * W + j];
}

}  // namespace

extern "C" int dbk_dense_step(int32_t step, int32_t width, const int32_t* step_group_begin,
                              const int32_t* group_fid, const int32_t* group_begin,
                              const int32_t* member_g, const int32_t* arity_of,
                              const int32_t* child_off, const int32_t* child_list,
                              const int32_t* example, const double* inputs, double* values,
                              int32_t* present, const double* const* weights,
                              const double* const* biases, int32_t* err, int32_t max_arity,
                              int32_t blocks, void* stream) {
  if (max_arity < 1) max_arity = 1;
  if (blocks < 1) blocks = 1;
  const size_t smem = sizeof(double) * static_cast<size_t>(kRows) * max_arity * width;
  if (smem > 227 * 1024) return static_cast<int>(cudaErrorInvalidValue);
  if (smem > 48 * 1024) {
    cudaFuncSetAttribute(k_dense_step, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
  }
  k_dense_step<<<blocks, 128, smem, static_cast<cudaStream_t>(stream)>>>(
      step, width, step_group_begin, group_fid, group_begin, member_g, arity_of, child_off,
      child_list, example, inputs, values, present, weights, biases,
      err);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_dense_gather_roots(int64_t b, int32_t width, const int32_t* root_g,
                                      const int32_t* present, const double* values,
                                      double* out, int32_t* err, void* stream) {
  if (b <= 0) return 0;
  k_dense_roots<<<static_cast<unsigned>(b), 128, 0, static_cast<cudaStream_t>(stream)>>>(
      b, width, root_g, present, values, out, err);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_dense_apply(int64_t rows, int32_t arity, int32_t width, const double* x, const double* w,
                               const double* bias, double* out, void* stream) {
  if (rows <= 0) return 0;
  const int32_t xw = arity * width;
  const size_t smem = sizeof(double) * kRows * static_cast<size_t>(xw);
  if (smem > 227 * 1024) return static_cast<int>(cudaErrorInvalidValue);
  cudaFuncSetAttribute(k_dense_apply, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  const int64_t tiles = (rows + kRows - 1) / kRows;
  const unsigned blocks = static_cast<unsigned>(tiles < 148 * 8 ? tiles : 148 * 8);
  k_dense_apply<<<blocks, 128, smem, static_cast<cudaStream_t>(stream)>>>(rows, xw, width, x, w, bias, out);
  return static_cast<int>(cudaGetLastError());
}
