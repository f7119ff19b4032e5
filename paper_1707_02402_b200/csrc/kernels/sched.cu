// sched.cu — device scheduler: level labels + stable (level, function) bucket
// sort → device-side call-group index lists.
//
// Replaces, bit-for-bit, max_root_distance_labels (src/program.cpp:239-272)
// and schedule_improved + make_step (src/schedule.cpp:66-79, 135-164): the
// reference pools nodes by label, emits pools deepest first, and within a
// pool sorts by (function id, example, node). Nodes are numbered in CSR order
// (example-major, node-minor), so a STABLE sort by
//     key = (d_max - label) * p + fid
// reproduces that order exactly. Stability comes from scan-based ranks, not
// atomics: every warp owns a 256-node segment, per-(key, segment) counts are
// exclusive-scanned key-major, and each warp then walks its segment in order
// assigning ranks with __match_any_sync.
#include <algorithm>
#include <cuda_runtime.h>
#include <stdint.h>

#include "dynbatch/dbk.h"

namespace {

constexpr int kSeg = 256;        // items per warp segment (8 rounds of 32)
constexpr int kScanChunk = 4096; // table entries per block of the multi-block scan
constexpr int kWarpsPerBlock = 8;

// One thread per program: Kahn's algorithm from the root with the queue and
// in-degree counters in the program's own slice of `scratch`.
__global__ void k_labels(int64_t b, const int32_t* __restrict__ prog_off,
                         const int32_t* __restrict__ child_off,
                         const int32_t* __restrict__ child_list,
                         const int32_t* __restrict__ root_g, int32_t* __restrict__ labels,
                         int32_t* __restrict__ indeg, int32_t* __restrict__ queue,
                         int32_t* __restrict__ scal) {
  const int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  int local_max = 0;
  constexpr int kSmall = 32;  // programs up to this size run in thread-local (L1) arrays
  if (e < b && prog_off[e + 1] - prog_off[e] <= kSmall) {
    const int32_t base = prog_off[e], n = prog_off[e + 1] - base;
    int32_t deg[kSmall], lab[kSmall], q[kSmall];
    for (int32_t v = 0; v < n; ++v) deg[v] = lab[v] = 0;
    for (int32_t v = 0; v < n; ++v)
      for (int32_t c = __ldg(child_off + base + v); c < __ldg(child_off + base + v + 1); ++c)
        ++deg[__ldg(child_list + c) - base];
    int32_t head = 0, tail = 0;
    q[tail++] = __ldg(root_g + e) - base;
    while (head < tail) {
      const int32_t v = q[head++];
      const int32_t next = lab[v] + 1;
      for (int32_t c = __ldg(child_off + base + v); c < __ldg(child_off + base + v + 1); ++c) {
        const int32_t u = __ldg(child_list + c) - base;
        if (lab[u] < next) lab[u] = next;
        if (--deg[u] == 0) q[tail++] = u;
      }
    }
    if (head != n) atomicOr(&scal[1], 1);
    for (int32_t v = 0; v < n; ++v) {
      labels[base + v] = lab[v];
      local_max = max(local_max, lab[v]);
    }
  } else if (e < b) {
    const int32_t base = prog_off[e], end = prog_off[e + 1];
    for (int32_t g = base; g < end; ++g) {
      indeg[g] = 0;
      labels[g] = 0;
    }
    for (int32_t g = base; g < end; ++g)
      for (int32_t c = child_off[g]; c < child_off[g + 1]; ++c) ++indeg[child_list[c]];
    int32_t head = base, tail = base;
    queue[tail++] = root_g[e];
    while (head < tail) {
      const int32_t v = queue[head++];
      const int32_t next = labels[v] + 1;
      for (int32_t c = child_off[v]; c < child_off[v + 1]; ++c) {
        const int32_t u = child_list[c];
        if (labels[u] < next) labels[u] = next;
        if (--indeg[u] == 0) queue[tail++] = u;
      }
    }
    if (head != end) atomicOr(&scal[1], 1);
    for (int32_t g = base; g < end; ++g) local_max = max(local_max, labels[g]);
  }
  for (int o = 16; o > 0; o >>= 1) local_max = max(local_max, __shfl_xor_sync(0xffffffffu, local_max, o));
  if ((threadIdx.x & 31) == 0 && local_max > 0) atomicMax(&scal[0], local_max);
}

// schedule_standard's column of a node (src/schedule.cpp:107-133): its
// position in postorder_flatten (src/program.cpp:274-303) — depth-first from
// the root, children in operand order, a node emitted once after all its
// children. One thread per program; the DFS stack (node, next child edge)
// lives in the program's slices of the two scratch arrays. A cycle (stack
// deeper than the program) or an unreachable node sets the error flag.
__global__ void k_labels_postorder(int64_t b, const int32_t* __restrict__ prog_off,
                                   const int32_t* __restrict__ child_off, const int32_t* __restrict__ child_list,
                                   const int32_t* __restrict__ root_g, int32_t* __restrict__ labels,
                                   int32_t* __restrict__ st_node, int32_t* __restrict__ st_next,
                                   int32_t* __restrict__ scal) {
  const int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  int local_max = 0;
  if (e < b) {
    const int32_t base = prog_off[e], n = prog_off[e + 1] - base;
    for (int32_t g = base; g < base + n; ++g) labels[g] = -1;
    int32_t depth = 1, pos = 0;
    bool bad = false;
    st_node[base] = root_g[e];
    st_next[base] = child_off[root_g[e]];
    while (depth > 0) {
      const int32_t v = st_node[base + depth - 1], nx = st_next[base + depth - 1];
      if (nx < child_off[v + 1]) {
        st_next[base + depth - 1] = nx + 1;
        const int32_t c = child_list[nx];
        if (labels[c] < 0) {
          if (depth == n) {
            bad = true;
            break;
          }
          st_node[base + depth] = c;
          st_next[base + depth] = child_off[c];
          ++depth;
        }
      } else {
        labels[v] = pos++;
        --depth;
      }
    }
    if (bad || pos != n) atomicOr(&scal[1], 1);
    local_max = pos - 1;
  }
  for (int o = 16; o > 0; o >>= 1) local_max = max(local_max, __shfl_xor_sync(0xffffffffu, local_max, o));
  if ((threadIdx.x & 31) == 0 && local_max > 0) atomicMax(&scal[0], local_max);
}

// schedule_online_full's round of a node (src/schedule.cpp:171-241): a node
// is ready once all its children ran, so it runs in round = its height
// (0 for a leaf, else 1 + the largest child height). Kahn's order from the
// root (parents first), then heights over that order reversed.
__global__ void k_labels_height(int64_t b, const int32_t* __restrict__ prog_off,
                                const int32_t* __restrict__ child_off, const int32_t* __restrict__ child_list,
                                const int32_t* __restrict__ root_g, int32_t* __restrict__ labels,
                                int32_t* __restrict__ indeg, int32_t* __restrict__ queue,
                                int32_t* __restrict__ scal) {
  const int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  int local_max = 0;
  if (e < b) {
    const int32_t base = prog_off[e], end = prog_off[e + 1];
    for (int32_t g = base; g < end; ++g) indeg[g] = 0;
    for (int32_t g = base; g < end; ++g)
      for (int32_t c = child_off[g]; c < child_off[g + 1]; ++c) ++indeg[child_list[c]];
    int32_t head = base, tail = base;
    queue[tail++] = root_g[e];
    while (head < tail) {
      const int32_t v = queue[head++];
      for (int32_t c = child_off[v]; c < child_off[v + 1]; ++c)
        if (--indeg[child_list[c]] == 0) queue[tail++] = child_list[c];
    }
    if (head != end) atomicOr(&scal[1], 1);
    for (int32_t i = tail - 1; i >= base; --i) {
      const int32_t v = queue[i];
      int32_t h = 0;
      for (int32_t c = child_off[v]; c < child_off[v + 1]; ++c) h = max(h, labels[child_list[c]] + 1);
      labels[v] = h;
      local_max = max(local_max, h);
    }
  }
  for (int o = 16; o > 0; o >>= 1) local_max = max(local_max, __shfl_xor_sync(0xffffffffu, local_max, o));
  if ((threadIdx.x & 31) == 0 && local_max > 0) atomicMax(&scal[0], local_max);
}

// Step of node i: improved runs labels from d_max down (descending);
// standard / online labels are the step itself (ascending).
struct LevelKey {
  const int32_t* fid;
  const int32_t* labels;
  const int32_t* scal;
  int32_t p;
  int32_t ascending;
  __device__ __forceinline__ int32_t operator()(int64_t i) const {
    return (ascending ? labels[i] : scal[0] - labels[i]) * p + fid[i];
  }
};

struct ExplicitKey {
  const int32_t* keys;
  __device__ __forceinline__ int32_t operator()(int64_t i) const { return keys[i]; }
};

// Per-(key, segment) counts into hist[key * nseg + seg] (pre-zeroed).
template <class Key, int SEG = kSeg>
__global__ void k_seg_hist(int64_t n, int32_t nseg, Key key, int32_t* __restrict__ hist) {
  const int lane = threadIdx.x & 31;
  const int32_t seg = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  if (seg >= nseg) return;
  const int64_t begin = static_cast<int64_t>(seg) * SEG;
#pragma unroll
  for (int it = 0; it < SEG / 32; ++it) {
    const int64_t i = begin + it * 32 + lane;
    const int32_t k = i < n ? key(i) : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, k);
    if (k >= 0 && lane == __ffs(peers) - 1) hist[static_cast<int64_t>(k) * nseg + seg] += __popc(peers);
  }
}

// Block-wide exclusive scan of one value per thread; *total = block sum.
__device__ __forceinline__ int32_t block_scan_excl(int32_t v, int32_t* total, int32_t* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int32_t x = v;
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int32_t w = lane < nw ? sh[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    sh[lane] = w;
  }
  __syncthreads();
  const int32_t excl = (warp > 0 ? sh[warp - 1] : 0) + x - v;
  *total = sh[nw - 1];
  __syncthreads();
  return excl;
}

__device__ __forceinline__ int64_t table_len(int32_t nseg, int32_t p, const int32_t* scal,
                                             int32_t fixed_keys) {
  const int32_t n_keys = fixed_keys > 0 ? fixed_keys : (scal[0] + 1) * p;
  return static_cast<int64_t>(n_keys) * nseg;
}

// Multi-block exclusive scan of hist[0 .. len): (1) each block scans its
// kScanChunk entries in place and records its total, (2) one block scans the
// totals, (3) each block adds its carry-in.
__global__ void __launch_bounds__(1024) k_scan_partial(int32_t nseg, int32_t p, const int32_t* __restrict__ scal,
                                                       int32_t fixed_keys, int32_t* __restrict__ hist,
                                                       int32_t* __restrict__ totals) {
  __shared__ int32_t sh[32];
  const int64_t len = table_len(nseg, p, scal, fixed_keys);
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanChunk;
  if (base >= len) return;
  int32_t v[4], sum = 0;
  const int64_t i0 = base + threadIdx.x * 4;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    v[j] = i0 + j < len ? hist[i0 + j] : 0;
    sum += v[j];
  }
  int32_t total;
  int32_t run = block_scan_excl(sum, &total, sh);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (i0 + j < len) hist[i0 + j] = run;
    run += v[j];
  }
  if (threadIdx.x == 0) totals[blockIdx.x] = total;
}

// Small tables: the whole exclusive scan in one block, 4096 entries per
// round with a carry (replaces the three-kernel scan).
constexpr int64_t kSmallScan = 65536;
__global__ void __launch_bounds__(1024) k_scan_single(int32_t nseg, int32_t p, const int32_t* __restrict__ scal,
                                                      int32_t fixed_keys, int32_t* __restrict__ hist) {
  __shared__ int32_t sh[32];
  const int64_t len = table_len(nseg, p, scal, fixed_keys);
  int32_t carry = 0;
  for (int64_t base = 0; base < len; base += kScanChunk) {
    int32_t v[4], sum = 0;
    const int64_t i0 = base + threadIdx.x * 4;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      v[j] = i0 + j < len ? hist[i0 + j] : 0;
      sum += v[j];
    }
    int32_t total;
    int32_t run = carry + block_scan_excl(sum, &total, sh);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (i0 + j < len) hist[i0 + j] = run;
      run += v[j];
    }
    carry += total;
  }
}

__global__ void __launch_bounds__(1024) k_scan_totals(int32_t nseg, int32_t p, const int32_t* __restrict__ scal,
                                                      int32_t fixed_keys, int32_t* __restrict__ totals) {
  __shared__ int32_t sh[32];
  const int64_t len = table_len(nseg, p, scal, fixed_keys);
  const int32_t nblk = static_cast<int32_t>((len + kScanChunk - 1) / kScanChunk);
  int32_t carry = 0;
  for (int32_t b0 = 0; b0 < nblk; b0 += blockDim.x) {
    const int32_t i = b0 + threadIdx.x;
    const int32_t v = i < nblk ? totals[i] : 0;
    int32_t total;
    const int32_t e = block_scan_excl(v, &total, sh);
    if (i < nblk) totals[i] = carry + e;
    carry += total;
  }
}

__global__ void __launch_bounds__(1024) k_scan_add(int32_t nseg, int32_t p, const int32_t* __restrict__ scal,
                                                   int32_t fixed_keys, int32_t* __restrict__ hist,
                                                   const int32_t* __restrict__ totals) {
  const int64_t len = table_len(nseg, p, scal, fixed_keys);
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanChunk;
  if (base >= len || blockIdx.x == 0) return;
  const int32_t add = totals[blockIdx.x];
  for (int64_t i = base + threadIdx.x; i < base + kScanChunk && i < len; i += blockDim.x) hist[i] += add;
}

// Single-block exclusive scan over hist[0 .. n_keys*nseg) (key-major), then
// the group table: one group per non-empty key, in key order.
__global__ void k_scan_groups(int64_t n, int32_t nseg, int32_t p, int32_t* __restrict__ hist,
                              int32_t* __restrict__ scal, int32_t fixed_keys,
                              int32_t* __restrict__ group_fid, int32_t* __restrict__ group_begin,
                              int32_t* __restrict__ step_group_begin,
                              int32_t* __restrict__ offsets, int32_t steps_cap = 0) {
  __shared__ int32_t warp_tot[32];
  __shared__ int32_t carry_s;
  const int32_t n_keys = fixed_keys > 0 ? fixed_keys : (scal[0] + 1) * p;
  const int64_t total = static_cast<int64_t>(n_keys) * nseg;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nthreads = blockDim.x;
  if (tid == 0) carry_s = 0;
  __syncthreads();
  (void)total;  // the table was scanned by k_scan_partial / k_scan_totals / k_scan_add
  // Pass 2: key k's bucket is [hist[k*nseg], hist[(k+1)*nseg]) (n at the end).
  if (offsets) {  // generic sort: bucket starts only
    for (int32_t k = tid; k <= n_keys; k += nthreads)
      offsets[k] = k < n_keys ? hist[static_cast<int64_t>(k) * nseg] : static_cast<int32_t>(n);
    return;
  }
  // Group numbering: exclusive scan of (bucket non-empty) over keys.
  if (tid == 0) carry_s = 0;
  __syncthreads();
  for (int32_t base = 0; base < n_keys; base += nthreads) {
    const int32_t k = base + tid;
    int32_t start = 0, end = 0, flag = 0;
    if (k < n_keys) {
      start = hist[static_cast<int64_t>(k) * nseg];
      end = k + 1 < n_keys ? hist[static_cast<int64_t>(k + 1) * nseg] : static_cast<int32_t>(n);
      flag = end > start;
    }
    int32_t x = flag;
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int32_t w = lane < (nthreads >> 5) ? warp_tot[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      warp_tot[lane] = w;
    }
    __syncthreads();
    const int32_t gidx = carry_s + (warp > 0 ? warp_tot[warp - 1] : 0) + x - flag;
    if (k < n_keys) {
      if (flag) {
        group_fid[gidx] = k % p;
        group_begin[gidx] = start;
      }
      if (k % p == 0) step_group_begin[k / p] = gidx;
    }
    __syncthreads();
    if (tid == nthreads - 1) carry_s = gidx + flag;
    __syncthreads();
  }
  if (tid == 0) {
    const int32_t G = carry_s;
    group_begin[G] = static_cast<int32_t>(n);
    // steps [d_max + 1, steps_cap] are empty (the host may launch per-step
    // work for an upper bound of the step count without reading d_max)
    for (int32_t st = n_keys / p; st <= max(steps_cap, n_keys / p); ++st) step_group_begin[st] = G;
    scal[2] = G;
  }
}

// Stable scatter: each warp walks its segment in order; the lowest lane of
// each equal-key peer set claims popc(peers) slots from the (key, segment)
// cursor, which no other warp touches.
template <class Key, int SEG = kSeg>
__global__ void k_seg_scatter(int64_t n, int32_t nseg, Key key, int32_t* __restrict__ hist,
                              int32_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int32_t seg = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  if (seg >= nseg) return;
  const int64_t begin = static_cast<int64_t>(seg) * SEG;
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int it = 0; it < SEG / 32; ++it) {
    const int64_t i = begin + it * 32 + lane;
    const int32_t k = i < n ? key(i) : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, k);
    const int leader = __ffs(peers) - 1;
    int32_t base = 0;
    if (k >= 0 && lane == leader) {
      int32_t* cur = hist + static_cast<int64_t>(k) * nseg + seg;
      base = *cur;
      *cur = base + __popc(peers);
    }
    base = __shfl_sync(0xffffffffu, base, leader);
    if (k >= 0) out[base + __popc(peers & lt)] = static_cast<int32_t>(i);
  }
}

inline int32_t n_segments(int64_t n, int seg = kSeg) { return static_cast<int32_t>((n + seg - 1) / seg); }

// Generic stable sort segment: short segments (more warps in flight) when
// the (key, segment) table stays small.
constexpr int kSegSmall = 64;
constexpr int64_t kSmallSortItems = 16384;  // scheduler sorts up to this many nodes use kSegSmall
inline int generic_seg(int32_t n_keys) { return n_keys <= 128 ? kSegSmall : kSeg; }

}  // namespace

extern "C" int dbk_sched_labels(int64_t b, int64_t N, const int32_t* prog_off,
                                const int32_t* child_off, const int32_t* child_list,
                                const int32_t* root_g, int32_t* labels, int32_t* scratch,
                                int32_t* dev_scalars, int32_t strategy, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (b <= 0) return 0;
  const int threads = 128;
  const int blocks = static_cast<int>((b + threads - 1) / threads);
  // scratch = indeg[N] | queue[N] (standard: DFS stack nodes | next edges)
  switch (strategy) {
    case 1:  // standard
      k_labels_postorder<<<blocks, threads, 0, s>>>(b, prog_off, child_off, child_list, root_g, labels, scratch,
                                                    scratch + N, dev_scalars);
      break;
    case 3:  // online
      k_labels_height<<<blocks, threads, 0, s>>>(b, prog_off, child_off, child_list, root_g, labels, scratch,
                                                 scratch + N, dev_scalars);
      break;
    case 2:  // improved
      k_labels<<<blocks, threads, 0, s>>>(b, prog_off, child_off, child_list, root_g, labels, scratch,
                                          scratch + N, dev_scalars);
      break;
    default:
      return static_cast<int>(cudaErrorInvalidValue);
  }
  return static_cast<int>(cudaGetLastError());
}

// Static schedule labels: every program has the same tree shape (e.g. the
// balanced-tree workload), so node g's label is the shape's table entry
// table[g − prog_off[example]]; d_max is known, no traversal is needed.
__global__ void k_labels_static(int64_t N, int32_t n, const int32_t* __restrict__ table, int32_t dmax,
                                int32_t* __restrict__ labels, int32_t* __restrict__ dev_scalars) {
  const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (g == 0) {
    dev_scalars[0] = dmax;
    dev_scalars[1] = 0;
  }
  if (g < N) labels[g] = table[g % n];
}

extern "C" int dbk_sched_labels_static(int64_t N, int32_t n, const int32_t* table, int32_t dmax, int32_t* labels,
                                       int32_t* dev_scalars, void* stream) {
  if (N <= 0) return 0;
  k_labels_static<<<static_cast<unsigned>((N + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      N, n, table, dmax, labels, dev_scalars);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_sched_bucket_sort(int64_t N, int32_t p, int32_t max_keys, const int32_t* fid,
                                     const int32_t* labels, int32_t* dev_scalars,
                                     int32_t* seg_hist, int32_t* member_g, int32_t* group_fid,
                                     int32_t* group_begin, int32_t* step_group_begin, int32_t steps_cap,
                                     int32_t ascending, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // short segments for small batches (more warps in flight on a latency-bound
  // sort); the table stays small either way
  const int seg = N <= kSmallSortItems ? kSegSmall : kSeg;
  const int32_t nseg = n_segments(N, seg);
  cudaMemsetAsync(seg_hist, 0, sizeof(int32_t) * static_cast<size_t>(max_keys) * (nseg > 0 ? nseg : 1), s);
  LevelKey key{fid, labels, dev_scalars, p, ascending};
  const int blocks = (nseg + kWarpsPerBlock - 1) / kWarpsPerBlock;
  if (nseg > 0) {
    if (seg == kSegSmall) k_seg_hist<LevelKey, kSegSmall><<<blocks, kWarpsPerBlock * 32, 0, s>>>(N, nseg, key, seg_hist);
    else k_seg_hist<LevelKey, kSeg><<<blocks, kWarpsPerBlock * 32, 0, s>>>(N, nseg, key, seg_hist);
  }
  const int32_t ns = nseg > 0 ? nseg : 1;
  int32_t* totals = seg_hist + static_cast<int64_t>(max_keys) * ns;
  const unsigned sblk = static_cast<unsigned>((static_cast<int64_t>(max_keys) * ns + kScanChunk - 1) / kScanChunk);
  if (static_cast<int64_t>(max_keys) * ns <= kSmallScan) {
    k_scan_single<<<1, 1024, 0, s>>>(ns, p, dev_scalars, 0, seg_hist);
  } else {
    k_scan_partial<<<sblk, 1024, 0, s>>>(ns, p, dev_scalars, 0, seg_hist, totals);
    k_scan_totals<<<1, 1024, 0, s>>>(ns, p, dev_scalars, 0, totals);
    k_scan_add<<<sblk, 1024, 0, s>>>(ns, p, dev_scalars, 0, seg_hist, totals);
  }
  k_scan_groups<<<1, 1024, 0, s>>>(N, ns, p, seg_hist, dev_scalars, 0, group_fid,
                                   group_begin, step_group_begin, nullptr, steps_cap);
  if (nseg > 0) {
    if (seg == kSegSmall)
      k_seg_scatter<LevelKey, kSegSmall><<<blocks, kWarpsPerBlock * 32, 0, s>>>(N, nseg, key, seg_hist, member_g);
    else
      k_seg_scatter<LevelKey, kSeg><<<blocks, kWarpsPerBlock * 32, 0, s>>>(N, nseg, key, seg_hist, member_g);
  }
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_stable_bucket_sort(int64_t n_items, int32_t n_keys, const int32_t* keys,
                                      int32_t* seg_hist, int32_t* order, int32_t* offsets,
                                      void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int seg = generic_seg(n_keys);
  const int32_t nseg = n_segments(n_items, seg) > 0 ? n_segments(n_items, seg) : 1;
  cudaMemsetAsync(seg_hist, 0, sizeof(int32_t) * static_cast<size_t>(n_keys) * nseg, s);
  ExplicitKey key{keys};
  const int blocks = (nseg + kWarpsPerBlock - 1) / kWarpsPerBlock;
  if (seg == kSegSmall)
    k_seg_hist<ExplicitKey, kSegSmall><<<blocks, kWarpsPerBlock * 32, 0, s>>>(n_items, nseg, key, seg_hist);
  else
    k_seg_hist<ExplicitKey, kSeg><<<blocks, kWarpsPerBlock * 32, 0, s>>>(n_items, nseg, key, seg_hist);
  int32_t* totals = seg_hist + static_cast<int64_t>(n_keys) * nseg;
  const unsigned sblk = static_cast<unsigned>((static_cast<int64_t>(n_keys) * nseg + kScanChunk - 1) / kScanChunk);
  if (static_cast<int64_t>(n_keys) * nseg <= kSmallScan) {
    k_scan_single<<<1, 1024, 0, s>>>(nseg, 1, nullptr, n_keys, seg_hist);
  } else {
    k_scan_partial<<<sblk, 1024, 0, s>>>(nseg, 1, nullptr, n_keys, seg_hist, totals);
    k_scan_totals<<<1, 1024, 0, s>>>(nseg, 1, nullptr, n_keys, totals);
    k_scan_add<<<sblk, 1024, 0, s>>>(nseg, 1, nullptr, n_keys, seg_hist, totals);
  }
  k_scan_groups<<<1, 1024, 0, s>>>(n_items, nseg, 1, seg_hist, nullptr, n_keys, nullptr, nullptr,
                                   nullptr, offsets);
  if (seg == kSegSmall)
    k_seg_scatter<ExplicitKey, kSegSmall><<<blocks, kWarpsPerBlock * 32, 0, s>>>(n_items, nseg, key, seg_hist, order);
  else
    k_seg_scatter<ExplicitKey, kSeg><<<blocks, kWarpsPerBlock * 32, 0, s>>>(n_items, nseg, key, seg_hist, order);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int64_t dbk_bucket_sort_scratch(int64_t n_items, int32_t max_keys) {
  // enough for every segment size a sort of up to n_items may use: the
  // scheduler's (kSegSmall up to kSmallSortItems nodes, else kSeg) and the
  // generic sort's (generic_seg(max_keys))
  auto table = [&](int64_t n, int seg) { return static_cast<int64_t>(max_keys) * (n > 0 ? (n + seg - 1) / seg : 1); };
  int64_t t = table(n_items, kSeg);
  t = std::max(t, table(std::min<int64_t>(n_items, kSmallSortItems), kSegSmall));
  if (generic_seg(max_keys) == kSegSmall) t = std::max(t, table(n_items, kSegSmall));
  return t + t / kScanChunk + 64;
}

// ------------------------------------------- program build from prefixes
// build_program_from_prefix (src/program.cpp:95-142) for a batch of
// concatenated prefix function sequences, one thread per program: the
// reference's explicit stack of (node, remaining arity), kept in the
// per-program slice of `stack` (≤ one entry per node). Writes the CSR the
// device scheduler and executors read, with node ids in sequence order
// (root = position 0). A tree of n nodes has n − 1 child edges, so program
// e's child list starts at seq_off[e] − e. fwd_ok[g] = expensive node with
// exactly one parent (every non-root node of a tree). Errors (first wins,
// Errc codes): 1 empty sequence, 2 unknown function, 3 underfull, 4 overfull.
__global__ void k_build_prefix(int64_t b, const int32_t* __restrict__ tokens, const int32_t* __restrict__ seq_off,
                               int32_t p, const int32_t* __restrict__ arity_of, int32_t* __restrict__ prog_off,
                               int32_t* __restrict__ fid, int32_t* __restrict__ child_off,
                               int32_t* __restrict__ child_list, int32_t* __restrict__ child0,
                               int32_t* __restrict__ child1, int32_t* __restrict__ example,
                               int32_t* __restrict__ root_g, int32_t* __restrict__ fwd_ok,
                               int2* __restrict__ stack, int32_t* __restrict__ err) {
  const int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (e >= b) return;
  const int32_t off = seq_off[e], n = seq_off[e + 1] - off;
  prog_off[e] = off;
  if (e == b - 1) {
    prog_off[b] = seq_off[b];
    child_off[seq_off[b]] = seq_off[b] - static_cast<int32_t>(b);
  }
  root_g[e] = off;
  if (n <= 0) {
    atomicCAS(err, 0, 1);
    return;
  }
  int2* st = stack + off;
  int32_t top = 0, cursor = off - static_cast<int32_t>(e);  // next free child-list slot
  for (int32_t i = 0; i < n; ++i) {
    const int32_t g = off + i;
    if (i > 0 && top == 0) {  // tokens remain after the root closed (checked first, as the reference)
      atomicCAS(err, 0, 4);
      return;
    }
    const int32_t f = tokens[g];
    if (f < 0 || f >= p) {
      atomicCAS(err, 0, 2);
      return;
    }
    const int32_t a = arity_of[f];
    fid[g] = f;
    example[g] = static_cast<int32_t>(e);
    child0[g] = -1;
    child1[g] = -1;
    child_off[g] = cursor;
    cursor += a;
    fwd_ok[g] = a > 0 && i > 0;
    if (i > 0) {
      int2& parent = st[top - 1];  // (node, children already attached)
      const int32_t k = parent.y++;
      child_list[child_off[parent.x] + k] = g;
      if (k == 0) child0[parent.x] = g;
      if (k == 1) child1[parent.x] = g;
      if (parent.y == arity_of[fid[parent.x]]) --top;
    }
    if (a > 0) st[top++] = make_int2(g, 0);
  }
  if (top != 0) atomicCAS(err, 0, 3);  // the sequence ends with unfilled arities
}

extern "C" int dbk_build_prefix(int64_t b, const int32_t* tokens, const int32_t* seq_off, int32_t p,
                                const int32_t* arity_of, int32_t* prog_off, int32_t* fid, int32_t* child_off,
                                int32_t* child_list, int32_t* child0, int32_t* child1, int32_t* example,
                                int32_t* root_g, int32_t* fwd_ok, void* stack, int32_t* err, void* stream) {
  if (b <= 0) return 0;
  k_build_prefix<<<static_cast<unsigned>((b + 127) / 128), 128, 0, static_cast<cudaStream_t>(stream)>>>(
      b, tokens, seq_off, p, arity_of, prog_off, fid, child_off, child_list, child0, child1, example, root_g,
      fwd_ok, static_cast<int2*>(stack), err);
  return static_cast<int>(cudaGetLastError());
}
