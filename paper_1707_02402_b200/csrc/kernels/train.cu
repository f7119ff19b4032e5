// train.cu — the IEP training step's data movement (the
// reference stops at the forward). The backward runs group by
// group in reverse step order (iep_train.cpp); its contractions are library
// GEMMs (cuBLAS, TF32 tensor cores), these kernels move and mask operands.
//
// Per-member tensors use the "padded image" layout PI: 257 rows × channels,
// fp32: 16 zero guard rows, the 225 positions of the packed 15×15 grid (row
// 14 and column 14 are pads, kept zero), 16 zero guard rows. A 3×3 tap is the
// row shift 15·dh + dw, as in the forward's staging, and every shifted read
// of a member stays inside its own PI.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "dynbatch/dbk.h"

namespace {

constexpr int kC = 128, kImg = 225, kPx = 196, kGuard = 32, kPI = 257, kPIG = 16;
constexpr int kFmap = 16 * kPx * 8;

__device__ __forceinline__ bool is_pad(int p) { return p / 15 == 14 || p % 15 == 14; }
__device__ __forceinline__ int px_of(int p) { return (p / 15) * 14 + p % 15; }  // real pixels only
__device__ __forceinline__ int shift_of(int tap) { return (tap / 3 - 1) * 15 + (tap % 3 - 1); }

// Staging byte offset of plane j (16 bytes: 8 channels) of row r.
__device__ __forceinline__ int64_t stage_off(int64_t ps, int j, int64_t r) {
  return ((static_cast<int64_t>(j >> 3) * ps + r) << 7) + (((j & 7) ^ static_cast<int>(r & 7)) << 4);
}

unsigned grid_for(int64_t n, int per_block = 256) {
  return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((n + per_block - 1) / per_block, 148 * 32)));
}

// fp16 staging (hi, + lo when given) of n member images (image k at staging
// position rows[k]) → fp32 PI [n][257][planes·8]; pads 0.
__global__ void k_stage_to_pi(int32_t n, const int64_t* __restrict__ rows, const uint8_t* __restrict__ hi,
                              const uint8_t* __restrict__ lo, int64_t ps, int32_t plane0, int32_t planes,
                              float* __restrict__ out) {
  const int64_t total = static_cast<int64_t>(n) * kImg * planes;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int j = static_cast<int>(i % planes);
    const int64_t kp = i / planes;
    const int32_t k = static_cast<int32_t>(kp / kImg);
    const int p = static_cast<int>(kp % kImg);
    float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (!is_pad(p)) {
      const int64_t r = kGuard + rows[k] + p;
      const uint4 h = *reinterpret_cast<const uint4*>(hi + stage_off(ps, plane0 + j, r));
      const __half2* h2 = reinterpret_cast<const __half2*>(&h);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 f = __half22float2(h2[q]);
        v[2 * q] = f.x;
        v[2 * q + 1] = f.y;
      }
      if (lo) {
        const uint4 l = *reinterpret_cast<const uint4*>(lo + stage_off(ps, plane0 + j, r));
        const __half2* l2 = reinterpret_cast<const __half2*>(&l);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 f = __half22float2(l2[q]);
          v[2 * q] += f.x;
          v[2 * q + 1] += f.y;
        }
      }
    }
    float4* o = reinterpret_cast<float4*>(out + (static_cast<int64_t>(k) * kPI + kPIG + p) * (planes * 8) + j * 8);
    o[0] = make_float4(v[0], v[1], v[2], v[3]);
    o[1] = make_float4(v[4], v[5], v[6], v[7]);
  }
}

// DA2 = dY ⊙ (y > 0) for the group's members: dY from the node-indexed PI
// buffer, y from the node's fp32 plane map; every PI row is written (pads
// and guard rows 0: shifted reads of the data gradient and the weight
// gradients' K range cover them).
__global__ void k_da_out(int32_t n, const int32_t* __restrict__ nodes, const float* __restrict__ dy_nodes,
                         const float* __restrict__ values, float* __restrict__ out, uint32_t* __restrict__ absmax) {
  float mx = 0.f;
  const int64_t total = static_cast<int64_t>(n) * kPI * 16;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int j = static_cast<int>(i % 16);
    const int64_t kp = i / 16;
    const int32_t k = static_cast<int32_t>(kp / kPI);
    const int p = static_cast<int>(kp % kPI) - kPIG;  // position, or a guard row outside [0, 225)
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
    if (p >= 0 && p < kImg && !is_pad(p)) {
      const int32_t v = nodes[k];
      const int64_t prow = (static_cast<int64_t>(v) * kPI + kPIG + p) * kC + j * 8;
      const float4* d = reinterpret_cast<const float4*>(dy_nodes + prow);
      const float4* y = reinterpret_cast<const float4*>(values + static_cast<int64_t>(v) * kFmap +
                                                        (static_cast<int64_t>(j) * kPx + px_of(p)) * 8);
      const float4 d0 = d[0], d1 = d[1], y0 = y[0], y1 = y[1];
      a = make_float4(y0.x > 0.f ? d0.x : 0.f, y0.y > 0.f ? d0.y : 0.f, y0.z > 0.f ? d0.z : 0.f, y0.w > 0.f ? d0.w : 0.f);
      b = make_float4(y1.x > 0.f ? d1.x : 0.f, y1.y > 0.f ? d1.y : 0.f, y1.z > 0.f ? d1.z : 0.f, y1.w > 0.f ? d1.w : 0.f);
    }
    float4* o = reinterpret_cast<float4*>(out + (static_cast<int64_t>(k) * kPI + kPIG + p) * kC + j * 8);
    o[0] = a;
    o[1] = b;
    mx = fmaxf(mx, fmaxf(fmaxf(fmaxf(fabsf(a.x), fabsf(a.y)), fmaxf(fabsf(a.z), fabsf(a.w))),
                         fmaxf(fmaxf(fabsf(b.x), fabsf(b.y)), fmaxf(fabsf(b.z), fabsf(b.w)))));
  }
  // |DA2| max for the fp16 operand scale of the implicit-GEMM gradients
  if (absmax) {
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0 && mx > 0.f) atomicMax(absmax, __float_as_uint(mx));
  }
}

// COLS[r][tap·ch + c] = X[r + shift(tap)][c] over the n members' PI rows
// (X has 16 zero rows before and after, so every shifted read is in bounds).
__global__ void k_im2col(int64_t rows, int32_t ch, const float* __restrict__ x, float* __restrict__ cols) {
  const int32_t groups = ch / 4;
  const int64_t total = rows * 9 * groups;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t g = static_cast<int32_t>(i % groups);
    const int64_t rt = i / groups;
    const int tap = static_cast<int>(rt % 9);
    const int64_t r = rt / 9;
    const float4 v = *reinterpret_cast<const float4*>(x + (r + shift_of(tap)) * ch + 4 * g);
    *reinterpret_cast<float4*>(cols + r * 9 * ch + tap * ch + 4 * g) = v;
  }
}

// OUT[k][q] = Σ_tap G[k][q − shift(tap)][tap·ch + :] (+ RES[k][q]), then
// ⊙ (MASK[k][q] > 0) when a mask is given; pads and guards 0.
__global__ void k_col2im(int32_t n, int32_t ch, const float* __restrict__ g, const float* __restrict__ res,
                         const float* __restrict__ mask, float* __restrict__ out) {
  const int32_t groups = ch / 4;
  const int64_t total = static_cast<int64_t>(n) * kPI * groups;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t c4 = static_cast<int32_t>(i % groups);
    const int64_t kr = i / groups;
    const int32_t k = static_cast<int32_t>(kr / kPI);
    const int r = static_cast<int>(kr % kPI);
    const int p = r - kPIG;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (p >= 0 && p < kImg && !is_pad(p)) {
      const int64_t base = static_cast<int64_t>(k) * kPI + r;
#pragma unroll
      for (int tap = 0; tap < 9; ++tap) {
        const float4 v = *reinterpret_cast<const float4*>(g + (base - shift_of(tap)) * 9 * ch + tap * ch + 4 * c4);
        acc.x += v.x;
        acc.y += v.y;
        acc.z += v.z;
        acc.w += v.w;
      }
      if (res) {
        const float4 v = *reinterpret_cast<const float4*>(res + base * ch + 4 * c4);
        acc.x += v.x;
        acc.y += v.y;
        acc.z += v.z;
        acc.w += v.w;
      }
      if (mask) {
        const float4 m = *reinterpret_cast<const float4*>(mask + base * ch + 4 * c4);
        acc = make_float4(m.x > 0.f ? acc.x : 0.f, m.y > 0.f ? acc.y : 0.f, m.z > 0.f ? acc.z : 0.f,
                          m.w > 0.f ? acc.w : 0.f);
      }
    }
    *reinterpret_cast<float4*>(out + (static_cast<int64_t>(k) * kPI + r) * ch + 4 * c4) = acc;
  }
}

// out = g ⊙ (act > 0), elementwise over `count` floats.
__global__ void k_mask(int64_t count, const float* __restrict__ g, const float* __restrict__ act,
                       float* __restrict__ out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = act[i] > 0.f ? g[i] : 0.f;
}

// db[c] += Σ_r a[r][c] (one block per 64-row slab, atomics per column).
__global__ void __launch_bounds__(256) k_colsum(int64_t rows, int32_t cols, const float* __restrict__ a,
                                                float* __restrict__ db) {
  for (int32_t c = threadIdx.x; c < cols; c += blockDim.x) {
    float s = 0.f;
    const int64_t r0 = static_cast<int64_t>(blockIdx.x) * 64, r1 = min(rows, r0 + 64);
    for (int64_t r = r0; r < r1; ++r) s += a[r * cols + c];
    if (s != 0.f) atomicAdd(db + c, s);
  }
}

// Segmented column sums of a 128-wide matrix: slab i covers rows
// [slab_row[2i], slab_row[2i + 1]) of one group, whose bias gradient is
// dst[i]; 128 threads per slab, one atomic per column and slab.
__global__ void __launch_bounds__(128) k_colsum_seg(const int64_t* __restrict__ slab_row, float* const* __restrict__ dst,
                                                    const float* __restrict__ a) {
  const int64_t r0 = slab_row[2 * blockIdx.x], r1 = slab_row[2 * blockIdx.x + 1];
  float s = 0.f;
  for (int64_t r = r0; r < r1; ++r) s += a[r * kC + threadIdx.x];
  if (s != 0.f) atomicAdd(dst[blockIdx.x] + threadIdx.x, s);
}

// Routes the gradient of member k's operand (PI rows of `src`, `ch` channels
// wide, channels [c0, c0 + 128)) to its child: an expensive child's
// node-indexed dY PI, or a leaf's input-map gradient (CHW rows). Atomic adds:
// children shared by several parents (DAGs) accumulate.
__global__ void k_route(int32_t n, const int32_t* __restrict__ nodes, const int32_t* __restrict__ child,
                        const int32_t* __restrict__ fid, const int32_t* __restrict__ arity_of,
                        const int32_t* __restrict__ example, const float* __restrict__ src, int32_t ch, int32_t c0,
                        float* __restrict__ dy_nodes, float* __restrict__ d_inputs) {
  // one thread per (member, position, 4 channels): a 16-byte load and one
  // vector atomic into the child's dY PI (channels contiguous); a leaf's
  // CHW input gradient takes four scalar atomics
  constexpr int kQ = kC / 4;
  const int64_t total = static_cast<int64_t>(n) * kImg * kQ;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i % kQ) * 4;
    const int64_t kp = i / kQ;
    const int32_t k = static_cast<int32_t>(kp / kImg);
    const int p = static_cast<int>(kp % kImg);
    if (is_pad(p)) continue;
    const float4 v = *reinterpret_cast<const float4*>(src + (static_cast<int64_t>(k) * kPI + kPIG + p) * ch + c0 + c);
    if (v.x == 0.f && v.y == 0.f && v.z == 0.f && v.w == 0.f) continue;
    const int32_t cn = child[nodes[k]];
    if (arity_of[fid[cn]] == 0) {
      float* d = d_inputs + static_cast<int64_t>(example[cn]) * (kC * kPx) + c * kPx + px_of(p);
      atomicAdd(d, v.x);
      atomicAdd(d + kPx, v.y);
      atomicAdd(d + 2 * kPx, v.z);
      atomicAdd(d + 3 * kPx, v.w);
    } else {
      atomicAdd(reinterpret_cast<float4*>(dy_nodes + (static_cast<int64_t>(cn) * kPI + kPIG + p) * kC + c), v);
    }
  }
}

// ---------------------------------------------------------------- head
// Softmax cross-entropy of b rows of `ld`-strided logits (A valid columns),
// one warp per row: loss[1 + e] = row loss, dlogits [b][A] = (softmax −
// onehot) / b. k_mean_loss then sums the rows in a fixed order into loss[0]
// (no atomics: the loss is bit-reproducible run to run and across schedules).
__global__ void k_softmax_ce(int64_t b, int32_t A, int32_t ld, const float* __restrict__ logits,
                             const int32_t* __restrict__ labels, float* __restrict__ dlogits, float* __restrict__ loss) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x >> 5) + (threadIdx.x >> 5); e < b; e += warps) {
    const float* z = logits + e * ld;
    float m = -INFINITY;
    for (int a = lane; a < A; a += 32) m = fmaxf(m, z[a]);
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    float s = 0.f;
    for (int a = lane; a < A; a += 32) s += __expf(z[a] - m);
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const int32_t y = labels[e];
    for (int a = lane; a < A; a += 32)
      dlogits[e * A + a] = (__expf(z[a] - m) / s - (a == y ? 1.f : 0.f)) / static_cast<float>(b);
    if (lane == 0) loss[1 + e] = logf(s) + m - z[y];
  }
}

// loss[0] = Σ_e loss[1 + e] / b: one block, contiguous per-thread chunks,
// then a fixed tree.
__global__ void __launch_bounds__(256) k_mean_loss(int64_t b, float* __restrict__ loss) {
  __shared__ float part[256];
  const int64_t per = (b + 255) / 256, lo = threadIdx.x * per, hi = min(b, lo + per);
  float s = 0.f;
  for (int64_t e = lo; e < hi; ++e) s += loss[1 + e];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w; w >>= 1) {
    if (threadIdx.x < w) part[threadIdx.x] += part[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) loss[0] = part[0] / static_cast<float>(b);
}

// Tiled SWIZZLE_NONE 16-bit operand ([row block][K/64][8][128][8], the grouped
// GEMM's H) → fp32 rows [rows][K].
__global__ void k_unpack_h(int64_t rows, int32_t K, const uint16_t* __restrict__ h, float* __restrict__ out) {
  const int32_t kc = K / 64;
  const int64_t total = rows * (K / 8);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t g = static_cast<int32_t>(i % (K / 8));
    const int64_t r = i / (K / 8);
    const int64_t off = ((r / 128) * kc + g / 8) * (128 * 64) + ((g % 8) * 128 + r % 128) * 8;
    const uint4 v = *reinterpret_cast<const uint4*>(h + off);
    const __half2* h2 = reinterpret_cast<const __half2*>(&v);
    float4* o = reinterpret_cast<float4*>(out + r * K + 8 * g);
    const float2 a = __half22float2(h2[0]), b = __half22float2(h2[1]), c = __half22float2(h2[2]),
                 d = __half22float2(h2[3]);
    o[0] = make_float4(a.x, a.y, b.x, b.y);
    o[1] = make_float4(c.x, c.y, d.x, d.y);
  }
}

// Tiled SWIZZLE_128B 16-bit operand ([row block][K/64][128 rows × 128 B]) →
// fp32 rows [rows][K].
__global__ void k_unpack_sw128(int64_t rows, int32_t K, const uint8_t* __restrict__ a, float* __restrict__ out) {
  const int32_t kc = K / 64;
  const int64_t total = rows * (K / 8);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t g = static_cast<int32_t>(i % (K / 8));
    const int64_t r = i / (K / 8);
    const int32_t rr = static_cast<int32_t>(r % 128);
    const int64_t off = ((r / 128) * kc + g / 8) * (128 * 128) + rr * 128 + (((g % 8) ^ (rr & 7)) << 4);
    const uint4 v = *reinterpret_cast<const uint4*>(a + off);
    const __half2* h2 = reinterpret_cast<const __half2*>(&v);
    float4* o = reinterpret_cast<float4*>(out + r * K + 8 * g);
    const float2 p = __half22float2(h2[0]), q = __half22float2(h2[1]), s = __half22float2(h2[2]),
                 t = __half22float2(h2[3]);
    o[0] = make_float4(p.x, p.y, q.x, q.y);
    o[1] = make_float4(s.x, s.y, t.x, t.y);
  }
}

// Max-pool backward: dproj[e·196 + px][c] = dpooled[e][q·P + c] where px is
// the first maximum of its 2×2 window in scan order (torch's choice), then
// ⊙ (proj > 0).
__global__ void k_pool_bwd(int64_t b, int32_t P, const float* __restrict__ proj, const float* __restrict__ dpooled,
                           float* __restrict__ dproj) {
  const int64_t total = b * 49 * P;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t c = static_cast<int32_t>(i % P);
    const int64_t eq = i / P;
    const int q = static_cast<int>(eq % 49);
    const int64_t e = eq / 49;
    const int ph = q / 7, pw = q % 7;
    int best = 0;
    float m = -INFINITY;
    int64_t rows[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      rows[t] = e * kPx + (2 * ph + (t >> 1)) * 14 + 2 * pw + (t & 1);
      const float v = proj[rows[t] * P + c];
      if (v > m) {
        m = v;
        best = t;
      }
    }
    const float g = dpooled[e * 49 * P + q * P + c];
#pragma unroll
    for (int t = 0; t < 4; ++t) dproj[rows[t] * P + c] = (t == best && m > 0.f) ? g : 0.f;
  }
}

// Root gradients [b·196][128] → the root nodes' dY PI (expensive roots) or
// the input-map gradient (a leaf root).
__global__ void k_droots(int64_t b, const int32_t* __restrict__ root_g, const int32_t* __restrict__ fid,
                         const int32_t* __restrict__ arity_of, const int32_t* __restrict__ example,
                         const float* __restrict__ droots, float* __restrict__ dy_nodes, float* __restrict__ d_inputs) {
  const int64_t total = b * kPx * kC;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i % kC);
    const int64_t ex = i / kC;
    const int px = static_cast<int>(ex % kPx);
    const int64_t e = ex / kPx;
    const float v = droots[i];
    const int32_t r = root_g[e];
    if (arity_of[fid[r]] == 0) {
      atomicAdd(d_inputs + static_cast<int64_t>(example[r]) * (kC * kPx) + c * kPx + px, v);
    } else {
      const int p = (px / 14) * 15 + px % 14;
      atomicAdd(dy_nodes + (static_cast<int64_t>(r) * kPI + kPIG + p) * kC + c, v);
    }
  }
}


// ------------------------------------------------------------- SGD update
// w -= lr · g over n fp32 values.
__global__ void k_sgd(int64_t n, float* __restrict__ w, const float* __restrict__ g, float lr) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    w[i] -= lr * g[i];
}

// The step kernel's fp16 weight blocks from fp32 input-major weights
// w[(tap·cin + ci)·C + co] (the device twin of iep_resblock.cpp pack_blocks):
// one 16 KB block per (64-channel K chunk, tap), output channel co = the
// 128-byte row, input channel k (mod 64) in 16-byte slot (k/8) ^ (co & 7).
__global__ void k_pack_conv_w(const float* __restrict__ w, int32_t cin, int32_t taps, uint16_t* __restrict__ out) {
  const int64_t total = static_cast<int64_t>(taps) * cin * kC;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int co = static_cast<int>(i % kC);
    const int64_t tc = i / kC;
    const int ci = static_cast<int>(tc % cin), tap = static_cast<int>(tc / cin);
    const int chunk = ci / 64, k = ci % 64;
    const int64_t base = static_cast<int64_t>(chunk * taps + tap) * 64 * kC;
    const __half h = __float2half_rn(w[(static_cast<int64_t>(tap) * cin + ci) * kC + co]);
    out[base + co * 64 + ((k / 8) ^ (co & 7)) * 8 + k % 8] = *reinterpret_cast<const uint16_t*>(&h);
  }
}

// The grouped GEMM's fp16 B tiles from fp32 input-major weights w[k][n] of K ×
// N_src, zero-padded to N columns (the device twin of moe_bf16.cpp
// tile_weights): blocks of 256 columns × 64 K, halves of 128 columns, [8 K
// groups][128 n][8 k].
__global__ void k_tile_w(const float* __restrict__ w, int32_t K, int32_t N_src, int32_t N, uint16_t* __restrict__ out) {
  const int64_t total = static_cast<int64_t>(K) * N;
  const int n_kc = K / 64;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int n = static_cast<int>(i % N);
    const int kk = static_cast<int>(i / N);
    const int kc = kk / 64, k8 = (kk % 64) / 8, ke = kk % 8;
    const int nt = n / 256, half = (n % 256) / 128, nn = n % 128;
    const int64_t blk = static_cast<int64_t>(nt) * n_kc + kc;
    const float v = n < N_src ? w[static_cast<int64_t>(kk) * N_src + n] : 0.f;
    const __half h = __float2half_rn(v);
    out[blk * 256 * 64 + ((static_cast<int64_t>(half) * 8 + k8) * 128 + nn) * 8 + ke] =
        *reinterpret_cast<const uint16_t*>(&h);
  }
}

}  // namespace

extern "C" int dbk_tr_stage_to_pi(int32_t n, const int64_t* rows, const void* hi, const void* lo, int64_t ps,
                                  int32_t plane0, int32_t planes, float* out, void* stream) {
  const int64_t total = static_cast<int64_t>(n) * kImg * planes;
  if (total <= 0) return 0;
  k_stage_to_pi<<<grid_for(total), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      n, rows, static_cast<const uint8_t*>(hi), static_cast<const uint8_t*>(lo), ps, plane0, planes, out);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_tr_colsum_seg(int32_t slabs, const int64_t* slab_row, float* const* dst, const float* a,
                                 void* stream) {
  if (slabs <= 0) return 0;
  k_colsum_seg<<<static_cast<unsigned>(slabs), kC, 0, static_cast<cudaStream_t>(stream)>>>(slab_row, dst, a);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_tr_da_out(int32_t n, const int32_t* nodes, const float* dy_nodes, const float* values,
                             float* out, uint32_t* absmax, void* stream) {
  const int64_t total = static_cast<int64_t>(n) * kPI * 16;
  if (total <= 0) return 0;
  k_da_out<<<grid_for(total), 256, 0, static_cast<cudaStream_t>(stream)>>>(n, nodes, dy_nodes, values, out, absmax);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_tr_im2col(int64_t rows, int32_t ch, const float* x, float* cols, void* stream) {
  const int64_t total = rows * 9 * (ch / 4);
  if (total <= 0) return 0;
  k_im2col<<<grid_for(total), 256, 0, static_cast<cudaStream_t>(stream)>>>(rows, ch, x, cols);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_tr_col2im(int32_t n, int32_t ch, const float* g, const float* res, const float* mask, float* out,
                             void* stream) {
  const int64_t total = static_cast<int64_t>(n) * kPI * (ch / 4);
  if (total <= 0) return 0;
  k_col2im<<<grid_for(total), 256, 0, static_cast<cudaStream_t>(stream)>>>(n, ch, g, res, mask, out);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_tr_mask(int64_t count, const float* g, const float* act, float* out, void* stream) {
  if (count <= 0) return 0;
  k_mask<<<grid_for(count), 256, 0, static_cast<cudaStream_t>(stream)>>>(count, g, act, out);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_tr_colsum(int64_t rows, int32_t cols, const float* a, float* db, void* stream) {
  if (rows <= 0) return 0;
  k_colsum<<<static_cast<unsigned>((rows + 63) / 64), 256, 0, static_cast<cudaStream_t>(stream)>>>(rows, cols, a, db);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_tr_route(int32_t n, const int32_t* nodes, const int32_t* child, const int32_t* fid,
                            const int32_t* arity_of, const int32_t* example, const float* src, int32_t ch,
                            int32_t c0, float* dy_nodes, float* d_inputs, void* stream) {
  const int64_t total = static_cast<int64_t>(n) * kImg * kC;
  if (total <= 0) return 0;
  k_route<<<grid_for(total / 4), 256, 0, static_cast<cudaStream_t>(stream)>>>(n, nodes, child, fid, arity_of, example,
                                                                         src, ch, c0, dy_nodes, d_inputs);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_tr_softmax_ce(int64_t b, int32_t A, int32_t ld, const float* logits, const int32_t* labels,
                                 float* dlogits, float* loss, void* stream) {
  if (b <= 0) return 0;
  k_softmax_ce<<<grid_for(b * 32), 256, 0, static_cast<cudaStream_t>(stream)>>>(b, A, ld, logits, labels, dlogits,
                                                                               loss);
  k_mean_loss<<<1, 256, 0, static_cast<cudaStream_t>(stream)>>>(b, loss);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_tr_unpack_h(int64_t rows, int32_t K, const void* h, float* out, void* stream) {
  if (rows <= 0) return 0;
  k_unpack_h<<<grid_for(rows * (K / 8)), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      rows, K, static_cast<const uint16_t*>(h), out);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_tr_unpack_sw128(int64_t rows, int32_t K, const void* a, float* out, void* stream) {
  if (rows <= 0) return 0;
  k_unpack_sw128<<<grid_for(rows * (K / 8)), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      rows, K, static_cast<const uint8_t*>(a), out);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_tr_pool_bwd(int64_t b, int32_t P, const float* proj, const float* dpooled, float* dproj,
                               void* stream) {
  if (b <= 0) return 0;
  k_pool_bwd<<<grid_for(b * 49 * P), 256, 0, static_cast<cudaStream_t>(stream)>>>(b, P, proj, dpooled, dproj);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_tr_droots(int64_t b, const int32_t* root_g, const int32_t* fid, const int32_t* arity_of,
                             const int32_t* example, const float* droots, float* dy_nodes, float* d_inputs,
                             void* stream) {
  if (b <= 0) return 0;
  k_droots<<<grid_for(b * kPx * kC), 256, 0, static_cast<cudaStream_t>(stream)>>>(b, root_g, fid, arity_of, example,
                                                                                 droots, dy_nodes, d_inputs);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_tr_sgd(int64_t n, float* w, const float* g, float lr, void* stream) {
  if (n <= 0) return 0;
  k_sgd<<<grid_for(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(n, w, g, lr);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_tr_pack_conv_weights(const float* w, int32_t cin, int32_t taps, void* out, void* stream) {
  const int64_t total = static_cast<int64_t>(taps) * cin * kC;
  k_pack_conv_w<<<grid_for(total), 256, 0, static_cast<cudaStream_t>(stream)>>>(w, cin, taps,
                                                                              static_cast<uint16_t*>(out));
  return static_cast<int>(cudaGetLastError());
}

extern "C" int dbk_tr_tile_weights(const float* w, int32_t K, int32_t N_src, int32_t N, void* out, void* stream) {
  const int64_t total = static_cast<int64_t>(K) * N;
  k_tile_w<<<grid_for(total), 256, 0, static_cast<cudaStream_t>(stream)>>>(w, K, N_src, N,
                                                                         static_cast<uint16_t*>(out));
  return static_cast<int>(cudaGetLastError());
}
