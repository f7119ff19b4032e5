// iep_train.cpp — one IEP training step on the device (
// PAPER.md:75 reports the paper's batched backward; the reference executor
// stops at the forward).
//
// Forward: the fused step kernel in training mode (every expensive node's
// fp32 value kept, mid images left in place), then the classifier head, then
// mean softmax cross-entropy. Backward: the head's GEMMs, then the module
// groups of the schedule in reverse step order — each group is one batched
// call per weight, exactly as the forward batches them:
//   da2 = dy ⊙ (y > 0);               dW2 += im2col(mid)ᵀ·da2,   db2 += Σ da2
//   da1 = col2im(da2·W2ᵀ) ⊙ (mid > 0); dW1 += im2col(x)ᵀ·da1,     db1 += Σ da1
//   dx  = col2im(da1·W1ᵀ) + da2        (the residual)
//   binary: da0 = dx ⊙ (z > 0); dW0 += [x; y]ᵀ·da0, d[x; y] = da0·W0ᵀ
// and the operand gradients are routed to the children (atomic adds, so
// children shared by several parents accumulate) or to the input maps.
// Activations come from the forward's own staging (fp16 hi + lo), so the
// backward differentiates the arithmetic the forward performed. The GEMMs
// are library GEMMs (cuBLAS, TF32 tensor cores, fp32 accumulation); the
// operand moves are train.cu.
#include "iep_train.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <array>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>

#include "dynbatch.hpp"
#include "iep_head.hpp"
#include "iep_rb.hpp"

#include "dynbatch/dbk.h"

namespace dynbatch::dev {

namespace {

constexpr int kC = 128, kPI = 257, kG = 16, kPx = 196, kK3 = 9 * kC;

void cublas_check(cublasStatus_t st, const char* what) {
  if (st != CUBLAS_STATUS_SUCCESS)
    throw std::runtime_error(std::string("cuBLAS error ") + std::to_string(static_cast<int>(st)) + " in " + what);
}

// TF32 tensor cores (default) or full fp32 (DYNBATCH_TRAIN_FP32=1, A/B of the
// backward's rounding).
// Gradients of the 3×3 convs: the implicit GEMMs of bwd_conv.cu (default) or
// cuBLAS on the im2col layout + col2im (DYNBATCH_TRAIN_DGRAD=0).
bool implicit_dgrad() {
  static const bool on = [] {
    const char* e = std::getenv("DYNBATCH_TRAIN_DGRAD");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}

// Operands of the implicit data gradient: fp16 (dA scaled from its max, the
// pack shared with the weight gradient; default) or tf32 (fp32 rows,
// DYNBATCH_TRAIN_DGRAD_TF32=1).
bool dgrad_f16() {
  static const bool on = [] {
    const char* e = std::getenv("DYNBATCH_TRAIN_DGRAD_TF32");
    return !(e && std::atoi(e) != 0);
  }();
  return on;
}

cublasComputeType_t compute_type() {
  static const cublasComputeType_t t = [] {
    const char* e = std::getenv("DYNBATCH_TRAIN_FP32");
    return e && std::atoi(e) ? CUBLAS_COMPUTE_32F : CUBLAS_COMPUTE_32F_FAST_TF32;
  }();
  return t;
}

// Row-major C[M×N] = op(A)·op(B) (+ beta·C); A is M×K (K×M stored when ta),
// B is K×N (N×K stored when tb); leading dimensions of the stored matrices.
void rm_gemm(cublasHandle_t h, bool ta, bool tb, std::int64_t M, std::int64_t N, std::int64_t K, const float* A,
             std::int64_t lda, const float* B, std::int64_t ldb, float beta, float* C, std::int64_t ldc) {
  if (M <= 0 || N <= 0 || K <= 0) return;
  const float alpha = 1.f;
  cublas_check(cublasGemmEx(h, tb ? CUBLAS_OP_T : CUBLAS_OP_N, ta ? CUBLAS_OP_T : CUBLAS_OP_N, static_cast<int>(N),
                            static_cast<int>(M), static_cast<int>(K), &alpha, B, CUDA_R_32F, static_cast<int>(ldb), A,
                            CUDA_R_32F, static_cast<int>(lda), &beta, C, CUDA_R_32F, static_cast<int>(ldc),
                            compute_type(), CUBLAS_GEMM_DEFAULT),
               "gemm");
}

std::vector<float> to_f32(const std::vector<double>& v) { return std::vector<float>(v.begin(), v.end()); }

}  // namespace

// One row-major GEMM of a grouped call (rm_gemm's arguments).
struct GemmDesc {
  bool ta, tb;
  std::int64_t M, N, K;
  const float* A;
  std::int64_t lda;
  const float* B;
  std::int64_t ldb;
  float* C;
  std::int64_t ldc;
  float beta;
};

// The GEMMs of one step and weight kind (one per group, different weights)
// as one cublasGemmGroupedBatchedEx call (TF32), operands swapped for the
// row-major layout as in rm_gemm. `ptrs` = the calls' device pointer arrays
// (cuBLAS A = our B, cuBLAS B = our A, C), uploaded with every step's.
void grouped_gemm(cublasHandle_t h, const std::vector<GemmDesc>& d, const void* const* ptrs) {
  if (d.empty()) return;
  const size_t n = d.size();
  std::vector<cublasOperation_t> ta(n), tb(n);
  std::vector<int> m(n), nn(n), k(n), lda(n), ldb(n), ldc(n), gs(n, 1);
  std::vector<float> alpha(n, 1.f), beta(n);
  for (size_t i = 0; i < n; ++i) {
    const GemmDesc& g = d[i];
    ta[i] = g.tb ? CUBLAS_OP_T : CUBLAS_OP_N;
    tb[i] = g.ta ? CUBLAS_OP_T : CUBLAS_OP_N;
    m[i] = static_cast<int>(g.N);
    nn[i] = static_cast<int>(g.M);
    k[i] = static_cast<int>(g.K);
    lda[i] = static_cast<int>(g.ldb);
    ldb[i] = static_cast<int>(g.lda);
    ldc[i] = static_cast<int>(g.ldc);
    beta[i] = g.beta;
  }
  const cublasStatus_t st = cublasGemmGroupedBatchedEx(
      h, ta.data(), tb.data(), m.data(), nn.data(), k.data(), alpha.data(), ptrs, CUDA_R_32F, lda.data(), ptrs + n,
      CUDA_R_32F, ldb.data(), beta.data(), const_cast<void* const*>(ptrs + 2 * n), CUDA_R_32F, ldc.data(),
      static_cast<int>(n), gs.data(), compute_type());
  if (st == CUBLAS_STATUS_NOT_SUPPORTED) {  // one call per group
    for (const GemmDesc& g : d) rm_gemm(h, g.ta, g.tb, g.M, g.N, g.K, g.A, g.lda, g.B, g.ldb, g.beta, g.C, g.ldc);
  } else {
    cublas_check(st, "grouped gemm");
  }
}

void IepSession::set_training(bool on) {
  if (!on) {
    train_.reset();
    return;
  }
  if (kind_ != ModuleKind::resblock) throw_error(Errc::invalid_argument, "training needs a resblock session");
  if (train_) return;
  auto t = std::make_unique<Train>();
  cublas_check(cublasCreate(&t->blas), "create");
  cublas_check(cublasSetStream(t->blas, stream_), "stream");

  const HostCSR& c = batch_->csr();
  t->arity = c.arity_of;
  const size_t p = t->arity.size();
  for (auto* v : {&t->w0, &t->w1, &t->w2, &t->gw0, &t->gb0, &t->gw1, &t->gb1, &t->gw2, &t->gb2}) v->resize(p);
  for (size_t f = 0; f < p; ++f) {
    const int a = t->arity[f];
    if (a == 0) continue;
    const ResBlockImpl m = make_resblock_impl(a, kC, module_seed_, static_cast<int>(f));
    if (a == 2) {
      t->w0[f].upload(to_f32(m.w0), stream_);
      t->gw0[f].alloc(m.w0.size());
      t->gb0[f].alloc(kC);
    }
    t->w1[f].upload(to_f32(m.w1), stream_);
    t->w2[f].upload(to_f32(m.w2), stream_);
    t->gw1[f].alloc(m.w1.size());
    t->gw2[f].alloc(m.w2.size());
    t->gb1[f].alloc(kC);
    t->gb2[f].alloc(kC);
    check(cudaStreamSynchronize(stream_), "training weights");  // the host vectors go out of scope
  }
  // transposed tap blocks for the implicit-GEMM data gradients
  t->wd1.resize(p);
  t->wd2.resize(p);
  std::vector<const void*> tab1(p, nullptr), tab2(p, nullptr);
  for (size_t f = 0; f < p; ++f) {
    if (t->arity[f] == 0) continue;
    const bool h = dgrad_f16();
    const size_t bytes = static_cast<size_t>(9) * (h ? 2 : 4) * 16384;
    t->wd1[f].alloc(bytes);
    t->wd2[f].alloc(bytes);
    const auto pack = h ? dbk_tr_pack_dgrad_weights_h : dbk_tr_pack_dgrad_weights;
    check(pack(t->w1[f].get(), t->wd1[f].get(), stream_), "dgrad weights");
    check(pack(t->w2[f].get(), t->wd2[f].get(), stream_), "dgrad weights");
    tab1[f] = t->wd1[f].get();
    tab2[f] = t->wd2[f].get();
  }
  t->wd1tab.upload(tab1, stream_);
  t->wd2tab.upload(tab2, stream_);
  std::vector<float*> g1(p, nullptr), g2(p, nullptr);
  for (size_t f = 0; f < p; ++f) {
    g1[f] = t->gw1[f].get();
    g2[f] = t->gw2[f].get();
  }
  t->gw1tab.upload(g1, stream_);
  t->gw2tab.upload(g2, stream_);
  check(cudaStreamSynchronize(stream_), "dgrad tables");
  train_ = std::move(t);
}

float IepSession::train_step(const std::int32_t* labels) {
  if (!train_) throw_error(Errc::invalid_argument, "training is off: call set_training first");
  require_head();
  Train& T = *train_;
  flush_programs();
  const std::int64_t b = batch_->csr().b;
  for (std::int64_t e = 0; e < b; ++e)
    if (labels[e] < 0 || labels[e] >= head_->answers()) throw_error(Errc::invalid_argument, "label out of range");
  T.labels.upload(labels, static_cast<size_t>(b), stream_);
  T.loss.ensure(static_cast<size_t>(b) + 1);  // [0] mean, [1 + e] per program
  train_fwd_ = true;
  try {
    forward_direct();
  } catch (...) {
    train_fwd_ = false;
    throw;
  }
  train_fwd_ = false;
  check_errors();
  head_forward();
  backward(T.loss.get());
  T.stepped = true;
  float loss = 0.f;
  check(cudaMemcpyAsync(&loss, T.loss.get(), sizeof(float), cudaMemcpyDeviceToHost, stream_), "D2H loss");
  check(cudaStreamSynchronize(stream_), "sync");
  return loss;
}

void IepSession::backward(float* loss_dev) {
  Train& T = *train_;
  RB& R = *rb_;
  DeviceProgramBatch& B = *batch_;
  cudaStream_t s = stream_;
  const HostCSR& c = B.csr();
  const std::int64_t b = c.b, N = c.N;
  const int A = head_->answers(), P = IepHead::kP, F = IepHead::kF, K1 = 49 * P;
  // ---- sizes, zeroed gradient accumulators
  if (b > T.cap_b) {
    T.d_inputs.alloc(static_cast<size_t>(b) * kC * kPx);
    T.dlogits.alloc(static_cast<size_t>(b) * A > 0 ? static_cast<size_t>(b) * 256 : 1);
    T.hid.alloc(static_cast<size_t>(b) * F);
    T.dhid.alloc(static_cast<size_t>(b) * F);
    T.pooled.alloc(static_cast<size_t>(b) * K1);
    T.dpooled.alloc(static_cast<size_t>(b) * K1);
    T.proj.alloc(static_cast<size_t>(b) * kPx * P);
    T.dproj.alloc(static_cast<size_t>(b) * kPx * P);
    T.roots.alloc(static_cast<size_t>(b) * kPx * kC);
    T.droots.alloc(static_cast<size_t>(b) * kPx * kC);
    T.cap_b = b;
  }
  if (N > T.cap_n) {
    T.dy_nodes.alloc(static_cast<size_t>(N) * kPI * kC);
    T.cap_n = N;
  }
  if (T.gwp.size() < static_cast<size_t>(kC) * P) {
    T.gwp.alloc(static_cast<size_t>(kC) * P);
    T.gbp.alloc(P);
    T.ghw1.alloc(static_cast<size_t>(K1) * F);
    T.ghb1.alloc(F);
  }
  T.ghw2.ensure(static_cast<size_t>(F) * A);
  T.ghb2.ensure(static_cast<size_t>(A));
  T.d_inputs.zero(s);
  T.dy_nodes.zero(s);
  for (Buf<float>* v : {&T.gwp, &T.gbp, &T.ghw1, &T.ghb1, &T.ghw2, &T.ghb2}) v->zero(s);
  for (size_t f = 0; f < T.arity.size(); ++f)
    for (Buf<float>* v : {&T.gw0[f], &T.gb0[f], &T.gw1[f], &T.gb1[f], &T.gw2[f], &T.gb2[f]}) v->zero(s);
  cublasHandle_t h = T.blas;

  // ---- head: loss, FC2, FC1, pool, projection
  check(dbk_tr_softmax_ce(b, A, IepHead::kPad, head_->logits(), T.labels.get(), T.dlogits.get(), loss_dev, s), "ce");
  check(dbk_tr_unpack_h(b, F, head_->hidden_tiled(), T.hid.get(), s), "unpack hidden");
  check(dbk_tr_unpack_sw128(b, K1, head_->pooled_tiled(), T.pooled.get(), s), "unpack pooled");
  check(dbk_tr_unpack_h(b * kPx, P, head_->proj_tiled(), T.proj.get(), s), "unpack projection");
  check(dbk_tr_unpack_sw128(b * kPx, kC, head_->roots_tiled(), T.roots.get(), s), "unpack roots");
  rm_gemm(h, true, false, F, A, b, T.hid.get(), F, T.dlogits.get(), A, 0.f, T.ghw2.get(), A);
  check(dbk_tr_colsum(b, A, T.dlogits.get(), T.ghb2.get(), s), "db2");
  rm_gemm(h, false, true, b, F, A, T.dlogits.get(), A, head_->w2_32(), A, 0.f, T.dhid.get(), F);
  check(dbk_tr_mask(b * F, T.dhid.get(), T.hid.get(), T.dhid.get(), s), "relu fc1");
  rm_gemm(h, true, false, K1, F, b, T.pooled.get(), K1, T.dhid.get(), F, 0.f, T.ghw1.get(), F);
  check(dbk_tr_colsum(b, F, T.dhid.get(), T.ghb1.get(), s), "db1");
  rm_gemm(h, false, true, b, K1, F, T.dhid.get(), F, head_->w1_32(), F, 0.f, T.dpooled.get(), K1);
  check(dbk_tr_pool_bwd(b, P, T.proj.get(), T.dpooled.get(), T.dproj.get(), s), "pool backward");
  rm_gemm(h, true, false, kC, P, b * kPx, T.roots.get(), kC, T.dproj.get(), P, 0.f, T.gwp.get(), P);
  check(dbk_tr_colsum(b * kPx, P, T.dproj.get(), T.gbp.get(), s), "dbp");
  rm_gemm(h, false, true, b * kPx, kC, P, T.dproj.get(), P, head_->wp32(), P, 0.f, T.droots.get(), kC);
  check(dbk_tr_droots(b, B.root_g.get(), B.fid.get(), B.arity_of.get(), B.example.get(), T.droots.get(),
                      T.dy_nodes.get(), T.d_inputs.get(), s),
        "route roots");

  // ---- module groups, reverse step order: each step's expensive members in
  // one set of PI buffers (unary groups first, then binary), elementwise
  // kernels over the whole step, one grouped GEMM per weight kind and step
  const int S = B.steps;
  const std::vector<std::int32_t> sgb = B.step_group_begin.download(static_cast<size_t>(S) + 1, s);
  const std::int64_t G = sgb[static_cast<size_t>(S)];
  const std::vector<std::int32_t> gfid = B.group_fid.download(static_cast<size_t>(G), s);
  const std::vector<std::int32_t> gbeg = B.group_begin.download(static_cast<size_t>(G) + 1, s);
  const std::vector<std::int32_t> seg = R.seg_start.download(static_cast<size_t>(G), s);
  const std::vector<std::int32_t> mem = B.member_g.download(static_cast<size_t>(gbeg[static_cast<size_t>(G)]), s);
  struct StepPlan {
    std::int64_t n = 0, n_u = 0;       // members, of which in unary groups
    std::int64_t m_off = 0;            // into the node / row tables
    std::vector<int> groups;           // schedule groups, unary first
    std::vector<std::int64_t> first;   // member index (within the step) of each group
  };
  std::vector<StepPlan> plan(static_cast<size_t>(S));
  std::vector<std::int32_t> h_nodes;
  std::vector<std::int64_t> h_rows, h_slab;
  std::vector<float*> h_slab_dst;
  std::int64_t n_max = 0;
  for (int st = 0; st < S; ++st) {
    StepPlan& sp = plan[static_cast<size_t>(st)];
    sp.m_off = static_cast<std::int64_t>(h_nodes.size());
    for (int pass = 1; pass <= 2; ++pass)
      for (std::int32_t g = sgb[static_cast<size_t>(st)]; g < sgb[static_cast<size_t>(st) + 1]; ++g) {
        const int a = T.arity[static_cast<size_t>(gfid[static_cast<size_t>(g)])];
        if (a != pass || seg[static_cast<size_t>(g)] < 0 || gbeg[g + 1] == gbeg[g]) continue;
        sp.groups.push_back(g);
        sp.first.push_back(sp.n);
        for (std::int32_t m = gbeg[g]; m < gbeg[g + 1]; ++m) {
          h_nodes.push_back(mem[static_cast<size_t>(m)]);
          h_rows.push_back(seg[static_cast<size_t>(g)] + static_cast<std::int64_t>(m - gbeg[g]) * 225);
        }
        sp.n += gbeg[g + 1] - gbeg[g];
        if (pass == 1) sp.n_u = sp.n;
      }
    n_max = std::max(n_max, sp.n);
  }
  const std::int64_t rows_max = n_max * kPI;
  if (rows_max > T.cap_rows) {
    const size_t r = static_cast<size_t>(rows_max), rg = r + 2 * kG;
    T.da2.alloc(r * kC);
    T.mid.alloc(rg * kC);
    T.xin.alloc(rg * kC);
    if (!implicit_dgrad()) {  // the im2col path's 9×-expanded operands (3.4 GB each at cfg3)
      T.cols.alloc(r * kK3);
      T.g.alloc(r * kK3);
    }
    T.da1.alloc(r * kC);
    T.dx.alloc(r * kC);
    T.da0.alloc(r * kC);
    T.cat.alloc(r * 2 * kC);
    T.dcat.alloc(r * 2 * kC);
    T.cap_rows = rows_max;
  }
  T.nodes.upload(h_nodes, s);
  T.rows.upload(h_rows, s);
  const std::int64_t ps = R.plane_stride;
  float* mid = T.mid.get() + kG * kC;  // row 0 of the first member (16 guard rows before)
  float* xin = T.xin.get() + kG * kC;
  // per (group, bias): slabs of ≤ 512 rows; the tables of every step and
  // bias kind are built here and uploaded once
  struct SlabRange { std::int64_t begin, count; };
  auto add_slabs = [&](const StepPlan& sp, size_t gi0, size_t gi1, std::int64_t row_base,
                       std::vector<Buf<float>>& dst) -> SlabRange {
    const SlabRange r{static_cast<std::int64_t>(h_slab_dst.size()), 0};
    SlabRange out = r;
    for (size_t gi = gi0; gi < gi1; ++gi) {
      const int g = sp.groups[gi];
      const std::int64_t r0 = sp.first[gi] * kPI - row_base;
      const std::int64_t r1 = (gi + 1 < sp.groups.size() ? sp.first[gi + 1] : sp.n) * kPI - row_base;
      for (std::int64_t x = r0; x < r1; x += 512) {
        h_slab.push_back(x);
        h_slab.push_back(std::min(r1, x + 512));
        h_slab_dst.push_back(dst[static_cast<size_t>(gfid[static_cast<size_t>(g)])].get());
        ++out.count;
      }
    }
    return out;
  };
  std::vector<std::array<SlabRange, 3>> slabs(static_cast<size_t>(S));
  for (int st = 0; st < S; ++st) {
    const StepPlan& sp = plan[static_cast<size_t>(st)];
    const size_t nu = static_cast<size_t>(std::count_if(sp.first.begin(), sp.first.end(),
                                                        [&](std::int64_t f) { return f < sp.n_u; }));
    slabs[static_cast<size_t>(st)][0] = add_slabs(sp, 0, sp.groups.size(), 0, T.gb2);
    slabs[static_cast<size_t>(st)][1] = add_slabs(sp, 0, sp.groups.size(), 0, T.gb1);
    slabs[static_cast<size_t>(st)][2] = add_slabs(sp, nu, sp.groups.size(), sp.n_u * kPI, T.gb0);
  }
  T.slab_row.upload(h_slab, s);  // pairs (begin, end) per slab
  T.slab_dst.upload(h_slab_dst, s);
  // implicit data-gradient tiles: 256 PI rows within one group, starting on
  // a multiple of 8 (the window swizzle), every step's in one table
  const bool dgrad = implicit_dgrad();
  std::vector<std::int64_t> tile_off(static_cast<size_t>(S) + 1, 0), item_off(static_cast<size_t>(S) + 1, 0);
  if (dgrad) {
    // weight-gradient items: a group's rows widened to multiples of 8 (the
    // extra rows are zero dA guard rows), in K ranges of kKR, per kernel row
    static const std::int64_t kKR = [] {  // K rows per weight-gradient item (A/B: DYNBATCH_WGRAD_KR)
      const char* e = std::getenv("DYNBATCH_WGRAD_KR");
      return e ? std::max<std::int64_t>(64, std::atoll(e) / 64 * 64) : 8192;
    }();
    std::vector<std::int32_t> t_row0, t_lo, t_hi, t_fn, w_k0, w_k1, w_dr, w_fn;
    for (int st = 0; st < S; ++st) {
      const StepPlan& sp = plan[static_cast<size_t>(st)];
      tile_off[static_cast<size_t>(st)] = static_cast<std::int64_t>(t_row0.size());
      item_off[static_cast<size_t>(st)] = static_cast<std::int64_t>(w_k0.size());
      for (size_t gi = 0; gi < sp.groups.size(); ++gi) {
        const std::int64_t lo = sp.first[gi] * kPI;
        const std::int64_t hi = (gi + 1 < sp.groups.size() ? sp.first[gi + 1] : sp.n) * kPI;
        const std::int32_t fn = gfid[static_cast<size_t>(sp.groups[gi])];
        for (std::int64_t r = lo / 8 * 8; r < hi; r += 256) {
          t_row0.push_back(static_cast<std::int32_t>(r));
          t_lo.push_back(static_cast<std::int32_t>(lo));
          t_hi.push_back(static_cast<std::int32_t>(hi));
          t_fn.push_back(fn);
        }
        // K ranges on multiples of 16 (one fp16 MMA): the widened rows are
        // zero-dA guard rows of the neighbouring members
        const std::int64_t k_end = (hi + 15) / 16 * 16;
        for (std::int64_t k = lo / 16 * 16; k < k_end; k += kKR)
          for (int dr = 0; dr < 3; ++dr) {
            w_k0.push_back(static_cast<std::int32_t>(k));
            w_k1.push_back(static_cast<std::int32_t>(std::min(k + kKR, k_end)));
            w_dr.push_back(dr);
            w_fn.push_back(fn);
          }
      }
    }
    tile_off[static_cast<size_t>(S)] = static_cast<std::int64_t>(t_row0.size());
    item_off[static_cast<size_t>(S)] = static_cast<std::int64_t>(w_k0.size());
    std::vector<std::int32_t> all;
    all.reserve(4 * t_row0.size());
    for (const auto* v : {&t_row0, &t_lo, &t_hi, &t_fn}) all.insert(all.end(), v->begin(), v->end());
    T.dtiles.upload(all, s);
    all.clear();
    for (const auto* v : {&w_k0, &w_k1, &w_dr, &w_fn}) all.insert(all.end(), v->begin(), v->end());
    T.witems.upload(all, s);
    const std::int64_t need_rows = rows_max + 16 + 256 + 32;
    if (need_rows > T.dpack_rows) {
      T.dpack.alloc(static_cast<size_t>(4 * need_rows * 128));
      T.apack.alloc(static_cast<size_t>(2 * need_rows * 128));
      T.hpack.alloc(static_cast<size_t>(2 * need_rows * 128));
      T.dpack_rows = need_rows;
    }
    T.absmax.ensure(2);  // |dA2|, |dA1| maxima of the step (the fp16 scales)
  }
  const std::int64_t n_items_all = item_off[static_cast<size_t>(S)];
  const std::int64_t n_tiles_all = tile_off[static_cast<size_t>(S)];
  const int sms = sm_count();
  // data gradient of one 3×3 conv over the step's PI rows (the dA operand
  // packed first); mask / resid as the col2im it replaces
  const bool f16 = dgrad_f16();
  // dA (PI rows) → fp16 rows scaled from its max, for both implicit GEMMs
  // dA (PI rows) → fp16 rows scaled from its max (word `mx` of T.absmax:
  // 0 = dA2, written by da_out; 1 = dA1, by the conv3x3 #2 data gradient,
  // or here with k_absmax on the tf32 path), for both implicit GEMMs
  std::uint32_t* amax = T.absmax.get();
  auto pack_da_h = [&](const float* da, std::int64_t rows, int mx, bool measure) {
    if (measure) check(dbk_tr_absmax(rows * kC, da, amax + mx, s), "dA max");
    check(dbk_tr_pack_sw128h(rows, T.dpack_rows, 16, da, amax + mx, T.hpack.get(), s), "pack dA");
  };
  auto dgrad_conv = [&](int st, const float* da, int mx, const Buf<const void*>& wtab, const void* mask_h,
                        const float* resid, float* out, std::uint32_t* out_max, std::int64_t rows) {
    if (f16) pack_da_h(da, rows, mx, false);
    else check(dbk_tr_pack_sw128f(rows, T.dpack_rows, 16, da, T.dpack.get(), s), "pack dA");
    const std::int64_t t0 = tile_off[static_cast<size_t>(st)], nt = tile_off[static_cast<size_t>(st) + 1] - t0;
    const std::int32_t* tb = T.dtiles.get();
    check(dbk_tr_dgrad(f16 ? T.hpack.get() : T.dpack.get(), f16 ? 1 : 0, amax + mx, T.dpack_rows, 16,
                       static_cast<std::int32_t>(nt), tb + t0, tb + n_tiles_all + t0, tb + 2 * n_tiles_all + t0,
                       tb + 3 * n_tiles_all + t0, wtab.get(), nullptr, mask_h, resid, out, out_max, sms, s),
          "dgrad");
  };
  // weight gradient of one 3×3 conv: its input activations (already packed
  // into apack from the forward's staging) and dA; dA's fp16 pack is
  // dgrad_conv's when that ran on fp16
  auto wgrad_conv = [&](int st, const float* da, int mx, const Buf<float*>& gwtab, std::int64_t rows) {
    if (!f16) pack_da_h(da, rows, mx, true);
    const std::int64_t i0 = item_off[static_cast<size_t>(st)], ni = item_off[static_cast<size_t>(st) + 1] - i0;
    check(dbk_tr_wgrad(T.apack.get(), T.hpack.get(), amax + mx, T.dpack_rows, 16, static_cast<std::int32_t>(ni),
                       T.witems.get() + i0, n_items_all, gwtab.get(), sms, s),
          "wgrad");
  };
  auto colsum = [&](const SlabRange& r, const float* a) {
    if (r.count)
      check(dbk_tr_colsum_seg(static_cast<std::int32_t>(r.count), T.slab_row.get() + 2 * r.begin,
                              T.slab_dst.get() + r.begin, a, s),
            "bias gradients");
  };
  // per-group GEMM descriptors of every step (6 kinds: dW2, G2, dW1, G1, dW0,
  // dcat) and their device pointer arrays, uploaded once
  std::vector<std::array<std::vector<GemmDesc>, 6>> descs(static_cast<size_t>(S));
  std::vector<std::array<std::int64_t, 6>> ptr_off(static_cast<size_t>(S));
  std::vector<const void*> h_ptrs;
  for (int st = 0; st < S; ++st) {
    const StepPlan& sp = plan[static_cast<size_t>(st)];
    auto& [w2, d2, w1, d1, w0, d0] = descs[static_cast<size_t>(st)];
    for (size_t gi = 0; gi < sp.groups.size(); ++gi) {
      const size_t f = static_cast<size_t>(gfid[static_cast<size_t>(sp.groups[gi])]);
      const std::int64_t r0 = sp.first[gi] * kPI;
      const std::int64_t rg = ((gi + 1 < sp.groups.size() ? sp.first[gi + 1] : sp.n) - sp.first[gi]) * kPI;
      if (!dgrad) {  // the im2col path's GEMMs (the implicit kernels need none)
        w2.push_back({true, false, kK3, kC, rg, T.cols.get() + r0 * kK3, kK3, T.da2.get() + r0 * kC, kC,
                      T.gw2[f].get(), kC, 1.f});
        d2.push_back({false, true, rg, kK3, kC, T.da2.get() + r0 * kC, kC, T.w2[f].get(), kC, T.g.get() + r0 * kK3,
                      kK3, 0.f});
        w1.push_back({true, false, kK3, kC, rg, T.cols.get() + r0 * kK3, kK3, T.da1.get() + r0 * kC, kC,
                      T.gw1[f].get(), kC, 1.f});
        d1.push_back({false, true, rg, kK3, kC, T.da1.get() + r0 * kC, kC, T.w1[f].get(), kC, T.g.get() + r0 * kK3,
                      kK3, 0.f});
      }
      if (r0 >= sp.n_u * kPI) {  // binary group: rows relative to the binary part
        const std::int64_t rb = r0 - sp.n_u * kPI;
        w0.push_back({true, false, 2 * kC, kC, rg, T.cat.get() + rb * 2 * kC, 2 * kC, T.da0.get() + rb * kC, kC,
                      T.gw0[f].get(), kC, 1.f});
        d0.push_back({false, true, rg, 2 * kC, kC, T.da0.get() + rb * kC, kC, T.w0[f].get(), kC,
                      T.dcat.get() + rb * 2 * kC, 2 * kC, 0.f});
      }
    }
    for (size_t kd = 0; kd < 6; ++kd) {
      const auto& d = descs[static_cast<size_t>(st)][kd];
      ptr_off[static_cast<size_t>(st)][kd] = static_cast<std::int64_t>(h_ptrs.size());
      for (const GemmDesc& g : d) h_ptrs.push_back(g.B);
      for (const GemmDesc& g : d) h_ptrs.push_back(g.A);
      for (const GemmDesc& g : d) h_ptrs.push_back(g.C);
    }
  }
  T.ptr_dev.upload(h_ptrs, s);
  check(cudaStreamSynchronize(s), "backward tables");  // the host tables go out of scope
  for (int st = S - 1; st >= 0; --st) {
    const StepPlan& sp = plan[static_cast<size_t>(st)];
    if (sp.n == 0) continue;
    const std::int64_t n = sp.n, rows = n * kPI;
    const std::int32_t* nodes = T.nodes.get() + sp.m_off;
    const std::int64_t* srows = T.rows.get() + sp.m_off;
    const auto& dd = descs[static_cast<size_t>(st)];
    const auto& po = ptr_off[static_cast<size_t>(st)];
    // one cuBLAS call per group: the weight gradients (K = the group's rows,
    // a small M × N) need split-K, and cublasGemmGroupedBatchedEx runs the
    // data gradients on sm_80 grouped kernels 4× slower than the per-call
    // sm_100 ones (measured); DYNBATCH_TRAIN_GROUPED=1 uses it for the latter
    static const bool grouped_dgrad = [] {
      const char* e = std::getenv("DYNBATCH_TRAIN_GROUPED");
      return e && std::atoi(e) != 0;
    }();
    auto gemms = [&](int kd) {
      const auto& d = dd[static_cast<size_t>(kd)];
      if (kd % 2 == 1 && grouped_dgrad) {
        grouped_gemm(T.blas, d, T.ptr_dev.get() + po[static_cast<size_t>(kd)]);
        return;
      }
      for (const GemmDesc& g : d) rm_gemm(T.blas, g.ta, g.tb, g.M, g.N, g.K, g.A, g.lda, g.B, g.ldb, g.beta, g.C, g.ldc);
    };
    if (!dgrad) {  // the im2col path's fp32 activations (the implicit path packs them straight from staging)
      check(cudaMemsetAsync(T.mid.get(), 0, sizeof(float) * static_cast<size_t>(rows + 2 * kG) * kC, s), "zero");
      check(cudaMemsetAsync(T.xin.get(), 0, sizeof(float) * static_cast<size_t>(rows + 2 * kG) * kC, s), "zero");
    }
    // conv3x3 #2: da2 → dW2, db2; da1 = col2im(da2·W2ᵀ) ⊙ (mid > 0)
    if (dgrad) check(cudaMemsetAsync(amax, 0, 2 * sizeof(std::uint32_t), s), "maxima");
    check(dbk_tr_da_out(static_cast<std::int32_t>(n), nodes, T.dy_nodes.get(), R.values.get(), T.da2.get(),
                        dgrad ? amax : nullptr, s),
          "da2");
    colsum(slabs[static_cast<size_t>(st)][0], T.da2.get());
    if (dgrad) {
      check(dbk_tr_stage_to_pack(static_cast<std::int32_t>(n), srows, R.stage_mid.get(), ps, T.dpack_rows, 16,
                                 T.apack.get(), s),
            "pack mid");
      dgrad_conv(st, T.da2.get(), 0, T.wd2tab, T.apack.get(), nullptr, T.da1.get(), f16 ? amax + 1 : nullptr, rows);
      wgrad_conv(st, T.da2.get(), 0, T.gw2tab, rows);
    } else {
      check(dbk_tr_stage_to_pi(static_cast<std::int32_t>(n), srows, R.stage_mid.get(), nullptr, ps, 0, 16, mid, s),
            "mid");
      check(dbk_tr_im2col(rows, kC, mid, T.cols.get(), s), "im2col mid");
      gemms(0);
      gemms(1);
      check(dbk_tr_col2im(static_cast<std::int32_t>(n), kC, T.g.get(), nullptr, mid, T.da1.get(), s), "col2im mid");
    }
    // conv3x3 #1: dW1, db1; dx = col2im(da1·W1ᵀ) + da2 (the residual)
    colsum(slabs[static_cast<size_t>(st)][1], T.da1.get());
    if (dgrad) {
      check(dbk_tr_stage_to_pack(static_cast<std::int32_t>(n), srows, R.stage_x.get(), ps, T.dpack_rows, 16,
                                 T.apack.get(), s),
            "pack x");
      dgrad_conv(st, T.da1.get(), 1, T.wd1tab, nullptr, T.da2.get(), T.dx.get(), nullptr, rows);
      wgrad_conv(st, T.da1.get(), 1, T.gw1tab, rows);
    } else {
      check(dbk_tr_stage_to_pi(static_cast<std::int32_t>(n), srows, R.stage_x.get(), R.stage_lo.get(), ps, 0, 16, xin,
                               s),
            "x");
      check(dbk_tr_im2col(rows, kC, xin, T.cols.get(), s), "im2col x");
      gemms(2);
      gemms(3);
      check(dbk_tr_col2im(static_cast<std::int32_t>(n), kC, T.g.get(), T.da2.get(), nullptr, T.dx.get(), s), "col2im x");
    }
    if (sp.n_u > 0)
      check(dbk_tr_route(static_cast<std::int32_t>(sp.n_u), nodes, B.child0.get(), B.fid.get(), B.arity_of.get(),
                         B.example.get(), T.dx.get(), kC, 0, T.dy_nodes.get(), T.d_inputs.get(), s),
            "route");
    const std::int64_t nb = n - sp.n_u;
    if (nb == 0) continue;
    // binary groups: z = relu(conv1x1([x; y]) + b0) was the block input
    const std::int64_t ub = sp.n_u * kPI;
    if (dgrad)  // z from the packed x rows
      check(dbk_tr_mask_h(ub, nb * kPI, T.dx.get(), T.apack.get(), T.dpack_rows, 16, T.da0.get(), s),
            "relu z");
    else
      check(dbk_tr_mask(nb * kPI * kC, T.dx.get() + ub * kC, xin + ub * kC, T.da0.get(), s), "relu z");
    colsum(slabs[static_cast<size_t>(st)][2], T.da0.get());
    check(cudaMemsetAsync(T.cat.get(), 0, sizeof(float) * static_cast<size_t>(nb * kPI) * 2 * kC, s), "zero");
    check(dbk_tr_stage_to_pi(static_cast<std::int32_t>(nb), srows + sp.n_u, R.stage_cat.get(), nullptr, ps, 0, 32,
                             T.cat.get(), s),
          "cat");
    gemms(4);
    gemms(5);
    for (int k = 0; k < 2; ++k)
      check(dbk_tr_route(static_cast<std::int32_t>(nb), nodes + sp.n_u, k == 0 ? B.child0.get() : B.child1.get(),
                         B.fid.get(), B.arity_of.get(), B.example.get(), T.dcat.get(), 2 * kC, k * kC,
                         T.dy_nodes.get(), T.d_inputs.get(), s),
            "route");
  }
}

std::int64_t IepSession::grad_size(int which, int fid) const {
  if (!train_ || !head_) throw_error(Errc::invalid_argument, "training is off or no head");
  const std::int64_t C = kC, P = IepHead::kP, F = IepHead::kF, A = head_->answers();
  if (which < 6) {
    if (fid < 0 || fid >= static_cast<int>(train_->arity.size()) || train_->arity[static_cast<size_t>(fid)] == 0)
      throw_error(Errc::unknown_function, "function " + std::to_string(fid) + " has no weights");
    const int a = train_->arity[static_cast<size_t>(fid)];
    switch (which) {
      case 0: return a == 2 ? 2 * C * C : 0;
      case 1: return a == 2 ? C : 0;
      case 2: case 4: return 9 * C * C;
      default: return C;
    }
  }
  switch (which) {
    case 6: return C * P;
    case 7: return P;
    case 8: return 49 * P * F;
    case 9: return F;
    case 10: return F * A;
    case 11: return A;
    case 12: return batch_->csr().b * C * kPx;
    default: throw_error(Errc::invalid_argument, "gradient index");
  }
}

void IepSession::download_grad(int which, int fid, float* out, std::int64_t n) {
  const std::int64_t want = grad_size(which, fid);
  if (n != want) throw_error(Errc::row_count_mismatch, "gradient buffer size");
  if (n == 0) return;
  Train& T = *train_;
  const float* src = nullptr;
  const size_t f = static_cast<size_t>(std::max(fid, 0));
  switch (which) {
    case 0: src = T.gw0[f].get(); break;
    case 1: src = T.gb0[f].get(); break;
    case 2: src = T.gw1[f].get(); break;
    case 3: src = T.gb1[f].get(); break;
    case 4: src = T.gw2[f].get(); break;
    case 5: src = T.gb2[f].get(); break;
    case 6: src = T.gwp.get(); break;
    case 7: src = T.gbp.get(); break;
    case 8: src = T.ghw1.get(); break;
    case 9: src = T.ghb1.get(); break;
    case 10: src = T.ghw2.get(); break;
    case 11: src = T.ghb2.get(); break;
    default: src = T.d_inputs.get(); break;
  }
  check(cudaMemcpyAsync(out, src, sizeof(float) * static_cast<size_t>(n), cudaMemcpyDeviceToHost, stream_), "D2H");
  check(cudaStreamSynchronize(stream_), "sync");
}

void IepSession::sgd_update(float lr) {
  if (!train_) throw_error(Errc::invalid_argument, "training is off: call set_training first");
  Train& T = *train_;
  if (!T.stepped) throw_error(Errc::invalid_argument, "no gradients: call train_step first");
  RB& R = *rb_;
  cudaStream_t s = stream_;
  const size_t p = T.arity.size();
  if (T.fw1.empty()) {
    T.fw0 = R.w0tab.download(p, s);
    T.fw1 = R.w1tab.download(p, s);
    T.fw2 = R.w2tab.download(p, s);
    T.fb0 = R.b0tab.download(p, s);
    T.fb1 = R.b1tab.download(p, s);
    T.fb2 = R.b2tab.download(p, s);
  }
  const bool h = dgrad_f16();
  for (size_t f = 0; f < p; ++f) {
    const int a = T.arity[f];
    if (a == 0) continue;
    const std::int64_t n3 = 9LL * kC * kC;
    check(dbk_tr_sgd(n3, T.w1[f].get(), T.gw1[f].get(), lr, s), "sgd");
    check(dbk_tr_sgd(n3, T.w2[f].get(), T.gw2[f].get(), lr, s), "sgd");
    check(dbk_tr_sgd(kC, const_cast<float*>(T.fb1[f]), T.gb1[f].get(), lr, s), "sgd");
    check(dbk_tr_sgd(kC, const_cast<float*>(T.fb2[f]), T.gb2[f].get(), lr, s), "sgd");
    check(dbk_tr_pack_conv_weights(T.w1[f].get(), kC, 9, const_cast<void*>(T.fw1[f]), s), "repack");
    check(dbk_tr_pack_conv_weights(T.w2[f].get(), kC, 9, const_cast<void*>(T.fw2[f]), s), "repack");
    if (a == 2) {
      check(dbk_tr_sgd(2LL * kC * kC, T.w0[f].get(), T.gw0[f].get(), lr, s), "sgd");
      check(dbk_tr_sgd(kC, const_cast<float*>(T.fb0[f]), T.gb0[f].get(), lr, s), "sgd");
      check(dbk_tr_pack_conv_weights(T.w0[f].get(), 2 * kC, 1, const_cast<void*>(T.fw0[f]), s), "repack");
    }
    if (!T.wd1.empty() && T.wd1[f].get()) {
      const auto pack = h ? dbk_tr_pack_dgrad_weights_h : dbk_tr_pack_dgrad_weights;
      check(pack(T.w1[f].get(), T.wd1[f].get(), s), "dgrad weights");
      check(pack(T.w2[f].get(), T.wd2[f].get(), s), "dgrad weights");
    }
  }
  head_->sgd(lr, T.gwp.get(), T.gbp.get(), T.ghw1.get(), T.ghb1.get(), T.ghw2.get(), T.ghb2.get(), s);
  check(cudaStreamSynchronize(s), "sgd");
}

double IepSession::time_train(int iters, const std::int32_t* labels) {
  train_step(labels);  // warm: sizes every buffer
  cudaEvent_t e0, e1;
  check(cudaEventCreate(&e0), "event");
  check(cudaEventCreate(&e1), "event");
  check(cudaEventRecord(e0, stream_), "event");
  for (int i = 0; i < iters; ++i) train_step(labels);
  check(cudaEventRecord(e1, stream_), "event");
  check(cudaEventSynchronize(e1), "sync");
  float ms = 0.f;
  check(cudaEventElapsedTime(&ms, e0, e1), "elapsed");
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return ms / std::max(iters, 1);
}

}  // namespace dynbatch::dev
