// iep_resblock.cpp — Tier-B residual conv module path of the IEP session:
// weight packing for the tcgen05 kernels, buffer sizing and the per-step
// launch sequence  plan → [gather → conv1x1 → conv3x3#1 → conv3x3#2]×steps.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "device.hpp"
#include "dynbatch/dbk.h"
#include "iep_head.hpp"
#include "iep_train.hpp"
#include "iep_rb.hpp"

namespace dynbatch::dev {

IepSession::~IepSession() {
  if (stream_) {
    cudaStreamSynchronize(stream_);
    cudaStreamDestroy(stream_);
  }
  for (CachedGraph& g : graphs_) release_graph(g);
  for (cudaEvent_t e : kev_pool_) cudaEventDestroy(e);
  for (cudaEvent_t e : kev_mark_)
    if (e) cudaEventDestroy(e);
}

namespace {

// fp32 → fp16 bits, round to nearest even, subnormals kept (the tensor-core
// operands of the conv kernels are fp16: 2^-11 relative rounding vs bf16's 2^-9).
std::uint16_t to_f16(double v) {
  const float f = static_cast<float>(v);
  std::uint32_t x;
  std::memcpy(&x, &f, 4);
  const std::uint32_t sign = (x >> 16) & 0x8000u;
  const std::uint32_t e8 = (x >> 23) & 0xffu;
  std::uint32_t mant = x & 0x7fffffu;
  if (e8 == 0xffu) return static_cast<std::uint16_t>(sign | 0x7c00u | (mant ? 0x200u : 0u));
  const std::int32_t e = static_cast<std::int32_t>(e8) - 127 + 15;
  if (e >= 31) return static_cast<std::uint16_t>(sign | 0x7c00u);
  if (e <= 0) {
    if (e < -10) return static_cast<std::uint16_t>(sign);
    mant |= 0x800000u;
    const std::uint32_t shift = static_cast<std::uint32_t>(14 - e);
    std::uint32_t h = mant >> shift;
    const std::uint32_t rem = mant & ((1u << shift) - 1u), halfway = 1u << (shift - 1u);
    if (rem > halfway || (rem == halfway && (h & 1u))) ++h;
    return static_cast<std::uint16_t>(sign | h);
  }
  std::uint32_t h = (static_cast<std::uint32_t>(e) << 10) | (mant >> 13);
  const std::uint32_t rem = mant & 0x1fffu;
  if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) ++h;
  return static_cast<std::uint16_t>(sign | h);
}

// Weights are streamed as 16 KB blocks, one per (64-channel K chunk, tap) in
// that order (rb_conv.cu). A block is the A operand (M = 128 output channels)
// in the K-major 128-byte-swizzle layout: output channel n is the 128-byte
// row n, input channel k (mod 64) sits in the 16-byte slot (k/8) ^ (n & 7)
// at element k % 8.
constexpr int kKChunk = 64;

std::vector<std::uint16_t> pack_blocks(const std::vector<double>& w, int C, int cin, int taps) {
  std::vector<std::uint16_t> out(static_cast<size_t>(taps) * cin * C);
  const size_t block = static_cast<size_t>(kKChunk) * C;
  for (int tap = 0; tap < taps; ++tap)
    for (int ci = 0; ci < cin; ++ci) {
      const int chunk = ci / kKChunk, k = ci % kKChunk;
      const size_t base = static_cast<size_t>(chunk * taps + tap) * block;
      for (int co = 0; co < C; ++co) {
        const size_t off = static_cast<size_t>(co) * kKChunk + static_cast<size_t>(((k / 8) ^ (co & 7)) * 8 + k % 8);
        out[base + off] = to_f16(w[(static_cast<size_t>(tap) * cin + ci) * C + co]);
      }
    }
  return out;
}

}  // namespace

void IepSession::init_resblock(const TensorBatch& inputs, std::uint64_t module_seed) {
  module_seed_ = module_seed;
  constexpr int C = 128;
  if (width_ != RB::kFmap) throw_error(Errc::width_mismatch, "resblock modules need width 25088 (128x14x14)");
  const HostCSR& c = batch_->csr();
  if (c.max_arity > 2) throw_error(Errc::arity_mismatch, "resblock modules support arity <= 2");
  rb_ = std::make_unique<RB>();
  RB& R = *rb_;
  check(dbk_rb_configure(), "step kernel attributes");
  for (std::int64_t g = 0; g < c.N; ++g)
    if (c.arity_of[static_cast<size_t>(c.fid[static_cast<size_t>(g)])] > 0) ++R.n_expensive;
  // Tile size: 256 positions, or 128 when a step has too few tiles to fill
  // the GPU (small batches are latency-bound: twice the tiles, each about
  // 60% as long). DYNBATCH_TILE_M overrides.
  {
    // the step count is d_max + 1 (longest root distance, host Kahn over the
    // CSR); s_max would undercount balanced trees' steps by far
    int d_max = 0;
    std::vector<std::int32_t> lab(static_cast<size_t>(c.N), 0), deg(static_cast<size_t>(c.N), 0), q;
    for (std::int32_t ch : c.child_list) ++deg[static_cast<size_t>(ch)];
    for (std::int64_t e = 0; e < c.b; ++e) {
      q.assign(1, c.root_g[static_cast<size_t>(e)]);
      for (size_t h = 0; h < q.size(); ++h) {
        const std::int32_t v = q[h];
        for (std::int32_t k = c.child_off[static_cast<size_t>(v)]; k < c.child_off[static_cast<size_t>(v) + 1]; ++k) {
          const std::int32_t u = c.child_list[static_cast<size_t>(k)];
          lab[static_cast<size_t>(u)] = std::max(lab[static_cast<size_t>(u)], lab[static_cast<size_t>(v)] + 1);
          if (--deg[static_cast<size_t>(u)] == 0) q.push_back(u);
        }
      }
      for (std::int32_t v : q) d_max = std::max(d_max, lab[static_cast<size_t>(v)]);
    }
    const double per_step = static_cast<double>(R.n_expensive) / (d_max + 1);
    const double tiles256 = per_step * 225.0 / RB::kTileM;
    R.tile_m = tiles256 < 2.0 * sm_count() ? 128 : RB::kTileM;
    if (const char* t = std::getenv("DYNBATCH_TILE_M")) {
      const int v = std::atoi(t);
      if (v == 64 || v == 128 || v == 256) R.tile_m = v;
    }
  }
  // buffers are sized for the session capacity (later set_programs batches)
  const size_t b = static_cast<size_t>(std::max<std::int64_t>(c.cap_b, 1));
  const size_t N = static_cast<size_t>(std::max<std::int64_t>(c.cap_N, 1));
  const std::int64_t n_exp_cap = std::max<std::int64_t>(R.n_expensive, c.cap_N - c.cap_b);  // trees: ≤ N − b
  R.inputs.alloc(b * RB::kFmap);
  R.values.alloc(N * RB::kFmap);
  R.chw_in.alloc(b * RB::kFmap);
  R.chw_out.alloc(b * RB::kFmap);
  // inputs: reference rows (CHW) → fp32 → plane maps
  std::vector<float> tmp(inputs.data().size());
  for (size_t i = 0; i < tmp.size(); ++i) tmp[i] = static_cast<float>(inputs.data()[i]);
  check(cudaMemcpyAsync(R.chw_in.get(), tmp.data(), tmp.size() * 4, cudaMemcpyHostToDevice, stream_), "H2D");
  check(dbk_rb_inputs_from_chw(c.b, R.chw_in.get(), R.inputs.get(), stream_), "inputs layout");
  // staging: every step owns its range (results are forwarded into their
  // parent's operand image); per group a kLead-row lead, ≤ one 256-position
  // alignment gap and ≤ one more tile to round it to whole tile pairs
  const std::int64_t max_groups = std::min<std::int64_t>(n_exp_cap, static_cast<std::int64_t>(std::max(1, c.cap_s)) * c.p);
  R.plane_stride = RB::kGuard + n_exp_cap * 225 + (2 * max_groups + 2) * (R.tile_m + RB::kLead) + 64;
  // forwarding eligibility: expensive nodes with exactly one parent
  {
    std::vector<std::int32_t> parents(static_cast<size_t>(N), 0), ok(static_cast<size_t>(N), 0);
    for (std::int32_t ch : c.child_list) ++parents[static_cast<size_t>(ch)];
    for (std::int64_t g = 0; g < c.N; ++g) {
      const bool exp = c.arity_of[static_cast<size_t>(c.fid[static_cast<size_t>(g)])] > 0;
      ok[static_cast<size_t>(g)] = exp && parents[static_cast<size_t>(g)] == 1;
      if (exp && parents[static_cast<size_t>(g)] > 1) R.n_shared += parents[static_cast<size_t>(g)];
    }
    R.fwd_ok.alloc(N);
    R.fwd_ok.upload(ok, stream_);
    R.fwd_pos.alloc(N);
    R.fwd_slot.alloc(N);
    R.fwd_parent.alloc(N);
    R.need.alloc(N);
    R.ready.alloc(N);
    R.memtab.alloc(N * 4);
    R.task_cap = std::max<std::int64_t>(static_cast<std::int64_t>(c.child_list.size()), c.cap_N) + 1;  // ≤ one task per operand
    R.tasks.alloc(static_cast<size_t>(R.task_cap) * 2 * 4);
    R.n_tasks.alloc(2);
  }
  const size_t ps = static_cast<size_t>(R.plane_stride);
  R.stage_x.alloc(ps * 16 * 8);
  R.stage_lo.alloc(ps * 16 * 8);
  R.stage_cat.alloc(ps * 32 * 8);
  R.stage_mid.alloc(ps * 16 * 8);
  R.stage_x.zero(stream_);
  R.stage_lo.zero(stream_);
  R.stage_cat.zero(stream_);
  R.stage_mid.zero(stream_);
  {  // identity weights: conv3x3 #2 adds the residual hi + lo on the tensor cores
    std::vector<double> eye(static_cast<size_t>(C) * C, 0.0);
    for (int c = 0; c < C; ++c) eye[static_cast<size_t>(c) * C + c] = 1.0;
    R.ident.upload(pack_blocks(eye, C, C, 1), stream_);
  }
  // schedule-derived tables (G ≤ max keys; tiles ≤ N_exp·225/256 + G)
  const size_t G = static_cast<size_t>(std::max(1, c.cap_s)) * c.p + 2;
  const size_t S = N + 2;  // naive: S = N
  const size_t T = static_cast<size_t>(n_exp_cap) * 225 / static_cast<size_t>(R.tile_m) + G + 2;
  R.seg_start.alloc(std::max(G, N + 2));
  R.group_tile0.alloc(std::max(G, N + 2));
  R.group_bintile0.alloc(std::max(G, N + 2));
  R.step_tile_begin.alloc(S);
  R.step_bintile_begin.alloc(S);
  R.step_positions.alloc(S + 1);
  R.tile_group.alloc(T + 2 * N);  // ≤ 2 tiles per group beyond the images (pairs)
  R.tile_q0.alloc(T + 2 * N);  // ≤ 2 tiles per group beyond the images (pairs)
  R.bin_group.alloc(T + 2 * N);  // ≤ 2 tiles per group beyond the images (pairs)
  R.bin_q0.alloc(T + 2 * N);  // ≤ 2 tiles per group beyond the images (pairs)
  R.done0.alloc(T + 2 * N);  // ≤ 2 tiles per group beyond the images (pairs)
  R.done1.alloc(T + 2 * N);  // ≤ 2 tiles per group beyond the images (pairs)
  R.done0.zero(stream_);
  R.done1.zero(stream_);
  R.order.alloc(3 * (T + 2 * N));
  R.order_prefix.alloc(T + 2 * N);
  R.queue.alloc(S + 1);
  R.step_done.alloc(S + 1);
  // weights
  std::vector<const void*> w0(static_cast<size_t>(c.p), nullptr), w1 = w0, w2 = w0;
  std::vector<const float*> b0(static_cast<size_t>(c.p), nullptr), b1 = b0, b2 = b0;
  for (int f = 0; f < c.p; ++f) {
    const int a = c.arity_of[static_cast<size_t>(f)];
    if (a == 0) continue;
    const ResBlockImpl m = make_resblock_impl(a, C, module_seed, f);
    auto put_w = [&](const std::vector<std::uint16_t>& v) {
      R.wbuf.emplace_back();
      R.wbuf.back().upload(v, stream_);
      return static_cast<const void*>(R.wbuf.back().get());
    };
    auto put_b = [&](const std::vector<double>& v) {
      std::vector<float> fv(v.begin(), v.end());
      R.bbuf.emplace_back();
      R.bbuf.back().upload(fv, stream_);
      return static_cast<const float*>(R.bbuf.back().get());
    };
    if (a == 2) {
      w0[static_cast<size_t>(f)] = put_w(pack_blocks(m.w0, C, 2 * C, 1));
      b0[static_cast<size_t>(f)] = put_b(m.b0);
    }
    w1[static_cast<size_t>(f)] = put_w(pack_blocks(m.w1, C, C, 9));
    b1[static_cast<size_t>(f)] = put_b(m.b1);
    w2[static_cast<size_t>(f)] = put_w(pack_blocks(m.w2, C, C, 9));
    b2[static_cast<size_t>(f)] = put_b(m.b2);
  }
  R.w0tab.upload(w0, stream_);
  R.w1tab.upload(w1, stream_);
  R.w2tab.upload(w2, stream_);
  R.b0tab.upload(b0, stream_);
  R.b1tab.upload(b1, stream_);
  R.b2tab.upload(b2, stream_);
}

namespace {
// DYNBATCH_STEP_LAUNCHES=1: one step-kernel launch per step (A/B timing)
bool per_step_launches() {
  static const bool v = [] {
    const char* e = std::getenv("DYNBATCH_STEP_LAUNCHES");
    return e && std::atoi(e) != 0;
  }();
  return v;
}
}  // namespace

void IepSession::forward_resblock() {
  RB& R = *rb_;
  DeviceProgramBatch& B = *batch_;
  const int S = B.steps;
  if (S == 0) return;
  const int sms = sm_count();
  // Every writer of a staged image writes its pads as zeros and the plan
  // zeroes the segment gaps, so a new layout (host schedule, set_programs)
  // needs no re-zeroing of the staging buffers.
  prof_.begin(1, stream_);
  check(dbk_rb_plan(S, B.step_group_begin.get(), B.group_fid.get(), B.group_begin.get(), B.arity_of.get(),
                    R.seg_start.get(), R.group_tile0.get(), R.group_bintile0.get(), R.step_tile_begin.get(),
                    R.step_bintile_begin.get(), R.step_positions.get(), R.tile_group.get(), R.tile_q0.get(),
                    R.bin_group.get(), R.bin_q0.get(), B.csr().N, B.member_g.get(), B.child0.get(),
                    B.child1.get(), R.fwd_ok.get(), R.fwd_pos.get(), R.fwd_slot.get(), R.fwd_parent.get(),
                    R.need.get(), R.tile_m, train_fwd_ ? 1 : 0, stream_),
        "dbk_rb_plan");
  check(dbk_rb_memtab(S, B.step_group_begin.get(), B.group_fid.get(), B.group_begin.get(), R.seg_start.get(),
                      B.member_g.get(), R.fwd_pos.get(), R.fwd_slot.get(), B.arity_of.get(), B.fid.get(),
                      B.child0.get(), B.child1.get(), B.example.get(), R.fwd_ok.get(), R.inputs.get(),
                      R.values.get(), R.memtab.get(), R.tasks.get(), R.n_tasks.get(), R.task_cap,
                      R.fwd_parent.get(), R.need.get(), R.tile_m, stream_),
        "dbk_rb_memtab");
  check(dbk_rb_order(S, R.step_tile_begin.get(), R.step_bintile_begin.get(), R.tile_group.get(), R.group_tile0.get(),
                     R.group_bintile0.get(), sms, R.order_prefix.get(), R.order.get(), stream_),
        "dbk_rb_order");
  check(dbk_rb_zero_gaps(S, B.step_group_begin.get(), B.group_begin.get(), R.seg_start.get(), R.stage_x.get(),
                         R.plane_stride, R.tile_m, stream_),
        "dbk_rb_zero_gaps");
  prof_.end(stream_);
  launches_ += 6;  // plan (+ tile lists), fwd init, fwd, memtab, claim order, zero gaps
  const int gather_blocks = sms * 16;  // grid-stride over the step's (member, operand, chunk, pixel) items
  check(cudaMemsetAsync(R.queue.get(), 0, sizeof(std::int32_t) * static_cast<size_t>(S), stream_), "queue reset");
  check(cudaMemsetAsync(R.step_done.get(), 0, sizeof(std::int32_t) * static_cast<size_t>(S), stream_),
        "step counters reset");
  // done flags are cleared every forward (the stamp is a constant), so a
  // captured forward replays as is
  check(cudaMemsetAsync(R.done0.get(), 0, sizeof(std::int32_t) * R.done0.size(), stream_), "done flags reset");
  check(cudaMemsetAsync(R.done1.get(), 0, sizeof(std::int32_t) * R.done1.size(), stream_), "done flags reset");
  check(cudaMemsetAsync(R.ready.get(), 0, sizeof(std::int32_t) * R.ready.size(), stream_), "image counters reset");
  R.epoch = 1;
  // leaf operands of every step in one launch (they only read the inputs)
  prof_.begin(2, stream_);
  check(dbk_rb_gather(R.tasks.get(), R.n_tasks.get(), 0, 0, R.task_cap, R.stage_x.get(), R.stage_lo.get(),
                      R.stage_cat.get(), R.plane_stride, err_.get(), gather_blocks, stream_),
        "dbk_rb_gather leaves");
  prof_.end(stream_);
  ++launches_;
  // All steps in one persistent launch (step s + 1 starts on each SM as soon
  // as step s is complete, with no launch gap, prologue or tail per step),
  // unless children shared by several parents need a gather between steps.
  const bool one_launch = R.n_shared == 0 && !per_step_launches();
  for (int s = 0; s < S; s = one_launch ? S : s + 1) {
    if (R.n_shared > 0) {  // children shared by several parents: values of earlier steps
      prof_.begin(2, stream_);
      check(dbk_rb_gather(R.tasks.get(), R.n_tasks.get(), 1, s, R.task_cap, R.stage_x.get(), R.stage_lo.get(),
                          R.stage_cat.get(), R.plane_stride, err_.get(), gather_blocks, stream_),
            "dbk_rb_gather shared");
      prof_.end(stream_);
      ++launches_;
    }
    // conv1x1 + conv3x3 #1 + conv3x3 #2 (+ residual) of the step(s), one launch
    prof_.begin(4, stream_);
    if (kevents_ && one_launch) {  // time_forwards(profile 2): the kernel's own events
      check(cudaEventRecordWithFlags(kev_cur_[0], stream_, cudaEventRecordExternal), "event");
      kev_recorded_ = true;
    }
    check(dbk_rb_step(s, one_launch ? S : s + 1, R.epoch, R.step_tile_begin.get(), R.tile_group.get(), R.tile_q0.get(),
                      R.step_bintile_begin.get(), R.bin_group.get(), R.bin_q0.get(), B.group_fid.get(),
                      B.group_begin.get(), R.seg_start.get(), R.group_tile0.get(), R.group_bintile0.get(),
                      R.memtab.get(), R.stage_x.get(), R.stage_lo.get(), R.stage_cat.get(), R.stage_mid.get(),
                      R.plane_stride, R.w0tab.get(), R.w1tab.get(), R.w2tab.get(), R.b0tab.get(), R.b1tab.get(),
                      R.b2tab.get(), R.ident.get(), R.done0.get(), R.done1.get(), R.step_done.get(), R.queue.get(), err_.get(),
                      R.ready.get(), R.need.get(), B.member_g.get(), R.order.get(), R.values.get(),
                      static_cast<std::int64_t>(R.values.size()), R.tile_m, sms, train_fwd_ ? 1 : 0, stream_),
          "conv step");
    if (kevents_ && one_launch) check(cudaEventRecordWithFlags(kev_cur_[1], stream_, cudaEventRecordExternal), "event");
    prof_.end(stream_);
    ++launches_;
  }
}

void IepSession::upload_resblock_inputs(const float* chw_rows) {
  RB& R = *rb_;
  const std::int64_t b = batch_->csr().b;
  check(cudaMemcpyAsync(R.chw_in.get(), chw_rows, sizeof(float) * static_cast<size_t>(b) * RB::kFmap,
                        cudaMemcpyHostToDevice, stream_), "H2D inputs");
  check(dbk_rb_inputs_from_chw(b, R.chw_in.get(), R.inputs.get(), stream_), "inputs layout");
}

// Root maps → reference rows (CHW) on the device, then one D2H copy. The
// layout pass belongs to the read-back, not to the forward.
void IepSession::download_resblock_outputs(float* chw_rows) {
  RB& R = *rb_;
  DeviceProgramBatch& B = *batch_;
  const std::int64_t b = B.csr().b;
  check(dbk_rb_outputs_to_chw(b, B.root_g.get(), B.fid.get(), B.arity_of.get(), B.example.get(), R.inputs.get(),
                              R.values.get(), R.chw_out.get(), stream_),
        "outputs layout");
  check(cudaMemcpyAsync(chw_rows, R.chw_out.get(), sizeof(float) * static_cast<size_t>(b) * RB::kFmap,
                        cudaMemcpyDeviceToHost, stream_), "D2H outputs");
  check(cudaStreamSynchronize(stream_), "sync");
}

void IepSession::forward_host(const float* inputs, float* outputs) {
  if (kind_ != ModuleKind::resblock) throw_error(Errc::invalid_argument, "forward_host needs a resblock session");
  upload_resblock_inputs(inputs);
  forward();
  download_resblock_outputs(outputs);
  check_errors();
}

// ------------------------------------------------------------ classifier head
void IepSession::set_head(int answers, std::uint64_t seed) {
  if (kind_ != ModuleKind::resblock) throw_error(Errc::invalid_argument, "the classifier head needs a resblock session");
  head_ = std::make_unique<IepHead>(answers, seed, stream_);
}

void IepSession::require_head() const {
  if (!head_) throw_error(Errc::invalid_argument, "no classifier head: call set_head first");
}

int IepSession::head_answers() const { return head_ ? head_->answers() : 0; }

double IepSession::head_flops() const {
  return head_ ? head_->flops_per_program() * static_cast<double>(batch_->csr().b) : 0.0;
}

void IepSession::head_forward() {
  require_head();
  flush_programs();
  DeviceProgramBatch& B = *batch_;
  RB& R = *rb_;
  launches_ += head_->forward(B.csr().b, B.root_g.get(), B.fid.get(), B.arity_of.get(), B.example.get(),
                              R.inputs.get(), R.values.get(), stream_);
}

void IepSession::download_logits(float* out, std::int64_t n) {
  require_head();
  const std::int64_t b = batch_->csr().b;
  if (n != b * head_->answers()) throw_error(Errc::row_count_mismatch, "logit buffer size");
  head_->download(b, out, stream_);
}

void IepSession::forward_logits_host(const float* inputs, float* logits) {
  require_head();
  upload_resblock_inputs(inputs);
  forward();
  head_forward();
  head_->download(batch_->csr().b, logits, stream_);
  check_errors();
}

double IepSession::time_head(int iters) {
  require_head();
  cudaEvent_t e0, e1;
  check(cudaEventCreate(&e0), "event");
  check(cudaEventCreate(&e1), "event");
  head_forward();  // warm (sizes the buffers)
  check(cudaEventRecord(e0, stream_), "event");
  for (int i = 0; i < iters; ++i) head_forward();
  check(cudaEventRecord(e1, stream_), "event");
  check(cudaEventSynchronize(e1), "sync");
  float ms = 0.f;
  check(cudaEventElapsedTime(&ms, e0, e1), "elapsed");
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return ms / std::max(iters, 1);
}

void IepSession::set_programs(const std::int32_t* tokens, const std::int32_t* seq_off, std::int64_t b) {
  if (kind_ != ModuleKind::resblock) throw_error(Errc::invalid_argument, "set_programs needs a resblock session");
  RB& R = *rb_;
  DeviceProgramBatch& B = *batch_;
  if (R.pipe) {
    // pipelined: stage the sequences in pinned memory; the next
    // forward_host_async uploads them with its inputs (one copy queue, no
    // small copy stuck behind a large one) and builds on the main stream
    RB::Pipe& Q = *R.pipe;
    const int k = static_cast<int>(Q.calls % RB::Pipe::kDepth);
    const std::int64_t N = B.begin_prefix_programs(seq_off, b);
    check(cudaEventSynchronize(Q.h2d_done[k]), "staging slot");  // the slot's last upload has finished
    Q.tok_pin[k].ensure(static_cast<size_t>(B.csr().cap_N));
    Q.off_pin[k].ensure(static_cast<size_t>(B.csr().cap_b) + 1);
    std::memcpy(Q.tok_pin[k].get(), tokens, sizeof(std::int32_t) * static_cast<size_t>(N));
    std::memcpy(Q.off_pin[k].get(), seq_off, sizeof(std::int32_t) * static_cast<size_t>(b + 1));
    Q.programs_pending = true;
  } else {
    B.set_prefix_programs(tokens, seq_off, b, stream_);
    programs_built();
  }
  const std::int64_t N = B.csr().N;
  host_tokens_.assign(tokens, tokens + N);
  host_seq_off_.assign(seq_off, seq_off + b + 1);
  mirror_stale_ = true;
}

void IepSession::programs_built() {
  RB& R = *rb_;
  DeviceProgramBatch& B = *batch_;
  check(cudaMemcpyAsync(R.fwd_ok.get(), B.fwd_ok.get(), sizeof(std::int32_t) * static_cast<size_t>(B.csr().N),
                        cudaMemcpyDeviceToDevice, stream_), "fwd_ok");
  R.n_shared = 0;  // prefix sequences describe trees: no child has two parents
  if (host_schedule_) {  // a host schedule described the old programs
    host_schedule_ = false;
    strategy_ = Strategy::improved;
  }
}

// A plain forward() after a pipelined set_programs: upload the staged
// sequences on the main stream and build.
void IepSession::flush_programs() {
  if (!rb_ || !rb_->pipe || !rb_->pipe->programs_pending) return;
  RB::Pipe& Q = *rb_->pipe;
  DeviceProgramBatch& B = *batch_;
  const int k = static_cast<int>(Q.calls % RB::Pipe::kDepth);
  Q.tok[k].ensure(static_cast<size_t>(B.csr().cap_N));
  Q.off[k].ensure(static_cast<size_t>(B.csr().cap_b) + 1);
  check(cudaMemcpyAsync(Q.tok[k].get(), Q.tok_pin[k].get(), sizeof(std::int32_t) * static_cast<size_t>(B.csr().N),
                        cudaMemcpyHostToDevice, stream_), "H2D tokens");
  check(cudaMemcpyAsync(Q.off[k].get(), Q.off_pin[k].get(), sizeof(std::int32_t) * static_cast<size_t>(B.csr().b + 1),
                        cudaMemcpyHostToDevice, stream_), "H2D offsets");
  B.build_prefix_programs(Q.tok[k].get(), Q.off[k].get(), stream_);
  programs_built();
  Q.programs_pending = false;
  // the pinned slot is reused by a later set_programs only after this slot's
  // h2d_done: record it here, after the copies
  check(cudaEventRecord(Q.h2d_done[k], stream_), "event");
}

// Host CSR arrays of the programs last set on the device (schedule download,
// profiling): rebuilt from the host copies of the sequences on demand.
void IepSession::ensure_host_mirror() {
  if (!mirror_stale_) return;
  std::vector<Program> progs;
  progs.reserve(host_seq_off_.size() - 1);
  for (size_t e = 0; e + 1 < host_seq_off_.size(); ++e) {
    const std::span<const int> seq(host_tokens_.data() + host_seq_off_[e],
                                   static_cast<size_t>(host_seq_off_[e + 1] - host_seq_off_[e]));
    progs.push_back(build_program_from_prefix(seq, vocab_));
  }
  batch_->replace_host_csr(make_csr(progs, vocab_));
  mirror_stale_ = false;
}

void IepSession::sync_pipeline() {
  if (!rb_ || !rb_->pipe) return;
  RB::Pipe& Q = *rb_->pipe;
  check(cudaStreamSynchronize(Q.h2d), "sync h2d");
  check(cudaStreamSynchronize(Q.d2h), "sync d2h");
  if (Q.trace && !Q.tev.empty()) {
    const cudaEvent_t base = Q.tev.front()[0];
    for (size_t c = 0; c < Q.tev.size(); ++c) {
      float t[6] = {-1, -1, -1, -1, -1, -1};
      for (int i = 0; i < 6; ++i) {
        const cudaError_t err = cudaEventElapsedTime(&t[i], base, Q.tev[c][static_cast<size_t>(i)]);
        if (err != cudaSuccess) {
          t[i] = -1;
          cudaGetLastError();
        }
      }
      std::fprintf(stderr, "call %zu: h2d %.2f-%.2f  main %.2f-%.2f  d2h %.2f-%.2f ms\n", c, t[0], t[1], t[2], t[3],
                   t[4], t[5]);
    }
    for (auto& te : Q.tev)
      for (auto e : te) cudaEventDestroy(e);
    Q.tev.clear();
    Q.trace = false;
  }
}

// Pipelined end-to-end call: the H2D of this call's inputs and the D2H of
// its outputs run on their own streams into triple-buffered device rows, so
// consecutive calls overlap upload(N+1) and download(N−1) with forward(N)
// (PCIe is full duplex). Ordering is by events only; synchronize() waits for
// everything. Host buffers must stay valid (and should be pinned) until then.
void IepSession::forward_host_async(const float* inputs, float* outputs) {
  if (kind_ != ModuleKind::resblock) throw_error(Errc::invalid_argument, "forward_host needs a resblock session");
  RB& R = *rb_;
  DeviceProgramBatch& B = *batch_;
  const std::int64_t b = B.csr().b;
  const size_t bytes = sizeof(float) * static_cast<size_t>(b) * RB::kFmap;
  if (!R.pipe) {
    R.pipe = std::make_unique<RB::Pipe>();
    RB::Pipe& Q = *R.pipe;
    check(cudaStreamCreateWithFlags(&Q.h2d, cudaStreamNonBlocking), "stream");
    check(cudaStreamCreateWithFlags(&Q.d2h, cudaStreamNonBlocking), "stream");
    const size_t rows = static_cast<size_t>(std::max<std::int64_t>(B.csr().cap_b, b));
    for (int k = 0; k < RB::Pipe::kDepth; ++k) {
      Q.in[k].alloc(rows * RB::kFmap);
      Q.out[k].alloc(rows * RB::kFmap);
      for (cudaEvent_t* e : {&Q.h2d_done[k], &Q.in_free[k], &Q.out_ready[k], &Q.out_free[k]}) {
        check(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event");
        check(cudaEventRecord(*e, stream_), "event");
      }
    }
  }
  RB::Pipe& Q = *R.pipe;
  const int k = static_cast<int>(Q.calls++ % RB::Pipe::kDepth);
  std::array<cudaEvent_t, 6> te{};
  if (Q.trace || std::getenv("DYNBATCH_PIPE_TRACE")) {
    Q.trace = true;
    for (auto& e : te) check(cudaEventCreate(&e), "event");
    Q.tev.push_back(te);
  }
  auto mark = [&](int i, cudaStream_t st) {
    if (Q.trace) check(cudaEventRecord(te[static_cast<size_t>(i)], st), "event");
  };
  check(cudaStreamWaitEvent(Q.h2d, Q.in_free[k]), "wait");
  mark(0, Q.h2d);
  const bool build = Q.programs_pending;
  if (build) {  // sequences staged by set_programs ride this call's upload
    Q.tok[k].ensure(static_cast<size_t>(B.csr().cap_N));
    Q.off[k].ensure(static_cast<size_t>(B.csr().cap_b) + 1);
    check(cudaMemcpyAsync(Q.tok[k].get(), Q.tok_pin[k].get(), sizeof(std::int32_t) * static_cast<size_t>(B.csr().N),
                          cudaMemcpyHostToDevice, Q.h2d), "H2D tokens");
    check(cudaMemcpyAsync(Q.off[k].get(), Q.off_pin[k].get(), sizeof(std::int32_t) * static_cast<size_t>(b + 1),
                          cudaMemcpyHostToDevice, Q.h2d), "H2D offsets");
    Q.programs_pending = false;
  }
  check(cudaMemcpyAsync(Q.in[k].get(), inputs, bytes, cudaMemcpyHostToDevice, Q.h2d), "H2D inputs");
  mark(1, Q.h2d);
  check(cudaEventRecord(Q.h2d_done[k], Q.h2d), "event");
  check(cudaStreamWaitEvent(stream_, Q.h2d_done[k]), "wait");
  mark(2, stream_);
  if (build) {
    B.build_prefix_programs(Q.tok[k].get(), Q.off[k].get(), stream_);
    programs_built();
  }
  check(dbk_rb_inputs_from_chw(b, Q.in[k].get(), R.inputs.get(), stream_), "inputs layout");
  check(cudaEventRecord(Q.in_free[k], stream_), "event");
  forward();
  mark(3, stream_);
  check(cudaStreamWaitEvent(stream_, Q.out_free[k]), "wait");
  check(dbk_rb_outputs_to_chw(b, B.root_g.get(), B.fid.get(), B.arity_of.get(), B.example.get(), R.inputs.get(),
                              R.values.get(), Q.out[k].get(), stream_),
        "outputs layout");
  check(cudaEventRecord(Q.out_ready[k], stream_), "event");
  check(cudaStreamWaitEvent(Q.d2h, Q.out_ready[k]), "wait");
  mark(4, Q.d2h);
  check(cudaMemcpyAsync(outputs, Q.out[k].get(), bytes, cudaMemcpyDeviceToHost, Q.d2h), "D2H outputs");
  mark(5, Q.d2h);
  check(cudaEventRecord(Q.out_free[k], Q.d2h), "event");
}

}  // namespace dynbatch::dev
