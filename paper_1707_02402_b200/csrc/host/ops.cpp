// ops.cpp — module registry, executor and MoE operator API (device-backed).
//
//   make_module_impl / ModuleSet ... src/modules.cpp:13-50
//   apply_module ................... src/modules.cpp:52-108 (runs on device)
//   ValueStore, gather/scatter_rows  src/executor.cpp:26-93 (host containers)
//   execute ........................ src/executor.cpp:95-182 (runs on device)
//   MoeConfig::check ............... src/moe.cpp:20-28
//   top_k_gate ..................... src/moe.cpp:36-69 (runs on device)
//   ExpertSet (+ apply on device) .. src/moe.cpp:71-145
//   moe_forward_{naive,batched} .... src/moe.cpp:162-270 (run on device)
//   memory model ................... src/moe.cpp:272-289
#include <algorithm>
#include <chrono>
#include <cmath>

#include "device.hpp"
#include "dynbatch/dbk.h"
#include "dynbatch.hpp"

namespace dynbatch {

ModuleImpl make_module_impl(const ModuleSpec& spec, int width, std::uint64_t seed) {
  ModuleImpl impl;
  impl.spec = spec;
  if (spec.arity == 0) return impl;
  const int fan_in = spec.arity * width;
  const double scale = 1.0 / std::sqrt(static_cast<double>(fan_in));
  Rng rng(mix_seed(seed, static_cast<std::uint64_t>(spec.function_id)));
  impl.weights.resize(static_cast<size_t>(fan_in) * static_cast<size_t>(width));
  for (double& w : impl.weights) w = rng.uniform(-0.5, 0.5) * scale;
  impl.bias.resize(static_cast<size_t>(width));
  for (double& b : impl.bias) b = rng.uniform(-0.5, 0.5) * scale;
  return impl;
}

ModuleSet::ModuleSet(const FunctionVocab& vocab, std::uint64_t seed) : width_(vocab.width()), seed_(seed) {
  for (const ModuleSpec& s : vocab.specs()) impls_.push_back(make_module_impl(s, width_, seed));
}

const ModuleImpl& ModuleSet::impl(int fid) const {
  if (fid < 0 || fid >= size()) throw_error(Errc::unknown_function, "function id " + std::to_string(fid));
  return impls_[static_cast<size_t>(fid)];
}

std::int64_t ModuleSet::weight_element_count() const {
  std::int64_t n = 0;
  for (const ModuleImpl& m : impls_) n += static_cast<std::int64_t>(m.weights.size() + m.bias.size());
  return n;
}

ResBlockImpl make_resblock_impl(int arity, int C, std::uint64_t seed, int fid) {
  ResBlockImpl m;
  m.arity = arity;
  if (arity == 0) return m;
  Rng rng(mix_seed(seed, static_cast<std::uint64_t>(fid)));
  const auto fill = [&rng](std::vector<double>& v, size_t n, double scale) {
    v.resize(n);
    for (double& x : v) x = rng.uniform(-0.5, 0.5) * scale;
  };
  const size_t CC = static_cast<size_t>(C) * C;
  if (arity == 2) {
    const double s0 = 1.0 / std::sqrt(2.0 * C);
    fill(m.w0, 2 * CC, s0);
    fill(m.b0, static_cast<size_t>(C), s0);
  }
  const double s = 1.0 / std::sqrt(9.0 * C);
  fill(m.w1, 9 * CC, s);
  fill(m.b1, static_cast<size_t>(C), s);
  fill(m.w2, 9 * CC, s);
  fill(m.b2, static_cast<size_t>(C), s);
  return m;
}

namespace {
// Trace counters from a schedule exactly as execute() accumulates them
// (src/executor.cpp:119-124): per group, leaf groups included.
ExecutionTrace count_trace(const Schedule& schedule, const FunctionVocab& vocab) {
  ExecutionTrace t;
  t.per_function_calls.assign(static_cast<size_t>(vocab.size()), 0);
  for (const Step& st : schedule.steps) {
    for (const CallGroup& g : st) {
      const ModuleSpec& spec = vocab.spec(g.function_id);
      t.peak_group_rows = std::max<std::int64_t>(t.peak_group_rows, static_cast<std::int64_t>(g.members.size()));
      ++t.per_function_calls[static_cast<size_t>(g.function_id)];
      if (spec.is_expensive()) ++t.expensive_calls;
    }
  }
  t.per_step_seconds.assign(schedule.steps.size(), 0.0);
  return t;
}
}  // namespace

ExecResult execute(const Schedule& schedule, std::span<const Program> batch,
                   const TensorBatch& inputs, const ModuleSet& modules) {
  const FunctionVocab vocab = [&] {
    std::vector<ModuleSpec> specs;
    for (int f = 0; f < modules.size(); ++f) specs.push_back(modules.impl(f).spec);
    return FunctionVocab(std::move(specs));
  }();
  const auto t0 = std::chrono::steady_clock::now();
  dev::IepSession session(vocab, batch, inputs, modules.seed(), dev::ModuleKind::dense);
  session.set_schedule(&schedule);
  const auto t1 = std::chrono::steady_clock::now();
  session.forward();
  ExecResult r;
  r.outputs = session.download_outputs();
  const auto t2 = std::chrono::steady_clock::now();
  r.trace = count_trace(schedule, vocab);
  r.trace.module_seconds = std::chrono::duration<double>(t2 - t1).count();
  r.trace.stacking_seconds = std::chrono::duration<double>(t1 - t0).count();
  r.trace.total_seconds = std::chrono::duration<double>(t2 - t0).count();
  return r;
}

ExecResult execute(const Schedule& schedule, std::span<const Program> batch,
                   const TensorBatch& inputs, const FunctionVocab& vocab, std::uint64_t seed) {
  return execute(schedule, batch, inputs, ModuleSet(vocab, seed));
}

// ------------------------------------------------------------------- MoE
void MoeConfig::check() const {
  if (experts < 1) throw_error(Errc::invalid_argument, "need at least one expert");
  if (active_per_example < 1 || active_per_example > experts) {
    throw_error(Errc::invalid_argument, "k must satisfy 1 <= k <= n");
  }
  if (batch < 1) throw_error(Errc::invalid_argument, "batch must be >= 1");
  if (data_dim < 1 || hidden < 1) throw_error(Errc::invalid_argument, "dims must be >= 1");
  if (examples_per_expert < 0) throw_error(Errc::invalid_argument, "m must be >= 0");
}

ExpertSet::ExpertSet(std::int64_t experts, std::int64_t data_dim, std::int64_t hidden, std::uint64_t seed)
    : data_dim_(data_dim), hidden_(hidden), seed_(seed) {
  if (experts < 1 || data_dim < 1 || hidden < 1) throw_error(Errc::invalid_argument, "expert set dims must be >= 1");
  const double s1 = 1.0 / std::sqrt(static_cast<double>(data_dim));
  const double s2 = 1.0 / std::sqrt(static_cast<double>(hidden));
  experts_.resize(static_cast<size_t>(experts));
  for (std::int64_t id = 0; id < experts; ++id) {
    Rng rng(mix_seed(seed, static_cast<std::uint64_t>(id)));
    Expert& ex = experts_[static_cast<size_t>(id)];
    ex.w1.resize(static_cast<size_t>(data_dim * hidden));
    for (double& w : ex.w1) w = rng.uniform(-0.5, 0.5) * s1;
    ex.w2.resize(static_cast<size_t>(hidden * data_dim));
    for (double& w : ex.w2) w = rng.uniform(-0.5, 0.5) * s2;
  }
}

std::int64_t ExpertSet::weight_element_count() const {
  std::int64_t n = 0;
  for (const Expert& e : experts_) n += static_cast<std::int64_t>(e.w1.size() + e.w2.size());
  return n;
}

std::int64_t moe_param_count(const MoeConfig& cfg) {
  cfg.check();
  return 2 * cfg.hidden * cfg.experts * cfg.data_dim;
}

double moe_activation_count(const MoeConfig& cfg) {
  cfg.check();
  return static_cast<double>(cfg.experts) * cfg.examples_per_expert *
         static_cast<double>(2 * cfg.data_dim + cfg.hidden) / static_cast<double>(cfg.active_per_example);
}

double moe_memory_ratio(const MoeConfig& cfg) {
  cfg.check();
  return cfg.examples_per_expert * static_cast<double>(2 * cfg.data_dim + cfg.hidden) /
         (2.0 * static_cast<double>(cfg.active_per_example) * static_cast<double>(cfg.hidden) *
          static_cast<double>(cfg.data_dim));
}

// ------------------------------------------------- operator-level API
namespace {
std::string ref_text(NodeRef r) {
  return "(" + std::to_string(r.example) + ", " + std::to_string(r.node) + ")";
}

// Device copies for one operator call; the result comes back to the host.
struct DeviceCall {
  cudaStream_t s = nullptr;
  DeviceCall() {
    dev::require_device();
    dev::check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
  }
  ~DeviceCall() {
    if (s) cudaStreamDestroy(s);
  }
};
}  // namespace

ValueStore::ValueStore(std::span<const Program> batch, std::int64_t width) : width_(width) {
  if (width <= 0) throw_error(Errc::invalid_argument, "width must be positive");
  for (const Program& p : batch) {
    values_.emplace_back(static_cast<size_t>(p.size()) * static_cast<size_t>(width), 0.0);
    present_.emplace_back(static_cast<size_t>(p.size()), 0);
  }
}

void ValueStore::check_ref(NodeRef ref) const {
  const bool ok = ref.example >= 0 && static_cast<size_t>(ref.example) < present_.size() && ref.node >= 0 &&
                  static_cast<size_t>(ref.node) < present_[static_cast<size_t>(ref.example)].size();
  if (!ok) throw_error(Errc::invalid_argument, "node ref out of range " + ref_text(ref));
}

bool ValueStore::has(NodeRef ref) const {
  check_ref(ref);
  return present_[static_cast<size_t>(ref.example)][static_cast<size_t>(ref.node)] != 0;
}

std::span<const double> ValueStore::row(NodeRef ref) const {
  if (!has(ref)) throw_error(Errc::missing_operand, "no value for node " + ref_text(ref));
  return {values_[static_cast<size_t>(ref.example)].data() + static_cast<size_t>(ref.node) * width_,
          static_cast<size_t>(width_)};
}

void ValueStore::set(NodeRef ref, std::span<const double> value) {
  check_ref(ref);
  if (static_cast<std::int64_t>(value.size()) != width_)
    throw_error(Errc::width_mismatch, "row width " + std::to_string(value.size()));
  char& here = present_[static_cast<size_t>(ref.example)][static_cast<size_t>(ref.node)];
  if (here) throw_error(Errc::single_assignment_violation, "node " + ref_text(ref) + " written twice");
  std::copy(value.begin(), value.end(),
            values_[static_cast<size_t>(ref.example)].begin() + static_cast<std::ptrdiff_t>(ref.node * width_));
  here = 1;
}

TensorBatch gather_rows(const ValueStore& store, std::span<const NodeRef> refs) {
  TensorBatch out(static_cast<std::int64_t>(refs.size()), store.width());
  for (size_t i = 0; i < refs.size(); ++i) {
    const auto src = store.row(refs[i]);
    std::copy(src.begin(), src.end(), out.row(static_cast<std::int64_t>(i)).begin());
  }
  return out;
}

void scatter_rows(ValueStore& store, std::span<const NodeRef> refs, const TensorBatch& values) {
  if (values.rows() != static_cast<std::int64_t>(refs.size()))
    throw_error(Errc::row_count_mismatch,
                std::to_string(values.rows()) + " rows for " + std::to_string(refs.size()) + " refs");
  if (values.width() != store.width())
    throw_error(Errc::width_mismatch, "value width " + std::to_string(values.width()));
  for (size_t i = 0; i < refs.size(); ++i) store.set(refs[i], values.row(static_cast<std::int64_t>(i)));
}

// One module call on stacked operand rows, on the device (dbk_dense_apply:
// the executor's fp64 fma chain, so the bits match execute() and the
// reference). Shape errors as the reference (src/modules.cpp:53-73).
TensorBatch apply_module(const ModuleImpl& impl, std::span<const TensorBatch> operands) {
  const int arity = impl.spec.arity;
  if (arity == 0) throw_error(Errc::arity_mismatch, "arity-0 functions fetch inputs, they are not applied");
  if (static_cast<int>(operands.size()) != arity)
    throw_error(Errc::arity_mismatch, "function " + std::to_string(impl.spec.function_id) + " expects " +
                                          std::to_string(arity) + " operands, got " +
                                          std::to_string(operands.size()));
  const std::int64_t rows = operands[0].rows();
  const std::int64_t width = impl.spec.out_width;
  for (const TensorBatch& op : operands) {
    if (op.rows() != rows) throw_error(Errc::row_count_mismatch, "operand row counts differ");
    if (op.width() != width)
      throw_error(Errc::width_mismatch,
                  "operand width " + std::to_string(op.width()) + ", expected " + std::to_string(width));
  }
  TensorBatch out(rows, width);
  if (rows == 0) return out;
  std::vector<double> x(static_cast<size_t>(rows * arity * width));
  for (std::int64_t r = 0; r < rows; ++r)
    for (int k = 0; k < arity; ++k) {
      const auto src = operands[static_cast<size_t>(k)].row(r);
      std::copy(src.begin(), src.end(), x.begin() + static_cast<std::ptrdiff_t>((r * arity + k) * width));
    }
  DeviceCall call;
  dev::Buf<double> dx, dw, db, dout;
  dx.upload(x, call.s);
  dw.upload(impl.weights, call.s);
  db.upload(impl.bias, call.s);
  dout.alloc(static_cast<size_t>(rows * width));
  dev::check(dbk_dense_apply(rows, arity, static_cast<std::int32_t>(width), dx.get(), dw.get(), db.get(), dout.get(),
                             call.s),
             "dbk_dense_apply");
  const auto y = dout.download(static_cast<size_t>(rows * width), call.s);
  std::copy(y.begin(), y.end(), out.data().begin());
  return out;
}

// One expert on stacked rows (src/moe.cpp:98-145), on the device through the
// MoE fp64 expert kernels (one expert, the identity order).
TensorBatch ExpertSet::apply(std::int64_t expert_id, const TensorBatch& rows) const {
  if (expert_id < 0 || expert_id >= size()) throw_error(Errc::invalid_argument, "expert id " + std::to_string(expert_id));
  if (rows.width() != data_dim_)
    throw_error(Errc::width_mismatch, "expert input width " + std::to_string(rows.width()));
  const std::int64_t n = rows.rows();
  TensorBatch out(n, data_dim_);
  if (n == 0) return out;
  const Expert& ex = experts_[static_cast<size_t>(expert_id)];
  DeviceCall call;
  std::vector<std::int32_t> order(static_cast<size_t>(n));
  for (std::int64_t i = 0; i < n; ++i) order[static_cast<size_t>(i)] = static_cast<std::int32_t>(i);
  const std::vector<std::int32_t> offsets{0, static_cast<std::int32_t>(n)};
  dev::Buf<double> dx, dw1, dw2, hidden, staged;
  dev::Buf<std::int32_t> dorder, doff, tiles;
  dev::Buf<const double*> w1tab, w2tab;
  dx.upload(rows.data().data(), rows.data().size(), call.s);
  dw1.upload(ex.w1, call.s);
  dw2.upload(ex.w2, call.s);
  w1tab.upload(std::vector<const double*>{dw1.get()}, call.s);
  w2tab.upload(std::vector<const double*>{dw2.get()}, call.s);
  dorder.upload(order, call.s);
  doff.upload(offsets, call.s);
  tiles.alloc(2);
  hidden.alloc(static_cast<size_t>(n * hidden_));
  staged.alloc(static_cast<size_t>(n * data_dim_));
  dev::check(dbk_moe_expert_fp64(n, 1, 1, static_cast<std::int32_t>(data_dim_), static_cast<std::int32_t>(hidden_),
                                 dorder.get(), doff.get(), dx.get(), w1tab.get(), w2tab.get(), hidden.get(),
                                 staged.get(), tiles.get(), call.s),
             "dbk_moe_expert_fp64");
  const auto y = staged.download(static_cast<size_t>(n * data_dim_), call.s);
  std::copy(y.begin(), y.end(), out.data().begin());
  return out;
}

}  // namespace dynbatch
