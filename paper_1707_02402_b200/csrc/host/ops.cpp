// ops.cpp — module registry, executor and MoE operator API (device-backed).
//
//   make_module_impl / ModuleSet ... src/modules.cpp:13-50
//   execute ........................ src/executor.cpp:95-182 (runs on device)
//   MoeConfig::check ............... src/moe.cpp:20-28
//   top_k_gate ..................... src/moe.cpp:36-69 (runs on device)
//   ExpertSet ...................... src/moe.cpp:71-96
//   moe_forward_{naive,batched} .... src/moe.cpp:162-270 (run on device)
//   memory model ................... src/moe.cpp:272-289
#include <algorithm>
#include <chrono>
#include <cmath>

#include "device.hpp"
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

}  // namespace dynbatch
