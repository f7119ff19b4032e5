// c_api.cpp — the drop-in C ABI (include/dynbatch/dynbatch.h) and its device
// extensions (include/dynbatch/dynbatch_device.h).
//
// Handle layout, error mapping and ownership follow the reference
// (src/c_api.cpp:19-336): status_from maps Errc → db_status (:38-60; shape
// errors collapse to DB_ERR_SHAPE_MISMATCH, single-assignment violations are
// DB_ERR_INTERNAL), guarded() turns exceptions into statuses and the
// thread-local db_last_error() text (:62-78), NULL arguments give
// DB_ERR_INVALID_ARG (:80-83), accessors return -1 on NULL (:184-186).
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "device.hpp"
#include "ep_nccl.hpp"
#include "dynbatch.hpp"
#include "dynbatch/dynbatch.h"
#include "dynbatch/dynbatch_device.h"
#include "dynbatch/dbk.h"

struct db_batch {
  dynbatch::FunctionVocab vocab;
  std::vector<dynbatch::Program> programs;
  dynbatch::TensorBatch inputs;
};

struct db_schedule {
  dynbatch::Schedule schedule;
};

struct db_run {
  dynbatch::TensorBatch outputs;
  dynbatch::ExecutionTrace trace;
};

struct db_iep_session {
  std::unique_ptr<dynbatch::dev::IepSession> s;
};

struct db_moe_session {
  std::unique_ptr<dynbatch::dev::MoeSession> s;
};

struct db_moe_ep_session {
  std::unique_ptr<dynbatch::dev::MoeEp> s;
};

namespace {

using dynbatch::Errc;

thread_local std::string t_error;

db_status to_status(Errc c) {
  switch (c) {
    case Errc::ok: return DB_OK;
    case Errc::invalid_argument: return DB_ERR_INVALID_ARG;
    case Errc::unknown_function: return DB_ERR_UNKNOWN_FUNCTION;
    case Errc::underfull_sequence: return DB_ERR_UNDERFULL_SEQUENCE;
    case Errc::overfull_sequence: return DB_ERR_OVERFULL_SEQUENCE;
    case Errc::invalid_program: return DB_ERR_INVALID_PROGRAM;
    case Errc::dependency_violation: return DB_ERR_DEPENDENCY_VIOLATION;
    case Errc::missing_operand: return DB_ERR_MISSING_OPERAND;
    case Errc::row_count_mismatch:
    case Errc::width_mismatch:
    case Errc::arity_mismatch:
    case Errc::k_too_large:
    case Errc::vocab_missing_arity: return DB_ERR_SHAPE_MISMATCH;
    case Errc::non_finite_value: return DB_ERR_NON_FINITE;
    case Errc::parse_error: return DB_ERR_PARSE;
    case Errc::verification_failed: return DB_ERR_VERIFICATION_FAILED;
    case Errc::single_assignment_violation: break;
  }
  return DB_ERR_INTERNAL;
}

template <class Fn>
db_status guarded(Fn&& fn) {
  try {
    fn();
    t_error.clear();
    return DB_OK;
  } catch (const dynbatch::Error& e) {
    t_error = e.what();
    return to_status(e.code());
  } catch (const std::exception& e) {
    t_error = e.what();
    return DB_ERR_INTERNAL;
  } catch (...) {
    t_error = "unknown error";
    return DB_ERR_INTERNAL;
  }
}

db_status null_arg() {
  t_error = "null argument";
  return DB_ERR_INVALID_ARG;
}

char* dup_string(const std::string& s) {
  char* out = new char[s.size() + 1];
  std::memcpy(out, s.c_str(), s.size() + 1);
  return out;
}

dynbatch::Strategy to_strategy(db_strategy s) {
  switch (s) {
    case DB_STRATEGY_NAIVE: return dynbatch::Strategy::naive;
    case DB_STRATEGY_STANDARD: return dynbatch::Strategy::standard;
    case DB_STRATEGY_IMPROVED: return dynbatch::Strategy::improved;
    case DB_STRATEGY_ONLINE: return dynbatch::Strategy::online;
  }
  dynbatch::throw_error(Errc::invalid_argument, "unknown strategy");
}

dynbatch::MoeConfig to_cfg(const db_moe_opts* o) {
  dynbatch::MoeConfig c;
  c.experts = o->experts;
  c.active_per_example = o->active_per_example;
  c.batch = o->batch;
  c.data_dim = o->data_dim;
  c.hidden = o->hidden;
  c.check();
  return c;
}

dynbatch::dev::ModuleKind to_kind(const db_module_opts* o) {
  if (!o || o->module_kind == DB_MODULE_DENSE) return dynbatch::dev::ModuleKind::dense;
  if (o->module_kind != DB_MODULE_RESBLOCK) dynbatch::throw_error(Errc::invalid_argument, "unknown module kind");
  if (o->channels != 128 || o->height != 14 || o->width_px != 14) {
    dynbatch::throw_error(Errc::invalid_argument, "resblock modules are built for 128x14x14 maps");
  }
  return dynbatch::dev::ModuleKind::resblock;
}

void fill_stats(db_session_stats_t* out, const dynbatch::ExecutionTrace& t, std::int64_t steps,
                std::int64_t groups, std::int64_t members, std::int64_t launches, std::int64_t h2d,
                std::int64_t d2h, double flops, double bytes) {
  out->steps = steps;
  out->groups = groups;
  out->expensive_calls = t.expensive_calls;
  out->peak_group_rows = t.peak_group_rows;
  out->members = members;
  out->kernel_launches = launches;
  out->h2d_bytes = h2d;
  out->d2h_bytes = d2h;
  out->algorithmic_flops = flops;
  out->algorithmic_bytes = bytes;
}

}  // namespace

extern "C" {

const char* db_version(void) { return "0.1.0-b200"; }
const char* db_last_error(void) { return t_error.c_str(); }
void db_string_free(char* text) { delete[] text; }

db_status db_batch_generate(const db_workload_opts* opts, db_batch** out) {
  if (!opts || !out) return null_arg();
  return guarded([&] {
    dynbatch::WorkloadSpec spec;
    switch (opts->kind) {
      case DB_WORKLOAD_BALANCED_TREE: spec.kind = dynbatch::WorkloadKind::balanced_tree; break;
      case DB_WORKLOAD_CHAIN_HEAVY: spec.kind = dynbatch::WorkloadKind::chain_heavy; break;
      case DB_WORKLOAD_RANDOM_DAG: spec.kind = dynbatch::WorkloadKind::random_dag; break;
      default: dynbatch::throw_error(Errc::invalid_argument, "unknown workload kind");
    }
    spec.b = opts->batch;
    spec.p = opts->vocab;
    spec.width = opts->width;
    spec.depth = opts->depth;
    spec.length = opts->length;
    spec.branch_prob = opts->branch_prob;
    spec.seed = opts->seed;
    dynbatch::GeneratedBatch g = dynbatch::gen_batch(spec);
    *out = new db_batch{std::move(g.vocab), std::move(g.programs), std::move(g.inputs)};
  });
}

db_status db_batch_load_json(const char* text, int32_t width, uint64_t input_seed, db_batch** out) {
  if (!text || !out) return null_arg();
  return guarded([&] {
    dynbatch::ProgramSet set = dynbatch::program_set_from_json(text, width);
    dynbatch::TensorBatch in = dynbatch::random_batch(static_cast<std::int64_t>(set.programs.size()), width, input_seed);
    *out = new db_batch{std::move(set.vocab), std::move(set.programs), std::move(in)};
  });
}

db_status db_batch_to_json(const db_batch* batch, char** out_text) {
  if (!batch || !out_text) return null_arg();
  return guarded([&] { *out_text = dup_string(dynbatch::program_set_to_json(batch->vocab, batch->programs)); });
}

db_status db_batch_stats(const db_batch* batch, db_batch_stats_t* out) {
  if (!batch || !out) return null_arg();
  return guarded([&] {
    const dynbatch::BatchStats st = dynbatch::compute_batch_stats(batch->programs, batch->vocab);
    out->batch = st.b;
    out->vocab = st.p;
    out->width = batch->vocab.width();
    out->s_max = st.s_max;
    out->d_max = st.d_max;
    out->total_nodes = dynbatch::count_total_nodes(batch->programs);
    out->expensive_nodes = dynbatch::count_expensive_nodes(batch->programs, batch->vocab);
  });
}

void db_batch_free(db_batch* batch) { delete batch; }

db_status db_schedule_build(const db_batch* batch, db_strategy strategy, db_schedule** out) {
  if (!batch || !out) return null_arg();
  return guarded([&] {
    *out = new db_schedule{dynbatch::build_schedule(to_strategy(strategy), batch->programs, batch->vocab)};
  });
}

db_status db_schedule_build_device(const db_batch* batch, db_strategy strategy, db_schedule** out) {
  if (!batch || !out) return null_arg();
  return guarded([&] {
    *out = new db_schedule{dynbatch::schedule_device(to_strategy(strategy), batch->programs, batch->vocab)};
  });
}

db_status db_schedule_verify(const db_schedule* schedule, const db_batch* batch) {
  if (!schedule || !batch) return null_arg();
  return guarded([&] {
    const dynbatch::ScheduleReport rep = dynbatch::verify_schedule(schedule->schedule, batch->programs);
    if (!rep.ok()) dynbatch::throw_error(Errc::verification_failed, rep.to_string());
  });
}

int64_t db_schedule_step_count(const db_schedule* schedule) {
  return schedule ? static_cast<int64_t>(schedule->schedule.steps.size()) : -1;
}

db_status db_schedule_expensive_calls(const db_schedule* schedule, const db_batch* batch, int64_t* out) {
  if (!schedule || !batch || !out) return null_arg();
  return guarded([&] { *out = dynbatch::count_expensive_calls(schedule->schedule, batch->vocab); });
}

db_status db_schedule_to_json(const db_schedule* schedule, char** out_text) {
  if (!schedule || !out_text) return null_arg();
  return guarded([&] { *out_text = dup_string(dynbatch::schedule_to_json(schedule->schedule)); });
}

db_status db_schedule_inject_fault(db_schedule* schedule, const char* kind) {
  if (!schedule || !kind) return null_arg();
  return guarded([&] {
    auto& steps = schedule->schedule.steps;
    const std::string k = kind;
    if (k == "dependency-order") {
      if (steps.size() < 2) dynbatch::throw_error(Errc::invalid_argument, "schedule has fewer than 2 steps");
      std::swap(steps.front(), steps.back());
    } else if (k == "duplicate") {
      if (steps.empty() || steps.front().empty() || steps.front().front().members.empty()) {
        dynbatch::throw_error(Errc::invalid_argument, "schedule is empty");
      }
      steps.back().push_back(steps.front().front());
    } else {
      dynbatch::throw_error(Errc::invalid_argument, "unknown fault kind '" + k + "'");
    }
  });
}

void db_schedule_free(db_schedule* schedule) { delete schedule; }

db_status db_execute(const db_batch* batch, const db_schedule* schedule, uint64_t module_seed, db_run** out) {
  if (!batch || !schedule || !out) return null_arg();
  return guarded([&] {
    dynbatch::ExecResult r = dynbatch::execute(schedule->schedule, batch->programs, batch->inputs, batch->vocab, module_seed);
    *out = new db_run{std::move(r.outputs), std::move(r.trace)};
  });
}

db_status db_run_outputs(const db_run* run, const double** data, int64_t* rows, int64_t* width) {
  if (!run || !data || !rows || !width) return null_arg();
  *data = run->outputs.data().data();
  *rows = run->outputs.rows();
  *width = run->outputs.width();
  return DB_OK;
}

int64_t db_run_expensive_calls(const db_run* run) { return run ? run->trace.expensive_calls : -1; }
int64_t db_run_peak_group_rows(const db_run* run) { return run ? run->trace.peak_group_rows : -1; }
double db_run_module_seconds(const db_run* run) { return run ? run->trace.module_seconds : -1.0; }
double db_run_stacking_seconds(const db_run* run) { return run ? run->trace.stacking_seconds : -1.0; }
double db_run_total_seconds(const db_run* run) { return run ? run->trace.total_seconds : -1.0; }

db_status db_run_trace_json(const db_run* run, char** out_text) {
  if (!run || !out_text) return null_arg();
  return guarded([&] { *out_text = dup_string(dynbatch::trace_to_json(run->trace)); });
}

void db_run_free(db_run* run) { delete run; }

db_status db_moe_run(const db_moe_opts* opts, int32_t batched, db_run** out) {
  if (!opts || !out) return null_arg();
  return guarded([&] {
    const dynbatch::MoeConfig cfg = to_cfg(opts);
    const dynbatch::MoeWorkload w = dynbatch::gen_moe_inputs(cfg, opts->seed);
    const dynbatch::ExpertSet experts(cfg.experts, cfg.data_dim, cfg.hidden, dynbatch::mix_seed(opts->seed, 0xe4be27ULL));
    const dynbatch::GateAssignment gates = dynbatch::top_k_gate(w.scores, cfg.active_per_example);
    dynbatch::MoeResult r = batched ? dynbatch::moe_forward_batched(w.inputs, experts, gates)
                                    : dynbatch::moe_forward_naive(w.inputs, experts, gates);
    *out = new db_run{std::move(r.outputs), std::move(r.trace)};
  });
}

db_status db_moe_memory_model(int64_t experts, int64_t active_per_example, int64_t hidden, int64_t data_dim,
                              double examples_per_expert, db_memory_model_t* out) {
  if (!out) return null_arg();
  return guarded([&] {
    dynbatch::MoeConfig c;
    c.experts = experts;
    c.active_per_example = active_per_example;
    c.hidden = hidden;
    c.data_dim = data_dim;
    c.examples_per_expert = examples_per_expert;
    out->param_count = dynbatch::moe_param_count(c);
    out->activation_count = dynbatch::moe_activation_count(c);
    out->memory_ratio = dynbatch::moe_memory_ratio(c);
  });
}

db_status db_verify_run(const db_verify_opts* opts, db_log_fn log, void* user) {
  if (!opts) return null_arg();
  dynbatch::VerifyReport report;
  const db_status st = guarded([&] {
    dynbatch::VerifyOptions o;
    o.seeds = opts->seeds;
    o.b = opts->batch;
    o.p = opts->vocab;
    o.length = opts->length;
    o.width = opts->width;
    o.base_seed = opts->seed;
    o.parallel = opts->parallel != 0;
    report = dynbatch::run_property_suite(o, [&](const std::string& line) { if (log) log(line.c_str(), user); });
  });
  if (st != DB_OK) return st;
  if (!report.ok()) {
    for (const std::string& f : report.failures) if (log) log(f.c_str(), user);
    t_error = std::to_string(report.failures.size()) + " verification failures";
    return DB_ERR_VERIFICATION_FAILED;
  }
  return DB_OK;
}

// ------------------------------------------------------ device extensions
int32_t db_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

void* db_host_alloc(int64_t bytes) {
  void* p = nullptr;
  if (bytes <= 0 || cudaHostAlloc(&p, static_cast<size_t>(bytes), cudaHostAllocPortable) != cudaSuccess) {
    cudaGetLastError();
    t_error = "cudaHostAlloc failed";
    return nullptr;
  }
  return p;
}

void db_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

db_status db_batch_generate_range(const db_workload_opts* opts, int64_t first, int64_t last, db_batch** out) {
  if (!opts || !out) return null_arg();
  return guarded([&] {
    dynbatch::WorkloadSpec spec;
    switch (opts->kind) {
      case DB_WORKLOAD_BALANCED_TREE: spec.kind = dynbatch::WorkloadKind::balanced_tree; break;
      case DB_WORKLOAD_CHAIN_HEAVY: spec.kind = dynbatch::WorkloadKind::chain_heavy; break;
      case DB_WORKLOAD_RANDOM_DAG: spec.kind = dynbatch::WorkloadKind::random_dag; break;
      default: dynbatch::throw_error(Errc::invalid_argument, "unknown workload kind");
    }
    spec.b = opts->batch;
    spec.p = opts->vocab;
    spec.width = opts->width;
    spec.depth = opts->depth;
    spec.length = opts->length;
    spec.branch_prob = opts->branch_prob;
    spec.seed = opts->seed;
    dynbatch::GeneratedBatch g = dynbatch::gen_batch_range(spec, first, last);
    *out = new db_batch{std::move(g.vocab), std::move(g.programs), std::move(g.inputs)};
  });
}

db_status db_debug_conv_waits(uint64_t* out64, int32_t reset, int32_t enable) {
  return guarded([&] {
    dynbatch::dev::require_device();
    dynbatch::dev::check(dbk_rb_debug(reinterpret_cast<unsigned long long*>(out64), reset, enable),
                         "dbk_rb_debug");
  });
}

db_status db_batch_inputs(const db_batch* batch, const double** data, int64_t* rows, int64_t* width) {
  if (!batch || !data || !rows || !width) return null_arg();
  *data = batch->inputs.data().data();
  *rows = batch->inputs.rows();
  *width = batch->inputs.width();
  return DB_OK;
}

static void copy_times(const dynbatch::dev::KernelTimes& k, db_kernel_times_t* out) {
  for (int c = 0; c < 8; ++c) {
    out->ms[c] = k.ms[c];
    out->launches[c] = k.launches[c];
    out->flops[c] = k.flops[c];
    out->bytes[c] = k.bytes[c];
  }
}

db_status db_iep_session_time(db_iep_session* s, int32_t iters, int32_t profile, double* ms,
                              db_kernel_times_t* kt) {
  if (!s || !ms) return null_arg();
  return guarded([&] {
    dynbatch::dev::KernelTimes k;
    *ms = s->s->time_forwards(iters, profile, &k);
    if (kt) copy_times(k, kt);
  });
}

db_status db_moe_session_time(db_moe_session* s, int32_t iters, int32_t profile, double* ms,
                              db_kernel_times_t* kt) {
  if (!s || !ms) return null_arg();
  return guarded([&] {
    dynbatch::dev::KernelTimes k;
    *ms = s->s->time_forwards(iters, profile != 0, &k);
    if (kt) copy_times(k, kt);
  });
}

db_status db_device_open(int32_t device) {
  return guarded([&] {
    dynbatch::dev::check(cudaSetDevice(device), "cudaSetDevice");
    dynbatch::dev::require_device();
  });
}

db_status db_iep_session_create(const db_batch* batch, int64_t first, int64_t last, uint64_t module_seed,
                                const db_module_opts* opts, db_iep_session** out) {
  if (!batch || !out) return null_arg();
  return guarded([&] {
    const auto kind = to_kind(opts);
    const std::int64_t b = static_cast<std::int64_t>(batch->programs.size());
    if (last <= first) { first = 0; last = b; }
    if (first < 0 || last > b) dynbatch::throw_error(Errc::invalid_argument, "program range out of bounds");
    std::span<const dynbatch::Program> progs(batch->programs.data() + first, static_cast<size_t>(last - first));
    dynbatch::TensorBatch in(last - first, batch->inputs.width());
    std::memcpy(in.data().data(), batch->inputs.data().data() + first * batch->inputs.width(),
                sizeof(double) * in.data().size());
    auto s = std::make_unique<dynbatch::dev::IepSession>(batch->vocab, progs, in, module_seed, kind,
                                                         opts ? opts->program_capacity : 0,
                                                         opts ? opts->node_capacity : 0,
                                                         opts ? opts->length_capacity : 0);
    *out = new db_iep_session{std::move(s)};
  });
}

db_status db_iep_session_set_schedule(db_iep_session* s, const db_schedule* schedule) {
  if (!s) return null_arg();
  return guarded([&] { s->s->set_schedule(schedule ? &schedule->schedule : nullptr); });
}

db_status db_iep_session_set_strategy(db_iep_session* s, db_strategy strategy) {
  if (!s) return null_arg();
  return guarded([&] { s->s->set_strategy(to_strategy(strategy)); });
}

db_status db_iep_session_forward(db_iep_session* s) {
  if (!s) return null_arg();
  return guarded([&] { s->s->forward(); });
}

db_status db_iep_session_forward_host(db_iep_session* s, const float* inputs, float* outputs) {
  if (!s || !inputs || !outputs) return null_arg();
  return guarded([&] { s->s->forward_host(inputs, outputs); });
}

db_status db_iep_session_set_programs(db_iep_session* s, const int32_t* tokens, const int32_t* seq_off, int64_t b) {
  // tokens may be NULL for an all-empty batch (reported as the empty-sequence error)
  if (!s || !seq_off || (!tokens && b > 0 && seq_off[b] > 0)) return null_arg();
  return guarded([&] { s->s->set_programs(tokens, seq_off, b); });
}

db_status db_iep_session_forward_host_async(db_iep_session* s, const float* inputs, float* outputs) {
  if (!s || !inputs || !outputs) return null_arg();
  return guarded([&] { s->s->forward_host_async(inputs, outputs); });
}

db_status db_iep_session_synchronize(db_iep_session* s) {
  if (!s) return null_arg();
  return guarded([&] { s->s->synchronize(); });
}

void* db_iep_session_stream(db_iep_session* s) { return s ? static_cast<void*>(s->s->stream()) : nullptr; }

db_status db_iep_session_stats(db_iep_session* s, db_session_stats_t* out) {
  if (!s || !out) return null_arg();
  return guarded([&] {
    s->s->synchronize();
    const dynbatch::ExecutionTrace t = s->s->trace();
    std::int64_t groups = 0;
    for (auto c : t.per_function_calls) groups += c;
    fill_stats(out, t, static_cast<std::int64_t>(t.per_step_seconds.size()), groups, s->s->csr().N,
               s->s->launches(), s->s->h2d_bytes(), s->s->d2h_bytes(), s->s->algorithmic_flops(),
               s->s->algorithmic_bytes());
  });
}

db_status db_iep_session_schedule(db_iep_session* s, db_schedule** out) {
  if (!s || !out) return null_arg();
  return guarded([&] {
    s->s->synchronize();
    *out = new db_schedule{s->s->download_schedule()};
  });
}

db_status db_iep_session_run(db_iep_session* s, db_run** out) {
  if (!s || !out) return null_arg();
  return guarded([&] {
    dynbatch::TensorBatch o = s->s->download_outputs();
    *out = new db_run{std::move(o), s->s->trace()};
  });
}

db_status db_iep_session_labels(db_iep_session* s, int32_t* labels, int64_t n) {
  if (!s || !labels) return null_arg();
  return guarded([&] {
    s->s->synchronize();
    const auto l = s->s->download_labels();
    if (static_cast<std::int64_t>(l.size()) != n) dynbatch::throw_error(Errc::row_count_mismatch, "label buffer size");
    std::memcpy(labels, l.data(), l.size() * sizeof(int32_t));
  });
}

db_status db_iep_session_set_head(db_iep_session* s, int32_t answers, uint64_t seed) {
  if (!s) return null_arg();
  return guarded([&] { s->s->set_head(answers, seed); });
}

db_status db_iep_session_head_forward(db_iep_session* s) {
  if (!s) return null_arg();
  return guarded([&] { s->s->head_forward(); });
}

db_status db_iep_session_logits(db_iep_session* s, float* out, int64_t n) {
  if (!s || !out) return null_arg();
  return guarded([&] { s->s->download_logits(out, n); });
}

db_status db_iep_session_forward_logits_host(db_iep_session* s, const float* inputs, float* logits) {
  if (!s || !inputs || !logits) return null_arg();
  return guarded([&] { s->s->forward_logits_host(inputs, logits); });
}

db_status db_iep_session_time_head(db_iep_session* s, int32_t iters, double* ms, double* flops) {
  if (!s || !ms) return null_arg();
  return guarded([&] {
    *ms = s->s->time_head(iters);
    if (flops) *flops = s->s->head_flops();
  });
}

db_status db_iep_session_set_training(db_iep_session* s, int32_t on) {
  if (!s) return null_arg();
  return guarded([&] { s->s->set_training(on != 0); });
}

db_status db_iep_session_train_step(db_iep_session* s, const int32_t* labels, float* loss) {
  if (!s || !labels) return null_arg();
  return guarded([&] {
    const float l = s->s->train_step(labels);
    if (loss) *loss = l;
  });
}

db_status db_iep_session_grad_size(db_iep_session* s, int32_t which, int32_t fid, int64_t* n) {
  if (!s || !n) return null_arg();
  return guarded([&] { *n = s->s->grad_size(which, fid); });
}

db_status db_iep_session_grad(db_iep_session* s, int32_t which, int32_t fid, float* out, int64_t n) {
  if (!s || (!out && n)) return null_arg();
  return guarded([&] { s->s->download_grad(which, fid, out, n); });
}

db_status db_iep_session_sgd(db_iep_session* s, float lr) {
  if (!s) return null_arg();
  return guarded([&] { s->s->sgd_update(lr); });
}

db_status db_iep_session_time_train(db_iep_session* s, int32_t iters, const int32_t* labels, double* ms) {
  if (!s || !labels || !ms) return null_arg();
  return guarded([&] { *ms = s->s->time_train(iters, labels); });
}

void db_iep_session_free(db_iep_session* s) { delete s; }

db_status db_execute_device(const db_batch* batch, const db_schedule* schedule, uint64_t module_seed,
                            const db_module_opts* opts, db_run** out) {
  if (!batch || !out) return null_arg();
  return guarded([&] {
    dynbatch::dev::IepSession s(batch->vocab, batch->programs, batch->inputs, module_seed, to_kind(opts));
    if (schedule) s.set_schedule(&schedule->schedule);
    s.forward();
    dynbatch::TensorBatch o = s.download_outputs();
    *out = new db_run{std::move(o), s.trace()};
  });
}

db_status db_moe_session_create(const db_moe_opts* opts, int32_t precision, int64_t first, int64_t last,
                                db_moe_session** out) {
  if (!opts || !out) return null_arg();
  return guarded([&] {
    auto s = std::make_unique<dynbatch::dev::MoeSession>(to_cfg(opts), opts->seed, precision, first, last);
    *out = new db_moe_session{std::move(s)};
  });
}

db_status db_moe_session_forward(db_moe_session* s) {
  if (!s) return null_arg();
  return guarded([&] { s->s->forward(); });
}

db_status db_moe_session_forward_host(db_moe_session* s, const float* inputs, const double* scores, float* outputs) {
  if (!s || !inputs || !scores || !outputs) return null_arg();
  return guarded([&] { s->s->forward_host(inputs, scores, outputs); });
}

db_status db_moe_session_forward_host_async(db_moe_session* s, const float* inputs, const double* scores,
                                           float* outputs) {
  if (!s || !inputs || !scores || !outputs) return null_arg();
  return guarded([&] { s->s->forward_host_async(inputs, scores, outputs); });
}

db_status db_moe_session_synchronize(db_moe_session* s) {
  if (!s) return null_arg();
  return guarded([&] { s->s->synchronize(); });
}

void* db_moe_session_stream(db_moe_session* s) { return s ? static_cast<void*>(s->s->stream()) : nullptr; }

db_status db_moe_session_stats(db_moe_session* s, db_session_stats_t* out) {
  if (!s || !out) return null_arg();
  return guarded([&] {
    s->s->synchronize();
    const dynbatch::ExecutionTrace t = s->s->trace();
    fill_stats(out, t, 1, t.expensive_calls, s->s->tokens(), s->s->launches(), s->s->h2d_bytes(),
               s->s->d2h_bytes(), s->s->algorithmic_flops(), s->s->algorithmic_bytes());
  });
}

db_status db_moe_session_routing(db_moe_session* s, int32_t* ids, double* weights, int32_t* offsets,
                                 int32_t* items) {
  if (!s) return null_arg();
  return guarded([&] { s->s->routing(ids, weights, offsets, items); });
}

db_status db_moe_session_run(db_moe_session* s, db_run** out) {
  if (!s || !out) return null_arg();
  return guarded([&] {
    dynbatch::TensorBatch o = s->s->download_outputs();
    *out = new db_run{std::move(o), s->s->trace()};
  });
}

db_status db_moe_session_outputs(db_moe_session* s, const int64_t* rows, int64_t n_rows, float* out) {
  if (!s || !out) return null_arg();
  return guarded([&] { s->s->download_rows(rows, n_rows, out); });
}

void db_moe_session_free(db_moe_session* s) { delete s; }

// ------------------------------------------------- expert-parallel MoE rank
db_status db_moe_ep_create(const db_moe_opts* opts, int32_t precision, int32_t rank, int32_t world,
                           db_moe_ep_session** out) {
  if (!opts || !out) return null_arg();
  return guarded([&] {
    auto s = std::make_unique<dynbatch::dev::MoeEp>(to_cfg(opts), opts->seed, precision, rank, world);
    *out = new db_moe_ep_session{std::move(s)};
  });
}

db_status db_moe_ep_nccl_id(void* unique_id) {
  if (!unique_id) return null_arg();
  return guarded([&] {
    const dynbatch::dev::Nccl& nc = dynbatch::dev::Nccl::get();
    ncclUniqueId id;
    nc.check(nc.GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(unique_id, &id, sizeof(id));
  });
}

db_status db_moe_ep_comm_init(db_moe_ep_session* s, const void* unique_id) {
  if (!s || !unique_id) return null_arg();
  return guarded([&] { s->s->comm_init(unique_id); });
}

db_status db_moe_ep_forward(db_moe_ep_session* s, int32_t chunks) {
  if (!s) return null_arg();
  return guarded([&] { s->s->forward(chunks); });
}

db_status db_moe_ep_recv_rows(db_moe_ep_session* s, int64_t* rows) {
  if (!s || !rows) return null_arg();
  *rows = s->s->last_recv_rows();
  return DB_OK;
}

db_status db_moe_ep_plan(int32_t G, int32_t E, const int32_t* send_counts, const int32_t* recv_counts,
                         int32_t chunks, int32_t* n_chunks, int64_t* send_off, int64_t* send_rows,
                         int64_t* recv_off, int64_t* recv_rows) {
  if (!send_counts || !recv_counts || !n_chunks) return null_arg();
  return guarded([&] {
    if (G < 1 || E < 1) dynbatch::throw_error(dynbatch::Errc::invalid_argument, "G and E must be positive");
    const dynbatch::dev::EpPlan p = dynbatch::dev::make_ep_plan(G, E, send_counts, recv_counts, chunks);
    *n_chunks = p.C;
    const size_t cg = static_cast<size_t>(p.C) * G;
    if (send_off) std::copy(p.s_off.begin(), p.s_off.begin() + cg, send_off);
    if (send_rows) std::copy(p.s_rows.begin(), p.s_rows.begin() + cg, send_rows);
    if (recv_off) std::copy(p.r_off.begin(), p.r_off.begin() + cg, recv_off);
    if (recv_rows) std::copy(p.r_rows.begin(), p.r_rows.begin() + cg, recv_rows);
  });
}

db_status db_moe_ep_sizes(db_moe_ep_session* s, int64_t* tokens, int64_t* items, int32_t* local_experts) {
  if (!s) return null_arg();
  if (tokens) *tokens = s->s->tokens();
  if (items) *items = s->s->items();
  if (local_experts) *local_experts = s->s->local_experts();
  return DB_OK;
}

db_status db_moe_ep_dispatch(db_moe_ep_session* s, void* send_rows, int32_t* expert_counts) {
  if (!s || !send_rows || !expert_counts) return null_arg();
  return guarded([&] { s->s->dispatch(send_rows, expert_counts); });
}

db_status db_moe_ep_experts(db_moe_ep_session* s, const void* recv_rows, const int32_t* recv_counts,
                            void* ret_rows) {
  if (!s || !recv_counts) return null_arg();
  return guarded([&] { s->s->experts(recv_rows, recv_counts, ret_rows); });
}

db_status db_moe_ep_forward_local(db_moe_ep_session* s) {
  if (!s) return null_arg();
  return guarded([&] { s->s->forward_local(); });
}

db_status db_moe_ep_layout(db_moe_ep_session* s, const int32_t* recv_counts) {
  if (!s || !recv_counts) return null_arg();
  return guarded([&] { s->s->layout(recv_counts); });
}

db_status db_moe_ep_experts_range(db_moe_ep_session* s, const void* recv_rows, void* ret_rows, int32_t e_begin,
                                  int32_t e_end) {
  if (!s) return null_arg();
  return guarded([&] { s->s->experts_range(recv_rows, ret_rows, e_begin, e_end); });
}

db_status db_moe_ep_combine(db_moe_ep_session* s, const void* ret_rows) {
  if (!s || !ret_rows) return null_arg();
  return guarded([&] { s->s->combine(ret_rows); });
}

db_status db_moe_ep_outputs(db_moe_ep_session* s, float* out) {
  if (!s || !out) return null_arg();
  return guarded([&] { s->s->download_outputs(out); });
}

db_status db_moe_ep_synchronize(db_moe_ep_session* s) {
  if (!s) return null_arg();
  return guarded([&] { s->s->synchronize(); });
}

void* db_moe_ep_stream(db_moe_ep_session* s) { return s ? static_cast<void*>(s->s->stream()) : nullptr; }

void db_moe_ep_free(db_moe_ep_session* s) { delete s; }

db_status db_moe_run_device(const db_moe_opts* opts, int32_t precision, db_run** out) {
  if (!opts || !out) return null_arg();
  return guarded([&] {
    dynbatch::dev::MoeSession s(to_cfg(opts), opts->seed, precision, 0, 0);
    s.forward();
    dynbatch::TensorBatch o = s.download_outputs();
    *out = new db_run{std::move(o), s.trace()};
  });
}

}  // extern "C"
