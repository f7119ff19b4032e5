// device.cpp — device context, batch upload, device scheduler and the IEP
// session (forward = device scheduler + per-step module kernels).
#include "device.hpp"

#include <algorithm>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>

#include "dynbatch/dbk.h"
#include "iep_head.hpp"
#include "iep_train.hpp"
#include "iep_rb.hpp"

namespace dynbatch::dev {

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
  }
}

namespace {
thread_local int t_checked_device = -1;
int g_sm_count = 0;
}  // namespace

void require_device() {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  int count = 0;
  if (e == cudaSuccess) e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    cudaGetLastError();
    throw std::runtime_error(
        "no CUDA device available: the dynbatch B200 library has no CPU fallback");
  }
  if (t_checked_device == dev) return;
  cudaDeviceProp prop{};
  check(cudaGetDeviceProperties(&prop, dev), "cudaGetDeviceProperties");
  if (prop.major != 10) {
    throw std::runtime_error("device " + std::to_string(dev) + " (" + prop.name +
                             ") is not sm_100; this library is built for sm_100a only");
  }
  g_sm_count = prop.multiProcessorCount;
  t_checked_device = dev;
}

int sm_count() {
  require_device();
  return g_sm_count;
}

// --------------------------------------------------------------- Profiler
Profiler::~Profiler() {
  for (cudaEvent_t e : pool_) cudaEventDestroy(e);
}

cudaEvent_t Profiler::next_event() {
  if (used_ == pool_.size()) {
    cudaEvent_t e;
    check(cudaEventCreate(&e), "cudaEventCreate");
    pool_.push_back(e);
  }
  return pool_[used_++];
}

void Profiler::begin(int cls, cudaStream_t s) {
  if (!on) return;
  Rec r{cls, next_event(), next_event()};
  check(cudaEventRecord(r.a, s), "event");
  recs_.push_back(r);
}

void Profiler::end(cudaStream_t s) {
  if (!on) return;
  check(cudaEventRecord(recs_.back().b, s), "event");
}

KernelTimes Profiler::collect() {
  KernelTimes kt;
  for (const Rec& r : recs_) {
    float ms = 0.f;
    check(cudaEventElapsedTime(&ms, r.a, r.b), "cudaEventElapsedTime");
    kt.ms[r.cls] += ms;
    ++kt.launches[r.cls];
  }
  for (int c = 0; c < 8; ++c) {
    kt.flops[c] = work_flops_[c];
    kt.bytes[c] = work_bytes_[c];
    work_flops_[c] = work_bytes_[c] = 0.0;
  }
  reset();
  return kt;
}

HostCSR make_csr(std::span<const Program> programs, const FunctionVocab& vocab) {
  HostCSR c;
  c.b = static_cast<std::int64_t>(programs.size());
  c.p = vocab.size();
  c.arity_of.resize(static_cast<size_t>(c.p));
  c.expensive_of.resize(static_cast<size_t>(c.p));
  for (const ModuleSpec& s : vocab.specs()) {
    c.arity_of[static_cast<size_t>(s.function_id)] = s.arity;
    c.expensive_of[static_cast<size_t>(s.function_id)] = s.is_expensive() ? 1 : 0;
    c.max_arity = std::max(c.max_arity, s.arity);
  }
  std::int64_t N = 0;
  for (const Program& p : programs) N += p.size();
  if (N >= (1LL << 31)) throw_error(Errc::invalid_argument, "batch too large for int32 node ids");
  c.N = N;
  c.prog_off.reserve(static_cast<size_t>(c.b) + 1);
  c.fid.reserve(static_cast<size_t>(N));
  c.child_off.reserve(static_cast<size_t>(N) + 1);
  c.example.reserve(static_cast<size_t>(N));
  std::int32_t off = 0;
  for (std::int64_t e = 0; e < c.b; ++e) {
    const Program& prog = programs[static_cast<size_t>(e)];
    c.prog_off.push_back(off);
    c.root_g.push_back(off + prog.root);
    c.s_max = std::max(c.s_max, prog.size());
    for (const ProgramNode& node : prog.nodes) {
      c.fid.push_back(node.function_id);
      c.example.push_back(static_cast<std::int32_t>(e));
      c.child_off.push_back(static_cast<std::int32_t>(c.child_list.size()));
      for (int ch : node.children) c.child_list.push_back(off + ch);
      c.child0.push_back(node.children.size() > 0 ? off + node.children[0] : -1);
      c.child1.push_back(node.children.size() > 1 ? off + node.children[1] : -1);
    }
    off += prog.size();
  }
  c.prog_off.push_back(off);
  c.child_off.push_back(static_cast<std::int32_t>(c.child_list.size()));
  c.cap_b = c.b;
  c.cap_N = c.N;
  c.cap_s = c.s_max;
  return c;
}

// ------------------------------------------------------ DeviceProgramBatch
DeviceProgramBatch::DeviceProgramBatch(const HostCSR& csr, cudaStream_t s) : csr_(csr) {
  const size_t cb = static_cast<size_t>(std::max<std::int64_t>(std::max(csr.cap_b, csr.b), 1));
  const size_t N = static_cast<size_t>(std::max<std::int64_t>(std::max(csr.cap_N, csr.N), 1));
  csr_.cap_b = static_cast<std::int64_t>(cb);
  csr_.cap_N = static_cast<std::int64_t>(N);
  csr_.cap_s = std::max(csr.cap_s, csr.s_max);
  prog_off.alloc(cb + 1);
  root_g.alloc(cb);
  for (Buf<std::int32_t>* bf : {&fid, &child0, &child1, &example, &fwd_ok}) bf->alloc(N);
  child_off.alloc(N + 1);
  child_list.alloc(N);
  prog_off.upload(csr.prog_off, s);
  fid.upload(csr.fid, s);
  child_off.upload(csr.child_off, s);
  child_list.upload(csr.child_list, s);
  child0.upload(csr.child0, s);
  child1.upload(csr.child1, s);
  example.upload(csr.example, s);
  root_g.upload(csr.root_g, s);
  arity_of.upload(csr.arity_of, s);
  labels.alloc(N);
  scratch.alloc(2 * N);
  scalars.alloc(8);
  member_g.alloc(N);
  // d_max + 1 <= s_max, so at most s_max * p (step, fid) keys / groups.
  max_keys_ = std::max(1, csr_.cap_s) * csr.p;
  seg_hist.alloc(static_cast<size_t>(dbk_bucket_sort_scratch(static_cast<std::int64_t>(N), max_keys_)));
  group_fid.alloc(static_cast<size_t>(max_keys_) + 1);
  group_begin.alloc(static_cast<size_t>(max_keys_) + 2);
  step_group_begin.alloc(static_cast<size_t>(std::max(1, csr_.cap_s)) + 2);
  detect_static_shape(s);
}

std::int64_t DeviceProgramBatch::begin_prefix_programs(const std::int32_t* seq_off, std::int64_t b) {
  if (b <= 0) throw_error(Errc::invalid_argument, "empty program batch");
  if (b > csr_.cap_b) throw_error(Errc::invalid_argument, "more programs than the session capacity");
  if (seq_off[0] != 0) throw_error(Errc::invalid_argument, "sequence offsets must start at 0");
  const std::int64_t N = seq_off[b];
  int s_max = 0;
  for (std::int64_t e = 0; e < b; ++e) {
    const std::int32_t n = seq_off[e + 1] - seq_off[e];
    if (n < 0) throw_error(Errc::invalid_argument, "sequence offsets must be non-decreasing");
    if (n == 0) throw_error(Errc::invalid_argument, "empty function sequence");
    s_max = std::max(s_max, n);
  }
  if (N > csr_.cap_N || s_max > csr_.cap_s)
    throw_error(Errc::invalid_argument, "batch exceeds the session capacity (nodes or program length)");
  csr_.b = b;
  csr_.N = N;
  csr_.s_max = s_max;
  shape_n_ = 0;  // the static-shape table described the old batch
  steps = 0;
  build_err_.ensure(1);
  build_stack_.ensure(static_cast<size_t>(csr_.cap_N));
  return N;
}

void DeviceProgramBatch::build_prefix_programs(const std::int32_t* tokens_dev, const std::int32_t* seq_off_dev,
                                               cudaStream_t s) {
  check(cudaMemsetAsync(build_err_.get(), 0, sizeof(std::int32_t), s), "memset");
  check(dbk_build_prefix(csr_.b, tokens_dev, seq_off_dev, csr_.p, arity_of.get(), prog_off.get(), fid.get(),
                         child_off.get(), child_list.get(), child0.get(), child1.get(), example.get(), root_g.get(),
                         fwd_ok.get(), build_stack_.get(), build_err_.get(), s),
        "dbk_build_prefix");
  build_pending_ = true;
}

void DeviceProgramBatch::set_prefix_programs(const std::int32_t* tokens, const std::int32_t* seq_off,
                                             std::int64_t b, cudaStream_t s) {
  const std::int64_t N = begin_prefix_programs(seq_off, b);
  tokens_dev_.ensure(static_cast<size_t>(csr_.cap_N));
  seq_off_dev_.ensure(static_cast<size_t>(csr_.cap_b) + 1);
  check(cudaMemcpyAsync(tokens_dev_.get(), tokens, sizeof(std::int32_t) * static_cast<size_t>(N), cudaMemcpyHostToDevice,
                        s), "H2D tokens");
  check(cudaMemcpyAsync(seq_off_dev_.get(), seq_off, sizeof(std::int32_t) * static_cast<size_t>(b + 1),
                        cudaMemcpyHostToDevice, s), "H2D offsets");
  build_prefix_programs(tokens_dev_.get(), seq_off_dev_.get(), s);
}

void DeviceProgramBatch::replace_host_csr(const HostCSR& csr) {
  const std::int64_t cb = csr_.cap_b, cn = csr_.cap_N;
  const int cs = csr_.cap_s;
  csr_ = csr;
  csr_.cap_b = cb;
  csr_.cap_N = cn;
  csr_.cap_s = cs;
}

// Balanced-tree static schedule (SURVEY.md §3 balanced_static_schedule):
// when every program has the same tree shape (node count, local child lists,
// root), the longest-root-distance labels are one per-shape table, computed
// here once with the reference's rule (src/program.cpp:239-272); the device
// scheduler then only fills labels from it and buckets by fid per level.
void DeviceProgramBatch::detect_static_shape(cudaStream_t s) {
  const HostCSR& c = csr_;
  if (c.b < 2) return;
  const std::int32_t n = c.prog_off[1] - c.prog_off[0];
  if (n <= 0 || static_cast<std::int64_t>(n) * c.b != c.N) return;
  for (std::int64_t e = 0; e < c.b; ++e) {
    const std::int32_t base = static_cast<std::int32_t>(e) * n;
    if (c.prog_off[static_cast<size_t>(e)] != base) return;
    if (c.root_g[static_cast<size_t>(e)] - base != c.root_g[0]) return;
    for (std::int32_t i = 0; i < n; ++i) {
      const size_t g = static_cast<size_t>(base + i), g0 = static_cast<size_t>(i);
      const std::int32_t a = c.child_off[g + 1] - c.child_off[g];
      if (a != c.child_off[g0 + 1] - c.child_off[g0]) return;
      for (std::int32_t k = 0; k < a; ++k) {
        if (c.child_list[static_cast<size_t>(c.child_off[g] + k)] - base !=
            c.child_list[static_cast<size_t>(c.child_off[g0] + k)])
          return;
      }
    }
  }
  // labels of the shape: longest distance from the root (Kahn over the DAG)
  std::vector<std::int32_t> lab(static_cast<size_t>(n), -1), indeg(static_cast<size_t>(n), 0), queue;
  for (std::int32_t i = 0; i < n; ++i)
    for (std::int32_t k = c.child_off[static_cast<size_t>(i)]; k < c.child_off[static_cast<size_t>(i) + 1]; ++k)
      ++indeg[static_cast<size_t>(c.child_list[static_cast<size_t>(k)])];
  const std::int32_t root = c.root_g[0];
  if (indeg[static_cast<size_t>(root)] != 0) return;
  lab[static_cast<size_t>(root)] = 0;
  queue.push_back(root);
  for (size_t h = 0; h < queue.size(); ++h) {
    const std::int32_t u = queue[h];
    for (std::int32_t k = c.child_off[static_cast<size_t>(u)]; k < c.child_off[static_cast<size_t>(u) + 1]; ++k) {
      const std::int32_t v = c.child_list[static_cast<size_t>(k)];
      lab[static_cast<size_t>(v)] = std::max(lab[static_cast<size_t>(v)], lab[static_cast<size_t>(u)] + 1);
      if (--indeg[static_cast<size_t>(v)] == 0) queue.push_back(v);
    }
  }
  if (static_cast<std::int32_t>(queue.size()) != n) return;  // unreachable node: the dynamic path reports it
  shape_dmax_ = *std::max_element(lab.begin(), lab.end());
  shape_labels_.upload(lab, s);
  shape_n_ = n;
}

int DeviceProgramBatch::run_scheduler(cudaStream_t s, bool upper_bound, Strategy strategy) {
  if (strategy == Strategy::naive) throw_error(Errc::invalid_argument, "the naive schedule is host-built");
  if (csr_.b == 0) {
    steps = 0;
    groups = 0;
    return 0;
  }
  check(cudaMemsetAsync(scalars.get(), 0, sizeof(std::int32_t) * 8, s), "memset");
  const bool shape = static_shape() && strategy == Strategy::improved;
  if (shape) {  // balanced-tree (shared shape) static schedule: labels from the shape table
    check(dbk_sched_labels_static(csr_.N, shape_n_, shape_labels_.get(), shape_dmax_, labels.get(), scalars.get(), s),
          "dbk_sched_labels_static");
  } else {
    check(dbk_sched_labels(csr_.b, csr_.N, prog_off.get(), child_off.get(), child_list.get(), root_g.get(),
                           labels.get(), scratch.get(), scalars.get(), static_cast<std::int32_t>(strategy), s),
          "dbk_sched_labels");
  }
  // improved, standard and online all take ≤ s_max steps
  const int cap = std::max(1, csr_.s_max);
  check(dbk_sched_bucket_sort(csr_.N, csr_.p, max_keys_, fid.get(), labels.get(), scalars.get(),
                              seg_hist.get(), member_g.get(), group_fid.get(), group_begin.get(),
                              step_group_begin.get(), cap, strategy == Strategy::improved ? 0 : 1, s),
        "dbk_sched_bucket_sort");
  if (shape) {  // the step count is known: no host sync in the forward
    steps = shape_dmax_ + 1;
    groups_pending_ = true;
    return steps;
  }
  if (upper_bound) {  // no host sync: per-step work for s_max steps, the empty ones exit on the device
    steps = cap;
    groups_pending_ = true;
    errors_pending_ = true;
    return steps;
  }
  std::int32_t host_scal[3];
  check(cudaMemcpyAsync(host_scal, scalars.get(), sizeof(host_scal), cudaMemcpyDeviceToHost, s),
        "D2H scalars");
  check(cudaStreamSynchronize(s), "scheduler sync");
  if (host_scal[1]) throw_error(Errc::invalid_program, "cycle or unreachable node");
  steps = host_scal[0] + 1;
  groups = host_scal[2];
  groups_pending_ = false;
  return steps;
}

// Reads the device scheduler's scalars (d_max, error flag, group count)
// when the last forward did not: the real step count replaces the upper
// bound once the forward is done.
void DeviceProgramBatch::resolve(cudaStream_t s) const {
  if (build_pending_) {
    std::int32_t e = 0;
    check(cudaMemcpyAsync(&e, build_err_.get(), sizeof(e), cudaMemcpyDeviceToHost, s), "D2H build error");
    check(cudaStreamSynchronize(s), "sync");
    build_pending_ = false;
    switch (e) {
      case 0: break;
      case 1: throw_error(Errc::invalid_argument, "empty function sequence");
      case 2: throw_error(Errc::unknown_function, "a sequence names an unknown function id");
      case 3: throw_error(Errc::underfull_sequence, "a sequence ends with unfilled arities");
      default: throw_error(Errc::overfull_sequence, "tokens remain after the root closes");
    }
  }
  if (!groups_pending_ && !errors_pending_) return;
  std::int32_t scal[3] = {0, 0, 0};
  check(cudaMemcpyAsync(scal, scalars.get(), sizeof(scal), cudaMemcpyDeviceToHost, s), "D2H scalars");
  check(cudaStreamSynchronize(s), "sync");
  const bool check_err = errors_pending_;
  groups_pending_ = errors_pending_ = false;
  groups = scal[2];
  steps = scal[0] + 1;
  if (check_err && scal[1]) throw_error(Errc::invalid_program, "cycle or unreachable node");
}

void DeviceProgramBatch::check_scheduler_error(cudaStream_t s) const { resolve(s); }

std::int64_t DeviceProgramBatch::group_count(cudaStream_t s) const {
  resolve(s);
  return groups;
}

// The reference executor's order checks replayed over a host schedule
// without arithmetic: a gather of a node not yet written raises
// MissingOperand (src/executor.cpp:48-51, gathered operand by operand for the
// whole group, :139-151), a second write raises SingleAssignmentViolation
// (:62-65, at the group's scatter, :161-163), and an absent root raises
// MissingOperand (:168-173). The resblock kernels trust the schedule order
// (forwarding and tile dependencies are planned from it), so a broken
// schedule fails here, before any kernel runs, with the error the reference
// raises first.
static void check_reference_order(const Schedule& schedule, const HostCSR& c) {
  std::vector<unsigned char> present(static_cast<size_t>(c.N), 0);
  auto ref = [&](std::int32_t g) {
    const std::int32_t e = c.example[static_cast<size_t>(g)];
    return "(" + std::to_string(e) + ", " + std::to_string(g - c.prog_off[static_cast<size_t>(e)]) + ")";
  };
  for (const Step& step : schedule.steps) {
    for (const CallGroup& grp : step) {
      const int a = c.arity_of[static_cast<size_t>(grp.function_id)];
      for (int k = 0; k < a; ++k) {
        for (const NodeRef& r : grp.members) {
          const std::int32_t g = c.prog_off[static_cast<size_t>(r.example)] + r.node;
          const std::int32_t ch = c.child_list[static_cast<size_t>(c.child_off[static_cast<size_t>(g)] + k)];
          if (!present[static_cast<size_t>(ch)]) throw_error(Errc::missing_operand, "no value for node " + ref(ch));
        }
      }
      for (const NodeRef& r : grp.members) {
        const std::int32_t g = c.prog_off[static_cast<size_t>(r.example)] + r.node;
        if (present[static_cast<size_t>(g)])
          throw_error(Errc::single_assignment_violation, "node " + ref(g) + " written twice");
        present[static_cast<size_t>(g)] = 1;
      }
    }
  }
  for (std::int64_t e = 0; e < c.b; ++e) {
    const std::int32_t g = c.root_g[static_cast<size_t>(e)];
    if (!present[static_cast<size_t>(g)]) throw_error(Errc::missing_operand, "no value for node " + ref(g));
  }
}

int DeviceProgramBatch::load_schedule(const Schedule& schedule, cudaStream_t s) {
  std::vector<std::int32_t> mg, gf, gb, sgb;
  sgb.reserve(schedule.steps.size() + 1);
  for (const Step& step : schedule.steps) {
    sgb.push_back(static_cast<std::int32_t>(gf.size()));
    for (const CallGroup& g : step) {
      if (g.function_id < 0 || g.function_id >= csr_.p) {
        throw_error(Errc::unknown_function, "function id " + std::to_string(g.function_id));
      }
      gf.push_back(g.function_id);
      gb.push_back(static_cast<std::int32_t>(mg.size()));
      for (const NodeRef& r : g.members) {
        if (r.example < 0 || r.example >= csr_.b || r.node < 0 ||
            r.node >= csr_.prog_off[static_cast<size_t>(r.example) + 1] -
                          csr_.prog_off[static_cast<size_t>(r.example)]) {
          throw_error(Errc::invalid_argument, "node ref out of range (" +
                                                  std::to_string(r.example) + ", " +
                                                  std::to_string(r.node) + ")");
        }
        const std::int32_t gid = csr_.prog_off[static_cast<size_t>(r.example)] + r.node;
        // a member runs its group's module: its own function must be the
        // group's (the reference indexes children by the group's arity, UB
        // on a mismatch; the device kernels would read absent children)
        if (csr_.fid[static_cast<size_t>(gid)] != g.function_id) {
          throw_error(Errc::invalid_argument, "node (" + std::to_string(r.example) + ", " + std::to_string(r.node) +
                                                  ") has function " + std::to_string(csr_.fid[static_cast<size_t>(gid)]) +
                                                  " but sits in a group of function " +
                                                  std::to_string(g.function_id));
        }
        mg.push_back(gid);
      }
    }
  }
  sgb.push_back(static_cast<std::int32_t>(gf.size()));
  gb.push_back(static_cast<std::int32_t>(mg.size()));
  member_g.upload(mg, s);
  group_fid.upload(gf, s);
  group_begin.upload(gb, s);
  step_group_begin.upload(sgb, s);
  steps = static_cast<int>(schedule.steps.size());
  groups = static_cast<std::int64_t>(gf.size());
  groups_pending_ = false;
  return steps;
}

Schedule DeviceProgramBatch::download_schedule(Strategy strategy, cudaStream_t s) const {
  Schedule out{strategy, {}};
  if (steps == 0) return out;
  group_count(s);
  const auto sgb = step_group_begin.download(static_cast<size_t>(steps) + 1, s);
  const auto gf = group_fid.download(static_cast<size_t>(groups), s);
  const auto gb = group_begin.download(static_cast<size_t>(groups) + 1, s);
  const auto mg = member_g.download(static_cast<size_t>(gb.back()), s);
  out.steps.resize(static_cast<size_t>(steps));
  for (int st = 0; st < steps; ++st) {
    for (std::int32_t g = sgb[static_cast<size_t>(st)]; g < sgb[static_cast<size_t>(st) + 1]; ++g) {
      CallGroup cg;
      cg.function_id = gf[static_cast<size_t>(g)];
      for (std::int32_t m = gb[static_cast<size_t>(g)]; m < gb[static_cast<size_t>(g) + 1]; ++m) {
        const std::int32_t node = mg[static_cast<size_t>(m)];
        const std::int32_t e = csr_.example[static_cast<size_t>(node)];
        cg.members.push_back({e, node - csr_.prog_off[static_cast<size_t>(e)]});
      }
      out.steps[static_cast<size_t>(st)].push_back(std::move(cg));
    }
  }
  return out;
}

ExecutionTrace DeviceProgramBatch::trace_counts(cudaStream_t s) const {
  ExecutionTrace t;
  t.per_function_calls.assign(static_cast<size_t>(csr_.p), 0);
  if (steps == 0) return t;
  group_count(s);
  const auto gf = group_fid.download(static_cast<size_t>(groups), s);
  const auto gb = group_begin.download(static_cast<size_t>(groups) + 1, s);
  for (std::int64_t g = 0; g < groups; ++g) {
    const std::int32_t f = gf[static_cast<size_t>(g)];
    ++t.per_function_calls[static_cast<size_t>(f)];
    if (csr_.expensive_of[static_cast<size_t>(f)]) ++t.expensive_calls;
    t.peak_group_rows = std::max<std::int64_t>(t.peak_group_rows,
                                                gb[static_cast<size_t>(g) + 1] - gb[static_cast<size_t>(g)]);
  }
  return t;
}

// ------------------------------------------------------------- IepSession
IepSession::IepSession(const FunctionVocab& vocab, std::span<const Program> programs,
                       const TensorBatch& inputs, std::uint64_t module_seed, ModuleKind kind,
                       std::int64_t cap_programs, std::int64_t cap_nodes, int cap_length)
    : vocab_(vocab), kind_(kind), width_(vocab.width()) {
  require_device();
  require_valid_batch(programs, vocab);
  if (inputs.rows() != static_cast<std::int64_t>(programs.size())) {
    throw_error(Errc::row_count_mismatch, "inputs have " + std::to_string(inputs.rows()) +
                                              " rows for batch of " + std::to_string(programs.size()));
  }
  if (!programs.empty() && inputs.width() != width_) {
    throw_error(Errc::width_mismatch, "inputs width " + std::to_string(inputs.width()));
  }
  if (!inputs.all_finite()) throw_error(Errc::non_finite_value, "non-finite input");
  check(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "stream");
  HostCSR csr = make_csr(programs, vocab);
  csr.cap_b = std::max(csr.b, cap_programs);
  csr.cap_N = std::max(csr.N, cap_nodes);
  csr.cap_s = std::max(csr.s_max, cap_length);
  batch_ = std::make_unique<DeviceProgramBatch>(csr, stream_);
  err_.alloc(4);
  present_.alloc(static_cast<size_t>(std::max<std::int64_t>(batch_->csr().cap_N, 1)));
  // cudaMalloc does not clear: the error word is read (synchronize) before
  // the first forward resets it, and a fresh allocation can hold the bytes
  // of a session destroyed earlier in the process
  err_.zero(stream_);
  present_.zero(stream_);
  if (kind_ == ModuleKind::dense) {
    in64_.upload(inputs.data().data(), inputs.data().size(), stream_);
    values64_.alloc(static_cast<size_t>(std::max<std::int64_t>(batch_->csr().cap_N, 1)) * static_cast<size_t>(width_));
    out64_.alloc(static_cast<size_t>(std::max<std::int64_t>(csr.b, 1)) * static_cast<size_t>(width_));
    ModuleSet modules(vocab, module_seed);
    std::vector<const double*> wt(static_cast<size_t>(vocab.size()), nullptr), bt = wt;
    w64_.resize(static_cast<size_t>(vocab.size()));
    for (int f = 0; f < vocab.size(); ++f) {
      const ModuleImpl& m = modules.impl(f);
      if (m.spec.arity == 0) continue;
      std::vector<double> blob(m.weights);
      blob.insert(blob.end(), m.bias.begin(), m.bias.end());
      w64_[static_cast<size_t>(f)].upload(blob, stream_);
      wt[static_cast<size_t>(f)] = w64_[static_cast<size_t>(f)].get();
      bt[static_cast<size_t>(f)] = w64_[static_cast<size_t>(f)].get() + m.weights.size();
    }
    wtab_.upload(wt, stream_);
    btab_.upload(bt, stream_);
  } else {
    init_resblock(inputs, module_seed);
  }
  check(cudaStreamSynchronize(stream_), "session upload");
}


void IepSession::set_strategy(Strategy strategy) {
  if (strategy == Strategy::naive)
    throw_error(Errc::invalid_argument, "naive runs one node per step: load it with set_schedule");
  ++schedule_gen_;
  host_schedule_ = false;
  strategy_ = strategy;
}

void IepSession::set_schedule(const Schedule* schedule) {
  // programs staged by a pipelined set_programs are built first (their build
  // would otherwise drop this schedule), and the host CSR must describe them
  flush_programs();
  ensure_host_mirror();
  ++schedule_gen_;  // a host schedule's step count and tables are baked into a capture
  if (schedule) {
    if (kind_ == ModuleKind::resblock) check_reference_order(*schedule, batch_->csr());
    batch_->load_schedule(*schedule, stream_);
    host_schedule_ = true;
    strategy_ = schedule->strategy;
  } else {
    host_schedule_ = false;
    strategy_ = Strategy::improved;
  }
}

void IepSession::forward() {
  flush_programs();
  if (graphs_enabled()) {
    forward_graph();
    return;
  }
  forward_direct();
}

bool IepSession::graphs_enabled() const {
  static const bool env_on = [] {
    const char* e = std::getenv("DYNBATCH_GRAPH");
    return !e || std::atoi(e) != 0;
  }();
  // resblock forwards need no host sync (upper-bound step count), so they
  // capture; profiled forwards record per-class events and run directly
  return env_on && kind_ == ModuleKind::resblock && !prof_.on && !train_;
}

void IepSession::forward_graph() {
  const HostCSR& c = batch_->csr();
  const GraphKey key{c.b, c.N, rb_ ? rb_->n_shared : 0, c.s_max, static_cast<int>(strategy_),
                     host_schedule_ ? 1 : 0, rb_ ? rb_->tile_m : 0, batch_->static_shape() ? 1 : 0,
                     dbk_rb_debug_enabled(), kevents_ ? 1 : 0, schedule_gen_};
  ++graph_clock_;
  // a kept graph with step-kernel event nodes records this forward's events
  const auto launch = [this](CachedGraph& g) {
    kev_recorded_ = g.kb != nullptr;
    if (g.kb) {
      check(cudaGraphExecEventRecordNodeSetEvent(g.exec, g.kb, kev_cur_[0]), "event node");
      check(cudaGraphExecEventRecordNodeSetEvent(g.exec, g.ke, kev_cur_[1]), "event node");
    }
    check(cudaGraphLaunch(g.exec, stream_), "graph launch");
  };
  for (CachedGraph& g : graphs_) {
    if (!(g.key == key)) continue;
    batch_->set_sched_state(g.sched);
    launches_ = g.launches;
    g.used = graph_clock_;
    launch(g);
    return;
  }
  // capture this forward (its host bookkeeping runs once, here) and keep it
  cudaGraph_t graph = nullptr;
  cudaEvent_t cur[2] = {kev_cur_[0], kev_cur_[1]};
  if (kevents_) {
    for (cudaEvent_t& m : kev_mark_)
      if (!m) check(cudaEventCreate(&m), "event");
    kev_cur_[0] = kev_mark_[0];
    kev_cur_[1] = kev_mark_[1];
  }
  check(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal), "begin capture");
  try {
    forward_direct();
  } catch (...) {
    cudaStreamEndCapture(stream_, &graph);
    if (graph) cudaGraphDestroy(graph);
    kev_cur_[0] = cur[0];
    kev_cur_[1] = cur[1];
    throw;
  }
  kev_cur_[0] = cur[0];
  kev_cur_[1] = cur[1];
  check(cudaStreamEndCapture(stream_, &graph), "end capture");
  CachedGraph g;
  g.key = key;
  const cudaError_t e = cudaGraphInstantiate(&g.exec, graph, 0);
  if (e == cudaSuccess && kevents_ && kev_recorded_) {
    size_t n = 0;
    check(cudaGraphGetNodes(graph, nullptr, &n), "graph nodes");
    std::vector<cudaGraphNode_t> nodes(n);
    check(cudaGraphGetNodes(graph, nodes.data(), &n), "graph nodes");
    for (cudaGraphNode_t node : nodes) {
      cudaGraphNodeType t;
      check(cudaGraphNodeGetType(node, &t), "node type");
      if (t != cudaGraphNodeTypeEventRecord) continue;
      cudaEvent_t ev = nullptr;
      check(cudaGraphEventRecordNodeGetEvent(node, &ev), "event node");
      if (ev == kev_mark_[0]) g.kb = node;
      if (ev == kev_mark_[1]) g.ke = node;
    }
    if (g.kb && g.ke) g.graph = graph;
    else g.kb = g.ke = nullptr;
  }
  if (!g.graph) cudaGraphDestroy(graph);
  check(e, "graph instantiate");
  g.sched = batch_->sched_state();
  g.launches = launches_;
  g.used = graph_clock_;
  constexpr size_t kMaxGraphs = 4;  // e.g. the alternating program sets of a serving loop
  if (graphs_.size() >= kMaxGraphs) {
    auto lru = std::min_element(graphs_.begin(), graphs_.end(),
                                [](const CachedGraph& a, const CachedGraph& b) { return a.used < b.used; });
    release_graph(*lru);
    graphs_.erase(lru);
  }
  graphs_.push_back(g);
  launch(graphs_.back());
}

void IepSession::release_graph(CachedGraph& g) {
  if (g.exec) cudaGraphExecDestroy(g.exec);
  if (g.graph) cudaGraphDestroy(g.graph);
  g.exec = nullptr;
  g.graph = nullptr;
}

void IepSession::forward_direct() {
  launches_ = 0;
  check(cudaMemsetAsync(err_.get(), 0, sizeof(std::int32_t) * 4, stream_), "memset err");
  check(cudaMemsetAsync(present_.get(), 0, present_.size() * sizeof(std::int32_t), stream_), "memset present");
  if (!host_schedule_) {
    prof_.begin(0, stream_);
    batch_->run_scheduler(stream_, kind_ == ModuleKind::resblock, strategy_);  // resblock: no host sync
    prof_.end(stream_);
    launches_ += 4;  // labels, histogram, scan, scatter
  }
  if (kind_ == ModuleKind::dense) forward_dense(); else forward_resblock();
  if (prof_.on) add_forward_work();
}

// Algorithmic work per kernel class of one forward: FLOPs are
// 2·MAC of the module contractions; bytes are the minimum HBM traffic of
// each kernel (operands read once, results written once).
void IepSession::add_forward_work() {
  ensure_host_mirror();
  const HostCSR& c = batch_->csr();
  double n_un = 0, n_bin = 0, dense_flops = 0, dense_bytes = 0;
  for (std::int64_t g = 0; g < c.N; ++g) {
    const int a = c.arity_of[static_cast<size_t>(c.fid[static_cast<size_t>(g)])];
    if (a == 1) n_un += 1;
    if (a == 2) n_bin += 1;
    if (a > 0) {
      dense_flops += 2.0 * a * width_ * static_cast<double>(width_);
      dense_bytes += 8.0 * (a + 1) * width_;
    }
  }
  if (kind_ == ModuleKind::dense) {
    prof_.add_work(7, dense_flops, dense_bytes);
    return;
  }
  // Tier B: fp32 maps for inputs / roots / shared children, fp16 staged
  // images (225 positions × 256 B) for everything else; block inputs are
  // staged as hi + lo images (the residual).
  const double map32 = 100352.0, stage16 = 225.0 * 16 * 16;
  const double n_exp = n_un + n_bin;
  const double b = static_cast<double>(c.b);
  // gather: the operands no child epilogue forwards — leaves and children
  // with several parents — fp32 map → hi (+ lo for a unary member's input)
  std::vector<std::int32_t> parents(static_cast<size_t>(c.N), 0);
  for (std::int32_t ch : c.child_list) ++parents[static_cast<size_t>(ch)];
  double gather_bytes = 0.0;
  for (std::int64_t g = 0; g < c.N; ++g) {
    const int a = c.arity_of[static_cast<size_t>(c.fid[static_cast<size_t>(g)])];
    for (std::int32_t e = c.child_off[static_cast<size_t>(g)]; e < c.child_off[static_cast<size_t>(g) + 1]; ++e) {
      const std::int32_t ch = c.child_list[static_cast<size_t>(e)];
      const bool leaf = c.arity_of[static_cast<size_t>(c.fid[static_cast<size_t>(ch)])] == 0;
      if (leaf || parents[static_cast<size_t>(ch)] > 1) gather_bytes += map32 + (a == 1 ? 2 : 1) * stage16;
    }
  }
  prof_.add_work(2, 0.0, gather_bytes);
  // fused conv step: conv1x1 (binary) + conv3x3 #1 + conv3x3 #2 with the
  // residual; reads x hi, mid, hi/lo; writes mid, hi/lo images (roots: fp32)
  const double conv_flops = n_bin * 12845056.0 + n_exp * 2 * 57802752.0;
  const double conv_bytes = n_bin * (2 * stage16 + 2 * stage16) + n_exp * (stage16 + stage16) +
                            n_exp * (3 * stage16) + (n_exp - b) * 2 * stage16 + b * map32;
  prof_.add_work(4, conv_flops, conv_bytes);
}

double IepSession::time_forwards(int iters, int profile, KernelTimes* kt) {
  synchronize();
  prof_.on = profile == 1;
  prof_.reset();
  const bool kev = profile == 2 && kind_ == ModuleKind::resblock;
  if (kev)
    while (kev_pool_.size() < 2 * static_cast<size_t>(std::max(iters, 0))) {
      cudaEvent_t e;
      check(cudaEventCreate(&e), "event");
      kev_pool_.push_back(e);
    }
  kevents_ = kev;
  std::vector<char> recorded(static_cast<size_t>(std::max(iters, 0)), 0);
  cudaEvent_t a, b;
  check(cudaEventCreate(&a), "event");
  check(cudaEventCreate(&b), "event");
  check(cudaEventRecord(a, stream_), "event");
  try {
    for (int i = 0; i < iters; ++i) {
      if (kev) {
        kev_cur_[0] = kev_pool_[2 * static_cast<size_t>(i)];
        kev_cur_[1] = kev_pool_[2 * static_cast<size_t>(i) + 1];
        kev_recorded_ = false;
      }
      forward();
      if (kev) recorded[static_cast<size_t>(i)] = kev_recorded_ ? 1 : 0;
    }
  } catch (...) {
    kevents_ = false;
    kev_cur_[0] = kev_cur_[1] = nullptr;
    throw;
  }
  kevents_ = false;
  kev_cur_[0] = kev_cur_[1] = nullptr;
  check(cudaEventRecord(b, stream_), "event");
  check(cudaEventSynchronize(b), "event sync");
  float ms = 0.f;
  check(cudaEventElapsedTime(&ms, a, b), "elapsed");
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  check_errors();
  if (profile == 1 && kt) *kt = prof_.collect();
  if (kev && kt) {
    // the step kernel's events of every forward that recorded them, and the
    // algorithmic work of those forwards (same accounting as profile 1)
    prof_.reset();
    KernelTimes w;
    std::int64_t n = 0;
    double step_ms = 0.0;
    for (int i = 0; i < iters; ++i) {
      if (!recorded[static_cast<size_t>(i)]) continue;
      float t = 0.f;
      check(cudaEventElapsedTime(&t, kev_pool_[2 * static_cast<size_t>(i)], kev_pool_[2 * static_cast<size_t>(i) + 1]),
            "elapsed");
      step_ms += t;
      ++n;
    }
    if (n > 0) {
      add_forward_work();
      w = prof_.collect();
    }
    *kt = KernelTimes{};
    kt->ms[4] = step_ms;
    kt->launches[4] = n;
    kt->flops[4] = w.flops[4] * static_cast<double>(n);
    kt->bytes[4] = w.bytes[4] * static_cast<double>(n);
  }
  prof_.on = false;
  return ms;
}

void IepSession::forward_dense() {
  const HostCSR& c = batch_->csr();
  const int blocks = std::min<std::int64_t>(std::max<std::int64_t>(1, (c.N + 7) / 8), sm_count() * 16);
  for (int st = 0; st < batch_->steps; ++st) {
    prof_.begin(7, stream_);
    check(dbk_dense_step(st, width_, batch_->step_group_begin.get(), batch_->group_fid.get(),
                         batch_->group_begin.get(), batch_->member_g.get(), batch_->arity_of.get(),
                         batch_->child_off.get(), batch_->child_list.get(), batch_->example.get(),
                         in64_.get(), values64_.get(), present_.get(), wtab_.get(), btab_.get(),
                         err_.get(), std::max(1, c.max_arity), blocks, stream_),
          "dbk_dense_step");
    prof_.end(stream_);
    ++launches_;
  }
  check(dbk_dense_gather_roots(c.b, width_, batch_->root_g.get(), present_.get(),
                               values64_.get(), out64_.get(), err_.get(), stream_),
        "dbk_dense_gather_roots");
  ++launches_;
}

void IepSession::check_errors() {
  batch_->check_scheduler_error(stream_);
  std::int32_t e = 0;
  check(cudaMemcpyAsync(&e, err_.get(), sizeof(e), cudaMemcpyDeviceToHost, stream_), "D2H err");
  check(cudaStreamSynchronize(stream_), "sync");
  switch (e) {
    case 0: return;
    case 7: throw_error(Errc::missing_operand, "a call group read a node that was not yet computed");
    case 9: throw_error(Errc::non_finite_value, "a module produced non-finite rows (or rows beyond the fp16 operand "
                                                "range of the conv kernels)");
    case 10: throw_error(Errc::non_finite_value, "an input is non-finite or beyond the fp16 operand range of the conv "
                                                 "kernels (|x| > 65504)");
    case 14: throw_error(Errc::single_assignment_violation, "a node was written twice");
    default: throw std::runtime_error("device executor error " + std::to_string(e));
  }
}

void IepSession::synchronize() {
  check(cudaStreamSynchronize(stream_), "sync");
  sync_pipeline();
  check_errors();
}

Schedule IepSession::download_schedule() {
  batch_->resolve(stream_);
  ensure_host_mirror();
  return batch_->download_schedule(strategy_, stream_);
}

std::vector<std::int32_t> IepSession::download_labels() { return batch_->download_labels(stream_); }

TensorBatch IepSession::download_outputs() {
  synchronize();
  const HostCSR& c = batch_->csr();
  TensorBatch out(c.b, width_);
  if (c.b == 0) return out;
  if (kind_ == ModuleKind::dense) {
    check(cudaMemcpyAsync(out.data().data(), out64_.get(), sizeof(double) * out.data().size(),
                          cudaMemcpyDeviceToHost, stream_), "D2H outputs");
    check(cudaStreamSynchronize(stream_), "sync");
  } else {
    std::vector<float> tmp(out.data().size());
    download_resblock_outputs(tmp.data());
    for (size_t i = 0; i < tmp.size(); ++i) out.data()[i] = tmp[i];
  }
  return out;
}

ExecutionTrace IepSession::trace() {
  ExecutionTrace t = batch_->trace_counts(stream_);
  t.per_step_seconds.assign(static_cast<size_t>(batch_->steps), 0.0);
  return t;
}

double IepSession::algorithmic_flops() const {
  const HostCSR& c = batch_->csr();
  double f = 0.0;
  for (std::int64_t g = 0; g < c.N; ++g) {
    const int fid = c.fid[static_cast<size_t>(g)];
    const int a = c.arity_of[static_cast<size_t>(fid)];
    if (a == 0) continue;
    if (kind_ == ModuleKind::dense) {
      f += 2.0 * a * width_ * static_cast<double>(width_);
    } else {
      // 2·MAC of the convolutions only: conv3x3 ×2 on
      // 128×14×14 = 115,605,504; binary adds conv1x1 256→128 = 12,845,056.
      f += a == 2 ? 128450560.0 : 115605504.0;
    }
  }
  return f;
}

double IepSession::algorithmic_bytes() const {
  const HostCSR& c = batch_->csr();
  const double row = (kind_ == ModuleKind::dense ? 8.0 : 4.0) * width_;
  double bytes = 0.0;
  for (std::int64_t g = 0; g < c.N; ++g) {
    const int a = c.arity_of[static_cast<size_t>(c.fid[static_cast<size_t>(g)])];
    if (a > 0) bytes += (a + 1) * row;  // read operands, write result
  }
  return bytes;
}

std::int64_t IepSession::h2d_bytes() const { return batch_->csr().b * width_ * 4; }
std::int64_t IepSession::d2h_bytes() const { return batch_->csr().b * width_ * 4; }

}  // namespace dynbatch::dev
