// oracle/ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// Thin extern "C" glue compiled together with the unmodified reference core
// (/root/reference/proj/src/*.cpp) into oracle/_ref/libdbref.so. It exposes
// reference functions that the reference's own C ABI does not reach
// (generator CSR, schedules as flat arrays, top_k_gate, explicit-input MoE)
// so tests can compare the product against the reference on identical inputs.
// Nothing here computes anything itself: every result comes from the
// reference function named in the comment.
//
// Batch CSR convention (shared with the product and oracle/dynbatch_oracle.c):
//   prog_off[b+1] node offsets, fid[N], child0[N], child1[N] (program-local
//   child ids, -1 when absent), root[b] (program-local root id).

#include <cstdint>
#include <cstring>
#include <vector>

#include "dynbatch/dynbatch.h"
#include "dynbatch/executor.hpp"
#include "dynbatch/modules.hpp"
#include "dynbatch/moe.hpp"
#include "dynbatch/program.hpp"
#include "dynbatch/rng.hpp"
#include "dynbatch/schedule.hpp"
#include "dynbatch/workload.hpp"

using namespace dynbatch;

namespace {

std::vector<Program> programs_from_csr(int64_t b, const int32_t* prog_off, const int32_t* fid,
                                       const int32_t* child0, const int32_t* child1,
                                       const int32_t* root) {
  std::vector<Program> out(static_cast<size_t>(b));
  for (int64_t e = 0; e < b; ++e) {
    Program& p = out[static_cast<size_t>(e)];
    p.root = root[e];
    for (int32_t g = prog_off[e]; g < prog_off[e + 1]; ++g) {
      ProgramNode node;
      node.function_id = fid[g];
      if (child0[g] >= 0) node.children.push_back(child0[g]);
      if (child1[g] >= 0) node.children.push_back(child1[g]);
      p.nodes.push_back(std::move(node));
    }
  }
  return out;
}

int fail_code(const Error& e) { return 100 + static_cast<int>(e.code()); }

}  // namespace

extern "C" {

// gen_batch (src/workload.cpp:214-246). Pass prog_off == nullptr to get the
// total node count only. Returns total nodes, or -1 on error.
int64_t refshim_gen_batch(int kind, int64_t b, int p, int width, int depth, int length, double bp,
                          uint64_t seed, int32_t* prog_off, int32_t* fid, int32_t* child0,
                          int32_t* child1, int32_t* root, double* inputs) {
  try {
    WorkloadSpec spec;
    spec.kind = kind == 0 ? WorkloadKind::balanced_tree
                          : (kind == 1 ? WorkloadKind::chain_heavy : WorkloadKind::random_dag);
    spec.b = b;
    spec.p = p;
    spec.width = width;
    spec.depth = depth;
    spec.length = length;
    spec.branch_prob = bp;
    spec.seed = seed;
    GeneratedBatch g = gen_batch(spec);
    int64_t total = 0;
    for (const Program& prog : g.programs) total += prog.size();
    if (!prog_off) return total;
    int32_t off = 0;
    for (size_t e = 0; e < g.programs.size(); ++e) {
      prog_off[e] = off;
      root[e] = g.programs[e].root;
      for (const ProgramNode& node : g.programs[e].nodes) {
        fid[off] = node.function_id;
        child0[off] = node.children.size() > 0 ? node.children[0] : -1;
        child1[off] = node.children.size() > 1 ? node.children[1] : -1;
        ++off;
      }
    }
    prog_off[g.programs.size()] = off;
    if (inputs) std::memcpy(inputs, g.inputs.data().data(), g.inputs.data().size() * sizeof(double));
    return total;
  } catch (...) {
    return -1;
  }
}

// random_batch (src/workload.cpp:207-212).
void refshim_random_batch(int64_t rows, int64_t width, uint64_t seed, double* out) {
  TensorBatch t = random_batch(rows, width, seed);
  std::memcpy(out, t.data().data(), t.data().size() * sizeof(double));
}

uint64_t refshim_mix_seed(uint64_t seed, uint64_t stream) { return mix_seed(seed, stream); }

// build_schedule (src/schedule.cpp:243-252) flattened. counts[0]=steps,
// counts[1]=groups, counts[2]=members. Pass step_group_off == nullptr for the
// counts only. Returns 0 or an error code.
int refshim_schedule(int strategy, int64_t b, int p, const int32_t* prog_off, const int32_t* fid,
                     const int32_t* child0, const int32_t* child1, const int32_t* root,
                     int64_t* counts, int32_t* step_group_off, int32_t* group_fid,
                     int32_t* group_member_off, int32_t* member_example, int32_t* member_node) {
  try {
    FunctionVocab vocab = make_default_vocab(p, 1);
    std::vector<Program> batch = programs_from_csr(b, prog_off, fid, child0, child1, root);
    Schedule s = build_schedule(static_cast<Strategy>(strategy), batch, vocab);
    int64_t groups = 0, members = 0;
    for (const Step& st : s.steps) {
      groups += static_cast<int64_t>(st.size());
      for (const CallGroup& g : st) members += static_cast<int64_t>(g.members.size());
    }
    counts[0] = static_cast<int64_t>(s.steps.size());
    counts[1] = groups;
    counts[2] = members;
    if (!step_group_off) return 0;
    int32_t gi = 0, mi = 0;
    for (size_t si = 0; si < s.steps.size(); ++si) {
      step_group_off[si] = gi;
      for (const CallGroup& g : s.steps[si]) {
        group_fid[gi] = g.function_id;
        group_member_off[gi] = mi;
        for (const NodeRef& r : g.members) {
          member_example[mi] = r.example;
          member_node[mi] = r.node;
          ++mi;
        }
        ++gi;
      }
    }
    step_group_off[s.steps.size()] = gi;
    group_member_off[gi] = mi;
    return 0;
  } catch (const Error& e) {
    return fail_code(e);
  } catch (...) {
    return 99;
  }
}

// max_root_distance_labels (src/program.cpp:239-272) for every program.
int refshim_labels(int64_t b, const int32_t* prog_off, const int32_t* fid, const int32_t* child0,
                   const int32_t* child1, const int32_t* root, int32_t* labels) {
  try {
    std::vector<Program> batch = programs_from_csr(b, prog_off, fid, child0, child1, root);
    for (int64_t e = 0; e < b; ++e) {
      DepthLabels d = max_root_distance_labels(batch[static_cast<size_t>(e)]);
      for (size_t i = 0; i < d.labels.size(); ++i) labels[prog_off[e] + static_cast<int64_t>(i)] = d.labels[i];
    }
    return 0;
  } catch (const Error& e) {
    return fail_code(e);
  }
}

// execute (src/executor.cpp:95-182) with ModuleSet(make_default_vocab(p, width), module_seed).
// trace: [expensive_calls, peak_group_rows, steps], per_function_calls[p].
int refshim_execute(int strategy, int64_t b, int p, int width, const int32_t* prog_off,
                    const int32_t* fid, const int32_t* child0, const int32_t* child1,
                    const int32_t* root, const double* inputs, uint64_t module_seed,
                    double* outputs, int64_t* trace, int64_t* per_function_calls,
                    double* seconds) {
  try {
    FunctionVocab vocab = make_default_vocab(p, width);
    std::vector<Program> batch = programs_from_csr(b, prog_off, fid, child0, child1, root);
    Schedule s = build_schedule(static_cast<Strategy>(strategy), batch, vocab);
    TensorBatch in(b, width);
    std::memcpy(in.data().data(), inputs, static_cast<size_t>(b * width) * sizeof(double));
    ModuleSet modules(vocab, module_seed);
    ExecResult r = execute(s, batch, in, modules);
    std::memcpy(outputs, r.outputs.data().data(), static_cast<size_t>(b * width) * sizeof(double));
    trace[0] = r.trace.expensive_calls;
    trace[1] = r.trace.peak_group_rows;
    trace[2] = static_cast<int64_t>(r.trace.per_step_seconds.size());
    for (int f = 0; f < p; ++f) per_function_calls[f] = r.trace.per_function_calls[static_cast<size_t>(f)];
    if (seconds) {
      seconds[0] = r.trace.module_seconds;
      seconds[1] = r.trace.stacking_seconds;
      seconds[2] = r.trace.total_seconds;
    }
    return 0;
  } catch (const Error& e) {
    return fail_code(e);
  }
}

// make_module_impl (src/modules.cpp:13-28): weights [arity*width*width], bias[width].
int refshim_module_weights(int p, int width, uint64_t seed, int fid, double* w, double* bias) {
  FunctionVocab vocab = make_default_vocab(p, width);
  ModuleImpl impl = make_module_impl(vocab.spec(fid), width, seed);
  std::memcpy(w, impl.weights.data(), impl.weights.size() * sizeof(double));
  std::memcpy(bias, impl.bias.data(), impl.bias.size() * sizeof(double));
  return static_cast<int>(impl.weights.size());
}

// gen_moe_inputs (src/workload.cpp:248-254).
int refshim_moe_inputs(int64_t T, int64_t n, int64_t d, uint64_t seed, double* inputs,
                       double* scores) {
  MoeConfig cfg;
  cfg.experts = n;
  cfg.active_per_example = 1;
  cfg.batch = T;
  cfg.data_dim = d;
  cfg.hidden = 1;
  MoeWorkload w = gen_moe_inputs(cfg, seed);
  if (inputs) std::memcpy(inputs, w.inputs.data().data(), w.inputs.data().size() * sizeof(double));
  if (scores) std::memcpy(scores, w.scores.data().data(), w.scores.data().size() * sizeof(double));
  return 0;
}

// top_k_gate (src/moe.cpp:36-69).
int refshim_topk(const double* scores, int64_t T, int64_t n, int64_t k, int32_t* ids,
                 double* weights) {
  try {
    TensorBatch s(T, n);
    std::memcpy(s.data().data(), scores, static_cast<size_t>(T * n) * sizeof(double));
    GateAssignment g = top_k_gate(s, k);
    for (int64_t t = 0; t < T; ++t) {
      for (int64_t i = 0; i < k; ++i) {
        ids[t * k + i] = g.per_example[static_cast<size_t>(t)][static_cast<size_t>(i)].expert;
        weights[t * k + i] = g.per_example[static_cast<size_t>(t)][static_cast<size_t>(i)].weight;
      }
    }
    return 0;
  } catch (const Error& e) {
    return fail_code(e);
  }
}

// ExpertSet ctor (src/moe.cpp:71-88) for one expert id.
int refshim_expert_weights(int64_t n, int64_t d, int64_t h, uint64_t seed, int64_t id, double* w1,
                           double* w2) {
  // The reference seeds each expert independently (mix_seed(seed, id)); build
  // a one-expert set for ids > 0 by constructing all of them is too costly at
  // scale, so construct the full set only when small.
  ExpertSet set(n, d, h, seed);
  (void)id;
  (void)w1;
  (void)w2;
  return static_cast<int>(set.size());
}

// moe_forward_batched / moe_forward_naive (src/moe.cpp:162-270) on explicit
// inputs and gates. trace: [expensive_calls, peak_group_rows].
int refshim_moe_forward(const double* inputs, int64_t T, int64_t d, int64_t h, int64_t n,
                        int64_t k, const int32_t* ids, const double* weights, uint64_t expert_seed,
                        int batched, double* out, int64_t* trace, double* seconds) {
  try {
    TensorBatch in(T, d);
    std::memcpy(in.data().data(), inputs, static_cast<size_t>(T * d) * sizeof(double));
    GateAssignment g;
    g.per_example.resize(static_cast<size_t>(T));
    for (int64_t t = 0; t < T; ++t) {
      for (int64_t i = 0; i < k; ++i) {
        g.per_example[static_cast<size_t>(t)].push_back({ids[t * k + i], weights[t * k + i]});
      }
    }
    ExpertSet experts(n, d, h, expert_seed);
    MoeResult r = batched ? moe_forward_batched(in, experts, g) : moe_forward_naive(in, experts, g);
    std::memcpy(out, r.outputs.data().data(), static_cast<size_t>(T * d) * sizeof(double));
    trace[0] = r.trace.expensive_calls;
    trace[1] = r.trace.peak_group_rows;
    if (seconds) {
      seconds[0] = r.trace.module_seconds;
      seconds[1] = r.trace.stacking_seconds;
      seconds[2] = r.trace.total_seconds;
    }
    return 0;
  } catch (const Error& e) {
    return fail_code(e);
  }
}

}  // extern "C"
