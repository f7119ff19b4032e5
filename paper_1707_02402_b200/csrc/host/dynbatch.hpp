// dynbatch.hpp — C++ operator API of the B200-native executor (host side).
//
// Mirrors the reference's C++ surface (include/dynbatch/{error,rng,tensor,
// program,schedule,modules,executor,moe,workload,serialize,verify}.hpp) with
// the same names, argument meaning and error behaviour, so code written
// against the reference compiles against this. The compute entry points
// (schedule_improved, execute, top_k_gate, moe_forward_batched) run on the
// current CUDA device through the thin dbk_* C-ABI (include/dynbatch/dbk.h);
// the host keeps only fixture generation, validation, host-side schedules
// (naive/standard/online, which the device executor can still run) and
// serialization.
#pragma once

#include <cstdint>
#include <functional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

namespace dynbatch {

// ------------------------------------------------------------------ errors
// Error codes and their printed names follow include/dynbatch/error.hpp:11-46
// and src/program.cpp:12-33 (messages are prefixed with the name).
enum class Errc {
  ok = 0,
  invalid_argument,
  unknown_function,
  underfull_sequence,
  overfull_sequence,
  invalid_program,
  dependency_violation,
  missing_operand,
  row_count_mismatch,
  width_mismatch,
  arity_mismatch,
  non_finite_value,
  k_too_large,
  vocab_missing_arity,
  single_assignment_violation,
  parse_error,
  verification_failed,
};

const char* errc_name(Errc code);

class Error : public std::runtime_error {
 public:
  Error(Errc code, const std::string& what)
      : std::runtime_error(std::string(errc_name(code)) + ": " + what), code_(code) {}
  Errc code() const { return code_; }

 private:
  Errc code_;
};

[[noreturn]] void throw_error(Errc code, const std::string& what);

// -------------------------------------------------------------------- rng
// mt19937_64 with the reference's explicit mappings (include/dynbatch/rng.hpp).
std::uint64_t splitmix64(std::uint64_t& state);
std::uint64_t mix_seed(std::uint64_t seed, std::uint64_t stream);

class Rng {
 public:
  explicit Rng(std::uint64_t seed);
  std::uint64_t next_u64();
  double uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  std::int64_t uniform_int(std::int64_t lo, std::int64_t hi) {
    const std::uint64_t span = static_cast<std::uint64_t>(hi - lo) + 1;
    return lo + static_cast<std::int64_t>(next_u64() % span);
  }
  bool bernoulli(double p) { return uniform() < p; }
  // Skips n outputs (whole 312-word blocks are regenerated without tempering).
  void discard(std::uint64_t n);

 private:
  void twist();
  std::uint64_t state_[312];
  int pos_;
};

// ----------------------------------------------------------------- tensor
// Row-major rows × width fp64 matrix (include/dynbatch/tensor.hpp).
class TensorBatch {
 public:
  TensorBatch() = default;
  TensorBatch(std::int64_t rows, std::int64_t width);
  std::int64_t rows() const { return rows_; }
  std::int64_t width() const { return width_; }
  double& at(std::int64_t r, std::int64_t c) { return data_[static_cast<size_t>(r * width_ + c)]; }
  double at(std::int64_t r, std::int64_t c) const { return data_[static_cast<size_t>(r * width_ + c)]; }
  std::span<double> row(std::int64_t r) { return {data_.data() + r * width_, static_cast<size_t>(width_)}; }
  std::span<const double> row(std::int64_t r) const {
    return {data_.data() + r * width_, static_cast<size_t>(width_)};
  }
  std::span<double> data() { return data_; }
  std::span<const double> data() const { return data_; }
  bool all_finite() const;
  friend bool operator==(const TensorBatch&, const TensorBatch&) = default;

 private:
  std::int64_t rows_ = 0;
  std::int64_t width_ = 0;
  std::vector<double> data_;
};

// --------------------------------------------------------------- programs
enum class CostClass { expensive, free };

struct ModuleSpec {
  int function_id = 0;
  int arity = 0;
  int in_width = 0;
  int out_width = 0;
  CostClass cost = CostClass::free;
  bool is_expensive() const { return cost == CostClass::expensive; }
};

class FunctionVocab {
 public:
  FunctionVocab() = default;
  explicit FunctionVocab(std::vector<ModuleSpec> specs);
  int size() const { return static_cast<int>(specs_.size()); }
  int width() const { return width_; }
  bool contains(int fid) const { return fid >= 0 && fid < size(); }
  const ModuleSpec& spec(int fid) const;
  const std::vector<ModuleSpec>& specs() const { return specs_; }

 private:
  std::vector<ModuleSpec> specs_;
  int width_ = 0;
};

struct ProgramNode {
  int function_id = 0;
  std::vector<int> children;
  friend bool operator==(const ProgramNode&, const ProgramNode&) = default;
};

struct Program {
  std::vector<ProgramNode> nodes;
  int root = 0;
  int size() const { return static_cast<int>(nodes.size()); }
};

struct DepthLabels {
  std::vector<int> labels;
  int max_label = 0;
};

enum class ViolationKind {
  bad_root,
  unknown_function,
  bad_child_ref,
  arity_mismatch,
  cycle_detected,
  unreachable_node,
  free_cost_required,
};
const char* violation_name(ViolationKind kind);

struct Violation {
  ViolationKind kind;
  std::string detail;
};

struct ValidationReport {
  std::vector<Violation> violations;
  bool ok() const { return violations.empty(); }
  std::string to_string() const;
};

Program build_program_from_prefix(std::span<const int> functions, const FunctionVocab& vocab);
ValidationReport validate(const Program& program, const FunctionVocab& vocab);
DepthLabels max_root_distance_labels(const Program& program);
std::vector<int> postorder_flatten(const Program& program);
std::vector<int> prefix_function_sequence(const Program& program);

// -------------------------------------------------------------- schedules
struct NodeRef {
  std::int32_t example = 0;
  std::int32_t node = 0;
  friend auto operator<=>(const NodeRef&, const NodeRef&) = default;
};

struct CallGroup {
  int function_id = 0;
  std::vector<NodeRef> members;
  friend bool operator==(const CallGroup&, const CallGroup&) = default;
};

using Step = std::vector<CallGroup>;

enum class Strategy { naive, standard, improved, online };
const char* strategy_name(Strategy s);
Strategy strategy_from_name(const std::string& name);

struct Schedule {
  Strategy strategy = Strategy::naive;
  std::vector<Step> steps;
  friend bool operator==(const Schedule&, const Schedule&) = default;
};

struct BatchStats {
  std::int64_t b = 0, p = 0, s_max = 0, d_max = 0;
};

struct FrontierItem {
  NodeRef ref;
  int function_id = 0;
};

enum class ScheduleViolationKind {
  invalid_ref,
  function_mismatch,
  empty_group,
  duplicate_execution,
  missing_execution,
  dependency_order_violation,
};
const char* schedule_violation_name(ScheduleViolationKind kind);

struct ScheduleViolation {
  ScheduleViolationKind kind;
  std::string detail;
};

struct ScheduleReport {
  std::vector<ScheduleViolation> violations;
  bool ok() const { return violations.empty(); }
  std::string to_string() const;
};

BatchStats compute_batch_stats(std::span<const Program> batch, const FunctionVocab& vocab);
Schedule schedule_naive(std::span<const Program> batch, const FunctionVocab& vocab);
Schedule schedule_standard(std::span<const Program> batch, const FunctionVocab& vocab);
// Device scheduler (dbk_schedule_*): bit-identical to the reference's.
Schedule schedule_improved(std::span<const Program> batch, const FunctionVocab& vocab);
// Device-built improved / standard / online schedule (same result as the
// host builders, bit for bit).
Schedule schedule_device(Strategy strategy, std::span<const Program> batch, const FunctionVocab& vocab);
Step group_by_function(std::span<const FrontierItem> items);
Step schedule_online(std::span<const Program> batch, std::span<const NodeRef> frontier,
                     const std::function<bool(NodeRef)>& already_executed,
                     const FunctionVocab& vocab);
Schedule schedule_online_full(std::span<const Program> batch, const FunctionVocab& vocab);
Schedule build_schedule(Strategy strategy, std::span<const Program> batch,
                        const FunctionVocab& vocab);
ScheduleReport verify_schedule(const Schedule& schedule, std::span<const Program> batch);
std::int64_t count_expensive_calls(const Schedule& schedule, const FunctionVocab& vocab);
std::int64_t count_expensive_nodes(std::span<const Program> batch, const FunctionVocab& vocab);
std::int64_t count_total_nodes(std::span<const Program> batch);
void require_valid_batch(std::span<const Program> batch, const FunctionVocab& vocab);

// ---------------------------------------------------------------- modules
// Dense module (src/modules.cpp:13-28): input-major weights, per-fid seeds.
struct ModuleImpl {
  ModuleSpec spec;
  std::vector<double> weights;
  std::vector<double> bias;
};
ModuleImpl make_module_impl(const ModuleSpec& spec, int width, std::uint64_t seed);

// One module call on stacked operand rows (src/modules.cpp:52-108; runs on
// the device, bit-identical to execute()).
TensorBatch apply_module(const ModuleImpl& impl, std::span<const TensorBatch> operands);

class ModuleSet {
 public:
  ModuleSet(const FunctionVocab& vocab, std::uint64_t seed);
  const ModuleImpl& impl(int fid) const;
  int size() const { return static_cast<int>(impls_.size()); }
  int width() const { return width_; }
  std::uint64_t seed() const { return seed_; }
  std::int64_t weight_element_count() const;

 private:
  std::vector<ModuleImpl> impls_;
  int width_ = 0;
  std::uint64_t seed_ = 0;
};

// Residual conv block weights (north-star module body; not in the
// reference). Draw order w0, b0 (binary), w1, b1, w2, b2; input-major
// w[(tap*Cin + ci)*C + co]; scale 1/sqrt(fan_in).
struct ResBlockImpl {
  int arity = 0;
  std::vector<double> w0, b0, w1, b1, w2, b2;
};
ResBlockImpl make_resblock_impl(int arity, int channels, std::uint64_t seed, int fid);

// --------------------------------------------------------------- executor
// Single-assignment store of per-node rows (src/executor.cpp:26-70): the
// reference executor's host container. Reading an absent node throws
// MissingOperand; writing a node twice throws SingleAssignmentViolation.
class ValueStore {
 public:
  ValueStore(std::span<const Program> batch, std::int64_t width);
  std::int64_t width() const { return width_; }
  bool has(NodeRef ref) const;
  std::span<const double> row(NodeRef ref) const;
  void set(NodeRef ref, std::span<const double> value);

 private:
  void check_ref(NodeRef ref) const;
  std::int64_t width_;
  std::vector<std::vector<double>> values_;
  std::vector<std::vector<char>> present_;
};
TensorBatch gather_rows(const ValueStore& store, std::span<const NodeRef> refs);
void scatter_rows(ValueStore& store, std::span<const NodeRef> refs, const TensorBatch& values);

struct ExecutionTrace {
  std::int64_t expensive_calls = 0;
  std::vector<std::int64_t> per_function_calls;
  std::vector<double> per_step_seconds;
  double module_seconds = 0.0;
  double stacking_seconds = 0.0;
  double total_seconds = 0.0;
  std::int64_t peak_group_rows = 0;
};

struct ExecResult {
  TensorBatch outputs;
  ExecutionTrace trace;
};

// Device execution of a (host) schedule with the dense module set.
ExecResult execute(const Schedule& schedule, std::span<const Program> batch,
                   const TensorBatch& inputs, const ModuleSet& modules);
ExecResult execute(const Schedule& schedule, std::span<const Program> batch,
                   const TensorBatch& inputs, const FunctionVocab& vocab, std::uint64_t seed);

// -------------------------------------------------------------------- MoE
struct MoeConfig {
  std::int64_t experts = 1;
  std::int64_t active_per_example = 1;
  std::int64_t batch = 1;
  std::int64_t data_dim = 1;
  std::int64_t hidden = 1;
  double examples_per_expert = 0.0;
  void check() const;
};

struct GateEntry {
  int expert = 0;
  double weight = 0.0;
};

struct GateAssignment {
  std::vector<std::vector<GateEntry>> per_example;
};

// Device top-k gate (dbk_moe_topk): ranks by (score desc, id asc).
GateAssignment top_k_gate(const TensorBatch& scores, std::int64_t k);

struct Expert {
  std::vector<double> w1;  // d × h input-major
  std::vector<double> w2;  // h × d input-major
};

class ExpertSet {
 public:
  ExpertSet(std::int64_t experts, std::int64_t data_dim, std::int64_t hidden, std::uint64_t seed);
  std::int64_t size() const { return static_cast<std::int64_t>(experts_.size()); }
  std::int64_t data_dim() const { return data_dim_; }
  std::int64_t hidden() const { return hidden_; }
  std::uint64_t seed() const { return seed_; }
  std::int64_t weight_element_count() const;
  const Expert& expert(std::int64_t id) const { return experts_[static_cast<size_t>(id)]; }
  // relu(rows · W1) · W2 for one expert (src/moe.cpp:98-145; on the device)
  TensorBatch apply(std::int64_t expert_id, const TensorBatch& rows) const;

 private:
  std::vector<Expert> experts_;
  std::int64_t data_dim_;
  std::int64_t hidden_;
  std::uint64_t seed_;
};

struct MoeResult {
  TensorBatch outputs;
  ExecutionTrace trace;
};

// Both run on the device in the reference's fp64 arithmetic order; naive
// issues one single-row expert call per assignment (k·b calls).
MoeResult moe_forward_naive(const TensorBatch& inputs, const ExpertSet& experts,
                            const GateAssignment& gates);
MoeResult moe_forward_batched(const TensorBatch& inputs, const ExpertSet& experts,
                              const GateAssignment& gates);

std::int64_t moe_param_count(const MoeConfig& cfg);
double moe_activation_count(const MoeConfig& cfg);
double moe_memory_ratio(const MoeConfig& cfg);

// -------------------------------------------------------------- workloads
enum class WorkloadKind { balanced_tree, chain_heavy, random_dag, moe };
const char* workload_kind_name(WorkloadKind kind);
WorkloadKind workload_kind_from_name(const std::string& name);

struct WorkloadSpec {
  WorkloadKind kind = WorkloadKind::chain_heavy;
  std::int64_t b = 1;
  int p = 8;
  int width = 8;
  int depth = 4;
  int length = 8;
  double branch_prob = 0.1;
  std::uint64_t seed = 0;
};

FunctionVocab make_default_vocab(int p, int width);
Program gen_balanced_tree(int depth, const FunctionVocab& vocab, std::uint64_t seed);
Program gen_chain_heavy(int length, double branch_prob, const FunctionVocab& vocab,
                        std::uint64_t seed);
Program gen_random_dag(int length, double share_prob, const FunctionVocab& vocab,
                       std::uint64_t seed);

struct GeneratedBatch {
  FunctionVocab vocab;
  std::vector<Program> programs;
  TensorBatch inputs;
};
GeneratedBatch gen_batch(const WorkloadSpec& spec);
GeneratedBatch gen_batch_range(const WorkloadSpec& spec, std::int64_t first, std::int64_t last);
TensorBatch random_batch(std::int64_t rows, std::int64_t width, std::uint64_t seed);
// Rows [first, last) of random_batch(rows, width, seed), bit-identical.
TensorBatch random_batch_range(std::int64_t first, std::int64_t last, std::int64_t width, std::uint64_t seed);

struct MoeWorkload {
  TensorBatch inputs;
  TensorBatch scores;
};
MoeWorkload gen_moe_inputs(const MoeConfig& cfg, std::uint64_t seed);

// ---------------------------------------------------------- serialization
struct ProgramSet {
  FunctionVocab vocab;
  std::vector<Program> programs;
};
std::string program_set_to_json(const FunctionVocab& vocab, std::span<const Program> programs);
ProgramSet program_set_from_json(const std::string& text, int width);
std::string schedule_to_json(const Schedule& schedule);
std::string trace_to_json(const ExecutionTrace& trace);
std::string workload_spec_to_json(const WorkloadSpec& spec);
WorkloadSpec workload_spec_from_json(const std::string& text);
std::string moe_config_to_json(const MoeConfig& cfg);
MoeConfig moe_config_from_json(const std::string& text);

// ----------------------------------------------------------- verification
struct VerifyOptions {
  int seeds = 100;
  std::int64_t b = 8;
  int p = 12;
  int length = 12;
  int width = 8;
  std::uint64_t base_seed = 0;
  bool parallel = false;
};

struct VerifyReport {
  int cases_run = 0;
  std::vector<std::string> failures;
  bool ok() const { return failures.empty(); }
};

VerifyReport run_property_suite(const VerifyOptions& options,
                                const std::function<void(const std::string&)>& log = {});

}  // namespace dynbatch
