// program.cpp — errors, RNG, TensorBatch, vocabulary and program graphs.
//
// Behaviour follows the reference (file:line under /root/reference/proj):
//   errc_name ............ src/program.cpp:12-33
//   Rng / mix_seed ....... include/dynbatch/rng.hpp:11-50
//   FunctionVocab ........ src/program.cpp:58-93
//   build_program_from_prefix  src/program.cpp:95-142
//   validate ............. src/program.cpp:144-220
//   max_root_distance_labels   src/program.cpp:239-272
//   postorder_flatten .... src/program.cpp:274-303
//   prefix_function_sequence   src/program.cpp:305-332
#include <algorithm>
#include <cmath>
#include <sstream>

#include "dynbatch.hpp"

namespace dynbatch {

const char* errc_name(Errc code) {
  static const char* const kNames[] = {
      "Ok",           "InvalidArgument",  "UnknownFunction",  "UnderfullSequence",
      "OverfullSequence", "InvalidProgram", "DependencyViolation", "MissingOperand",
      "RowCountMismatch", "WidthMismatch", "ArityMismatch",    "NonFiniteValue",
      "KTooLarge",    "VocabMissingArity", "SingleAssignmentViolation", "ParseError",
      "VerificationFailed"};
  const int i = static_cast<int>(code);
  return (i >= 0 && i < static_cast<int>(sizeof(kNames) / sizeof(kNames[0]))) ? kNames[i]
                                                                             : "UnknownError";
}

void throw_error(Errc code, const std::string& what) { throw Error(code, what); }

// ------------------------------------------------------------------- RNG
std::uint64_t splitmix64(std::uint64_t& state) {
  state += 0x9e3779b97f4a7c15ULL;
  std::uint64_t z = state;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

std::uint64_t mix_seed(std::uint64_t seed, std::uint64_t stream) {
  std::uint64_t s = seed ^ (0x9e3779b97f4a7c15ULL + (stream << 1));
  const std::uint64_t first = splitmix64(s);
  s ^= stream;
  return first ^ splitmix64(s);
}

// mt19937_64: w=64, n=312, m=156, r=31 (standard parameters).
Rng::Rng(std::uint64_t seed) : pos_(312) {
  state_[0] = seed;
  for (int i = 1; i < 312; ++i) {
    const std::uint64_t prev = state_[i - 1];
    state_[i] = 6364136223846793005ULL * (prev ^ (prev >> 62)) + static_cast<std::uint64_t>(i);
  }
}

void Rng::twist() {
  constexpr std::uint64_t hi = ~0ULL << 31, lo = ~hi;
  for (int i = 0; i < 312; ++i) {
    const std::uint64_t bits = (state_[i] & hi) | (state_[(i + 1) % 312] & lo);
    state_[i] = state_[(i + 156) % 312] ^ (bits >> 1) ^ ((bits & 1ULL) ? 0xB5026F5AA96619E9ULL : 0ULL);
  }
  pos_ = 0;
}

void Rng::discard(std::uint64_t n) {
  const std::uint64_t left = static_cast<std::uint64_t>(312 - pos_);
  if (n <= left) {
    pos_ += static_cast<int>(n);
    return;
  }
  n -= left;
  pos_ = 312;
  while (n >= 312) {
    twist();
    n -= 312;
  }
  twist();
  pos_ = static_cast<int>(n);
}

std::uint64_t Rng::next_u64() {
  if (pos_ == 312) twist();
  std::uint64_t y = state_[pos_++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  return y ^ (y >> 43);
}

// ----------------------------------------------------------- TensorBatch
TensorBatch::TensorBatch(std::int64_t rows, std::int64_t width) : rows_(rows), width_(width) {
  if (rows < 0 || width < 0) throw_error(Errc::invalid_argument, "negative tensor shape");
  data_.assign(static_cast<size_t>(rows * width), 0.0);
}

bool TensorBatch::all_finite() const {
  return std::all_of(data_.begin(), data_.end(), [](double v) { return std::isfinite(v); });
}

// ------------------------------------------------------------ vocabulary
FunctionVocab::FunctionVocab(std::vector<ModuleSpec> specs) : specs_(std::move(specs)) {
  if (specs_.empty()) throw_error(Errc::invalid_argument, "vocabulary is empty");
  bool input_provider = false;
  const int w = specs_.front().out_width;
  for (size_t pos = 0; pos < specs_.size(); ++pos) {
    const ModuleSpec& s = specs_[pos];
    if (s.function_id != static_cast<int>(pos)) {
      throw_error(Errc::invalid_argument,
                  "function ids must be exactly 0..p-1, got " + std::to_string(s.function_id) +
                      " at position " + std::to_string(pos));
    }
    if (s.arity < 0) throw_error(Errc::invalid_argument, "negative arity");
    if (s.in_width <= 0 || s.out_width <= 0) throw_error(Errc::invalid_argument, "widths must be positive");
    if (s.out_width != w || s.in_width != s.out_width) {
      throw_error(Errc::invalid_argument, "feature width must be uniform across the vocabulary");
    }
    if (s.arity == 0) {
      if (s.cost != CostClass::free) {
        throw_error(Errc::invalid_argument, "arity-0 function " + std::to_string(s.function_id) +
                                                " must be free (input provider)");
      }
      input_provider = true;
    }
  }
  if (!input_provider) throw_error(Errc::invalid_argument, "vocabulary needs an arity-0 function");
  width_ = w;
}

const ModuleSpec& FunctionVocab::spec(int fid) const {
  if (!contains(fid)) throw_error(Errc::unknown_function, "function id " + std::to_string(fid));
  return specs_[static_cast<size_t>(fid)];
}

// -------------------------------------------------------------- programs
const char* violation_name(ViolationKind kind) {
  switch (kind) {
    case ViolationKind::bad_root: return "BadRoot";
    case ViolationKind::unknown_function: return "UnknownFunction";
    case ViolationKind::bad_child_ref: return "BadChildRef";
    case ViolationKind::arity_mismatch: return "ArityMismatch";
    case ViolationKind::cycle_detected: return "CycleDetected";
    case ViolationKind::unreachable_node: return "UnreachableNode";
    case ViolationKind::free_cost_required: return "FreeCostRequired";
  }
  return "UnknownViolation";
}

std::string ValidationReport::to_string() const {
  if (violations.empty()) return "ok";
  std::string out;
  for (const Violation& v : violations) {
    if (!out.empty()) out += "; ";
    out += violation_name(v.kind);
    out += ": ";
    out += v.detail;
  }
  return out;
}

// Each token becomes node `pos` (prefix order) and fills the next free
// operand slot of the innermost node that still has one.
Program build_program_from_prefix(std::span<const int> functions, const FunctionVocab& vocab) {
  if (functions.empty()) throw_error(Errc::invalid_argument, "empty function sequence");
  Program prog;
  prog.root = 0;
  prog.nodes.resize(functions.size());
  std::vector<std::pair<int, int>> holes;  // (node id, operands still missing)
  size_t pos = 0;
  for (; pos < functions.size(); ++pos) {
    if (pos > 0 && holes.empty()) break;  // root already closed
    const int fid = functions[pos];
    if (!vocab.contains(fid)) throw_error(Errc::unknown_function, "function id " + std::to_string(fid));
    const int id = static_cast<int>(pos);
    prog.nodes[pos].function_id = fid;
    if (!holes.empty()) {
      auto& parent = holes.back();
      prog.nodes[static_cast<size_t>(parent.first)].children.push_back(id);
      if (--parent.second == 0) holes.pop_back();
    }
    const int arity = vocab.spec(fid).arity;
    if (arity > 0) holes.emplace_back(id, arity);
  }
  if (!holes.empty()) {
    throw_error(Errc::underfull_sequence, "sequence of length " + std::to_string(functions.size()) +
                                              " ends with unfilled arities");
  }
  if (pos != functions.size()) {
    throw_error(Errc::overfull_sequence,
                std::to_string(functions.size() - pos) + " tokens remain after the root closes");
  }
  return prog;
}

ValidationReport validate(const Program& program, const FunctionVocab& vocab) {
  ValidationReport rep;
  const int n = program.size();
  if (n == 0 || program.root < 0 || program.root >= n) {
    rep.violations.push_back({ViolationKind::bad_root, "root " + std::to_string(program.root) +
                                                           " with " + std::to_string(n) + " nodes"});
    return rep;
  }
  for (int v = 0; v < n; ++v) {
    const ProgramNode& node = program.nodes[static_cast<size_t>(v)];
    if (!vocab.contains(node.function_id)) {
      rep.violations.push_back({ViolationKind::unknown_function,
                                "node " + std::to_string(v) + " uses function id " +
                                    std::to_string(node.function_id)});
      continue;
    }
    const int arity = vocab.spec(node.function_id).arity;
    if (static_cast<int>(node.children.size()) != arity) {
      rep.violations.push_back({ViolationKind::arity_mismatch,
                                "node " + std::to_string(v) + " has " +
                                    std::to_string(node.children.size()) + " children, function " +
                                    std::to_string(node.function_id) + " has arity " +
                                    std::to_string(arity)});
    }
    for (int c : node.children) {
      if (c < 0 || c >= n) {
        rep.violations.push_back({ViolationKind::bad_child_ref, "node " + std::to_string(v) +
                                                                    " references node " +
                                                                    std::to_string(c)});
      }
    }
  }
  // Three-colour DFS from the root: an edge into an open node is a cycle,
  // anything never reached is unreachable.
  std::vector<unsigned char> state(static_cast<size_t>(n), 0);  // 0 new, 1 open, 2 done
  std::vector<std::pair<int, size_t>> stack{{program.root, 0}};
  state[static_cast<size_t>(program.root)] = 1;
  bool cycle = false;
  while (!stack.empty()) {
    auto& [v, next] = stack.back();
    const auto& ch = program.nodes[static_cast<size_t>(v)].children;
    if (next == ch.size()) {
      state[static_cast<size_t>(v)] = 2;
      stack.pop_back();
      continue;
    }
    const int c = ch[next++];
    if (c < 0 || c >= n) continue;
    if (state[static_cast<size_t>(c)] == 1) {
      if (!cycle) {
        rep.violations.push_back({ViolationKind::cycle_detected, "edge " + std::to_string(v) +
                                                                     "->" + std::to_string(c) +
                                                                     " closes a cycle"});
        cycle = true;
      }
    } else if (state[static_cast<size_t>(c)] == 0) {
      state[static_cast<size_t>(c)] = 1;
      stack.emplace_back(c, 0);
    }
  }
  for (int v = 0; v < n; ++v) {
    if (state[static_cast<size_t>(v)] == 0) {
      rep.violations.push_back({ViolationKind::unreachable_node, "node " + std::to_string(v)});
    }
  }
  return rep;
}

namespace {
void require_well_formed(const Program& program) {
  const int n = program.size();
  if (n == 0 || program.root < 0 || program.root >= n) throw_error(Errc::invalid_program, "bad root");
  for (const ProgramNode& node : program.nodes) {
    for (int c : node.children) {
      if (c < 0 || c >= n) throw_error(Errc::invalid_program, "child reference out of range");
    }
  }
}
}  // namespace

// Longest root-to-node path: relax edges in a topological order obtained by
// peeling zero-in-degree nodes starting from the root.
DepthLabels max_root_distance_labels(const Program& program) {
  require_well_formed(program);
  const size_t n = program.nodes.size();
  std::vector<int> pending(n, 0);
  for (const ProgramNode& node : program.nodes)
    for (int c : node.children) ++pending[static_cast<size_t>(c)];
  DepthLabels out;
  out.labels.assign(n, 0);
  std::vector<int> order{program.root};
  order.reserve(n);
  for (size_t i = 0; i < order.size(); ++i) {
    const int v = order[i];
    const int next_label = out.labels[static_cast<size_t>(v)] + 1;
    for (int c : program.nodes[static_cast<size_t>(v)].children) {
      int& lc = out.labels[static_cast<size_t>(c)];
      lc = std::max(lc, next_label);
      if (--pending[static_cast<size_t>(c)] == 0) order.push_back(c);
    }
  }
  if (order.size() != n) throw_error(Errc::invalid_program, "cycle or unreachable node");
  out.max_label = *std::max_element(out.labels.begin(), out.labels.end());
  return out;
}

std::vector<int> postorder_flatten(const Program& program) {
  require_well_formed(program);
  const size_t n = program.nodes.size();
  std::vector<int> order;
  order.reserve(n);
  std::vector<unsigned char> emitted(n, 0);
  std::vector<std::pair<int, size_t>> stack{{program.root, 0}};
  while (!stack.empty()) {
    auto& [v, next] = stack.back();
    const auto& ch = program.nodes[static_cast<size_t>(v)].children;
    if (next < ch.size()) {
      const int c = ch[next++];
      if (!emitted[static_cast<size_t>(c)]) stack.emplace_back(c, 0);
    } else {
      emitted[static_cast<size_t>(v)] = 1;
      order.push_back(v);
      stack.pop_back();
    }
  }
  if (order.size() != n) throw_error(Errc::invalid_program, "cycle or unreachable node");
  return order;
}

std::vector<int> prefix_function_sequence(const Program& program) {
  require_well_formed(program);
  std::vector<int> seq;
  const size_t limit = program.nodes.size() * 64 + 64;
  std::vector<std::pair<int, size_t>> stack{{program.root, 0}};
  seq.push_back(program.nodes[static_cast<size_t>(program.root)].function_id);
  while (!stack.empty()) {
    auto& [v, next] = stack.back();
    const auto& ch = program.nodes[static_cast<size_t>(v)].children;
    if (next == ch.size()) {
      stack.pop_back();
      continue;
    }
    const int c = ch[next++];
    if (seq.size() > limit) throw_error(Errc::invalid_program, "prefix expansion blow-up");
    seq.push_back(program.nodes[static_cast<size_t>(c)].function_id);
    stack.emplace_back(c, 0);
  }
  return seq;
}

}  // namespace dynbatch
