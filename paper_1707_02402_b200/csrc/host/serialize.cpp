// serialize.cpp — JSON wire formats (host; off the hot path).
//
// Output is byte-compatible with the reference's nlohmann::json dump(2)
// (src/serialize.cpp:26-116): objects with sorted keys, two-space indent,
// one array element per line — the layout pinned by the reference's golden
// test (tests/test_serialize.cpp:69-110). Parsing accepts the documented
// program-set wire format {"vocab": [{"id","arity","cost"}...],
// "programs": [[fid, ...], ...]} (src/serialize.cpp:37-80) with ParseError
// on malformed input.
#include <cerrno>
#include <cmath>
#include <type_traits>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <memory>
#include <string>
#include <variant>

#include "dynbatch.hpp"

namespace dynbatch {

namespace {

// ------------------------------------------------------------- emitter
struct Out {
  std::string s;
  void indent(int level) { s.append(static_cast<size_t>(2 * level), ' '); }
};

// nlohmann's number layout (serializer::dump_float -> to_chars ->
// format_buffer, min_exp -4, max_exp 15): the shortest round-trip digits
// d1..dk with decimal exponent n (value = 0.d1..dk × 10^n) are written
// fixed when -4 < n <= 15 (with a trailing ".0" for integers), else as
// d[.ddd]e±XX with at least two exponent digits.
std::string number(double v) {
  if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
  if (!std::isfinite(v)) return "null";
  char buf[48];
  for (int prec = 1; prec <= 17; ++prec) {
    std::snprintf(buf, sizeof buf, "%.*e", prec - 1, v);
    if (std::strtod(buf, nullptr) == v) break;
  }
  const std::string t(buf);
  const size_t e_at = t.find('e');
  std::string digits;
  for (size_t i = 0; i < e_at; ++i)
    if (t[i] >= '0' && t[i] <= '9') digits += t[i];
  while (digits.size() > 1 && digits.back() == '0') digits.pop_back();
  const int k = static_cast<int>(digits.size());
  const int n = std::atoi(t.c_str() + e_at + 1) + 1;
  std::string s = v < 0 ? "-" : "";
  if (k <= n && n <= 15) {
    s += digits + std::string(static_cast<size_t>(n - k), '0') + ".0";
  } else if (0 < n && n <= 15) {
    s += digits.substr(0, static_cast<size_t>(n)) + "." + digits.substr(static_cast<size_t>(n));
  } else if (-4 < n && n <= 0) {
    s += "0." + std::string(static_cast<size_t>(-n), '0') + digits;
  } else {
    s += digits.substr(0, 1);
    if (k > 1) s += "." + digits.substr(1);
    const int e = n - 1;
    char eb[16];
    std::snprintf(eb, sizeof eb, "e%c%02d", e < 0 ? '-' : '+', e < 0 ? -e : e);
    s += eb;
  }
  return s;
}

// ---------------------------------------------------------------- parser
struct Value;
using Array = std::vector<Value>;
using Object = std::map<std::string, Value>;
struct Value {
  std::variant<std::nullptr_t, bool, double, std::string, std::shared_ptr<Array>, std::shared_ptr<Object>> v;
  std::string num{};  // a number's source text (exact 64-bit integers)
  bool is_obj() const { return v.index() == 5; }
  bool is_arr() const { return v.index() == 4; }
  const Object& obj() const { return *std::get<5>(v); }
  const Array& arr() const { return *std::get<4>(v); }
};

class Parser {
 public:
  explicit Parser(const std::string& t) : t_(t) {}
  Value parse_document() {
    Value v = value();
    ws();
    if (i_ != t_.size()) fail("unexpected trailing characters");
    return v;
  }

 private:
  [[noreturn]] void fail(const std::string& what) {
    throw_error(Errc::parse_error, "[json] " + what + " at byte " + std::to_string(i_));
  }
  void ws() {
    while (i_ < t_.size() && (t_[i_] == ' ' || t_[i_] == '\n' || t_[i_] == '\t' || t_[i_] == '\r')) ++i_;
  }
  bool lit(const char* w) {
    const size_t n = std::char_traits<char>::length(w);
    if (t_.compare(i_, n, w) == 0) { i_ += n; return true; }
    return false;
  }
  Value value() {
    ws();
    if (i_ >= t_.size()) fail("unexpected end of input");
    const char c = t_[i_];
    if (c == '{') return object();
    if (c == '[') return array();
    if (c == '"') return Value{string()};
    if (lit("true")) return Value{true};
    if (lit("false")) return Value{false};
    if (lit("null")) return Value{nullptr};
    if (c == '-' || (c >= '0' && c <= '9')) {
      const char* begin = t_.c_str() + i_;
      char* end = nullptr;
      const double d = std::strtod(begin, &end);
      if (end == begin) fail("bad number");
      i_ += static_cast<size_t>(end - begin);
      Value out{d};
      out.num.assign(begin, static_cast<size_t>(end - begin));
      return out;
    }
    fail(std::string("unexpected character '") + c + "'");
  }
  std::string string() {
    ++i_;  // opening quote
    std::string out;
    while (i_ < t_.size() && t_[i_] != '"') {
      if (t_[i_] == '\\' && i_ + 1 < t_.size()) {
        const char e = t_[++i_];
        out += e == 'n' ? '\n' : e == 't' ? '\t' : e;
        ++i_;
        continue;
      }
      out += t_[i_++];
    }
    if (i_ >= t_.size()) fail("unterminated string");
    ++i_;
    return out;
  }
  Value array() {
    ++i_;
    auto a = std::make_shared<Array>();
    ws();
    if (i_ < t_.size() && t_[i_] == ']') { ++i_; return Value{a}; }
    for (;;) {
      a->push_back(value());
      ws();
      if (i_ < t_.size() && t_[i_] == ',') { ++i_; continue; }
      if (i_ < t_.size() && t_[i_] == ']') { ++i_; return Value{a}; }
      fail("expected ',' or ']'");
    }
  }
  Value object() {
    ++i_;
    auto o = std::make_shared<Object>();
    ws();
    if (i_ < t_.size() && t_[i_] == '}') { ++i_; return Value{o}; }
    for (;;) {
      ws();
      if (i_ >= t_.size() || t_[i_] != '"') fail("expected object key");
      std::string key = string();
      ws();
      if (i_ >= t_.size() || t_[i_] != ':') fail("expected ':'");
      ++i_;
      (*o)[key] = value();
      ws();
      if (i_ < t_.size() && t_[i_] == ',') { ++i_; continue; }
      if (i_ < t_.size() && t_[i_] == '}') { ++i_; return Value{o}; }
      fail("expected ',' or '}'");
    }
  }
  const std::string& t_;
  size_t i_ = 0;
};

int as_int(const Value& v, const char* what) {
  if (v.v.index() != 2) throw_error(Errc::parse_error, std::string("[json] ") + what + " must be a number");
  const double d = std::get<2>(v.v);
  if (d != std::floor(d) || std::fabs(d) > 2147483647.0) {
    throw_error(Errc::parse_error, std::string("[json] ") + what + " must be an integer");
  }
  return static_cast<int>(d);
}

// A 64-bit integer member (exact, from the number's text).
template <typename T>
T as_integer(const Value& v, const char* what) {
  if (v.v.index() != 2 || v.num.find_first_of(".eE") != std::string::npos)
    throw_error(Errc::parse_error, std::string("[json] ") + what + " must be an integer");
  errno = 0;
  char* end = nullptr;
  if constexpr (std::is_signed_v<T>) {
    const long long x = std::strtoll(v.num.c_str(), &end, 10);
    if (errno != 0 || *end) throw_error(Errc::parse_error, std::string("[json] ") + what + " is out of range");
    return static_cast<T>(x);
  } else {
    if (!v.num.empty() && v.num[0] == '-')
      throw_error(Errc::parse_error, std::string("[json] ") + what + " must not be negative");
    const unsigned long long x = std::strtoull(v.num.c_str(), &end, 10);
    if (errno != 0 || *end) throw_error(Errc::parse_error, std::string("[json] ") + what + " is out of range");
    return static_cast<T>(x);
  }
}

double as_double(const Value& v, const char* what) {
  if (v.v.index() != 2) throw_error(Errc::parse_error, std::string("[json] ") + what + " must be a number");
  return std::get<2>(v.v);
}

const Value& member(const Object& o, const char* key) {
  auto it = o.find(key);
  if (it == o.end()) throw_error(Errc::parse_error, std::string("[json] key '") + key + "' not found");
  return it->second;
}

}  // namespace

std::string program_set_to_json(const FunctionVocab& vocab, std::span<const Program> programs) {
  Out o;
  o.s = "{\n  \"programs\": [";
  for (size_t e = 0; e < programs.size(); ++e) {
    const std::vector<int> seq = prefix_function_sequence(programs[e]);
    o.s += e ? ",\n    [" : "\n    [";
    for (size_t i = 0; i < seq.size(); ++i) {
      o.s += i ? ",\n      " : "\n      ";
      o.s += std::to_string(seq[i]);
    }
    o.s += "\n    ]";
  }
  o.s += programs.empty() ? "]" : "\n  ]";
  o.s += ",\n  \"vocab\": [";
  for (int f = 0; f < vocab.size(); ++f) {
    const ModuleSpec& s = vocab.spec(f);
    o.s += f ? ",\n    {\n" : "\n    {\n";
    o.s += "      \"arity\": " + std::to_string(s.arity) + ",\n";
    o.s += std::string("      \"cost\": \"") + (s.is_expensive() ? "expensive" : "free") + "\",\n";
    o.s += "      \"id\": " + std::to_string(s.function_id) + "\n    }";
  }
  o.s += vocab.size() ? "\n  ]\n}" : "]\n}";
  return o.s;
}

ProgramSet program_set_from_json(const std::string& text, int width) {
  const Value doc = Parser(text).parse_document();
  if (!doc.is_obj() || !doc.obj().count("vocab") || !doc.obj().count("programs")) {
    throw_error(Errc::parse_error, "expected {\"vocab\": [...], \"programs\": [...]}");
  }
  const Value& vv = doc.obj().at("vocab");
  const Value& pv = doc.obj().at("programs");
  if (!vv.is_arr() || !pv.is_arr()) throw_error(Errc::parse_error, "[json] vocab and programs must be arrays");
  std::vector<ModuleSpec> specs;
  for (const Value& entry : vv.arr()) {
    if (!entry.is_obj()) throw_error(Errc::parse_error, "[json] vocab entries must be objects");
    ModuleSpec s;
    s.function_id = as_int(member(entry.obj(), "id"), "id");
    s.arity = as_int(member(entry.obj(), "arity"), "arity");
    s.in_width = s.out_width = width;
    const Value& cost = member(entry.obj(), "cost");
    if (cost.v.index() != 3) throw_error(Errc::parse_error, "[json] cost must be a string");
    const std::string& c = std::get<3>(cost.v);
    if (c == "expensive") s.cost = CostClass::expensive;
    else if (c == "free") s.cost = CostClass::free;
    else throw_error(Errc::parse_error, "cost must be 'expensive' or 'free', got '" + c + "'");
    specs.push_back(s);
  }
  ProgramSet set{FunctionVocab(std::move(specs)), {}};
  for (const Value& seq : pv.arr()) {
    if (!seq.is_arr()) throw_error(Errc::parse_error, "[json] programs must be arrays of function ids");
    std::vector<int> fns;
    for (const Value& x : seq.arr()) fns.push_back(as_int(x, "function id"));
    set.programs.push_back(build_program_from_prefix(fns, set.vocab));
  }
  return set;
}

std::string schedule_to_json(const Schedule& schedule) {
  std::string s = "{\n  \"steps\": [";
  for (size_t st = 0; st < schedule.steps.size(); ++st) {
    const Step& step = schedule.steps[st];
    s += st ? ",\n    [" : "\n    [";
    for (size_t g = 0; g < step.size(); ++g) {
      s += g ? ",\n      {\n" : "\n      {\n";
      s += "        \"function_id\": " + std::to_string(step[g].function_id) + ",\n";
      s += "        \"members\": [";
      const auto& m = step[g].members;
      for (size_t i = 0; i < m.size(); ++i) {
        s += i ? ",\n          [\n" : "\n          [\n";
        s += "            " + std::to_string(m[i].example) + ",\n";
        s += "            " + std::to_string(m[i].node) + "\n          ]";
      }
      s += m.empty() ? "]" : "\n        ]";
      s += "\n      }";
    }
    s += step.empty() ? "]" : "\n    ]";
  }
  s += schedule.steps.empty() ? "]" : "\n  ]";
  s += ",\n  \"strategy\": \"";
  s += strategy_name(schedule.strategy);
  s += "\"\n}";
  return s;
}

std::string trace_to_json(const ExecutionTrace& trace) {
  std::string s = "{\n  \"expensive_calls\": " + std::to_string(trace.expensive_calls);
  s += ",\n  \"module_seconds\": " + number(trace.module_seconds);
  s += ",\n  \"peak_group_rows\": " + std::to_string(trace.peak_group_rows);
  std::map<std::string, std::int64_t> calls;  // string keys sort like nlohmann's
  for (size_t f = 0; f < trace.per_function_calls.size(); ++f)
    if (trace.per_function_calls[f] > 0) calls[std::to_string(f)] = trace.per_function_calls[f];
  s += ",\n  \"per_function_calls\": {";
  bool first = true;
  for (const auto& [k, v] : calls) {
    s += first ? "\n    \"" : ",\n    \"";
    s += k + "\": " + std::to_string(v);
    first = false;
  }
  s += calls.empty() ? "}" : "\n  }";
  s += ",\n  \"per_step_seconds\": [";
  for (size_t i = 0; i < trace.per_step_seconds.size(); ++i) {
    s += i ? ",\n    " : "\n    ";
    s += number(trace.per_step_seconds[i]);
  }
  s += trace.per_step_seconds.empty() ? "]" : "\n  ]";
  s += ",\n  \"stacking_seconds\": " + number(trace.stacking_seconds);
  s += ",\n  \"total_seconds\": " + number(trace.total_seconds);
  s += "\n}";
  return s;
}

// WorkloadSpec and MoeConfig as JSON objects (src/serialize.cpp:118-175):
// keys in sorted order, two-space indent. Parsing takes the same keys,
// optional ones defaulting to the struct defaults; errors are ParseError.
std::string workload_spec_to_json(const WorkloadSpec& spec) {
  std::string s = "{\n";
  s += "  \"b\": " + std::to_string(spec.b) + ",\n";
  s += "  \"branch_prob\": " + number(spec.branch_prob) + ",\n";
  s += "  \"depth\": " + std::to_string(spec.depth) + ",\n";
  s += std::string("  \"kind\": \"") + workload_kind_name(spec.kind) + "\",\n";
  s += "  \"length\": " + std::to_string(spec.length) + ",\n";
  s += "  \"p\": " + std::to_string(spec.p) + ",\n";
  s += "  \"seed\": " + std::to_string(spec.seed) + ",\n";
  s += "  \"width\": " + std::to_string(spec.width) + "\n}";
  return s;
}

WorkloadSpec workload_spec_from_json(const std::string& text) {
  const Value doc = Parser(text).parse_document();
  if (!doc.is_obj()) throw_error(Errc::parse_error, "[json] a workload spec is an object");
  const Object& o = doc.obj();
  WorkloadSpec spec;
  const Value& kind = member(o, "kind");
  if (kind.v.index() != 3) throw_error(Errc::parse_error, "[json] kind must be a string");
  spec.kind = workload_kind_from_name(std::get<3>(kind.v));
  if (o.count("b")) spec.b = as_integer<std::int64_t>(o.at("b"), "b");
  if (o.count("p")) spec.p = as_integer<int>(o.at("p"), "p");
  if (o.count("width")) spec.width = as_integer<int>(o.at("width"), "width");
  if (o.count("depth")) spec.depth = as_integer<int>(o.at("depth"), "depth");
  if (o.count("length")) spec.length = as_integer<int>(o.at("length"), "length");
  if (o.count("branch_prob")) spec.branch_prob = as_double(o.at("branch_prob"), "branch_prob");
  if (o.count("seed")) spec.seed = as_integer<std::uint64_t>(o.at("seed"), "seed");
  return spec;
}

std::string moe_config_to_json(const MoeConfig& cfg) {
  std::string s = "{\n";
  s += "  \"b\": " + std::to_string(cfg.batch) + ",\n";
  s += "  \"data_dim\": " + std::to_string(cfg.data_dim) + ",\n";
  s += "  \"hidden\": " + std::to_string(cfg.hidden) + ",\n";
  s += "  \"k\": " + std::to_string(cfg.active_per_example) + ",\n";
  s += "  \"m\": " + number(cfg.examples_per_expert) + ",\n";
  s += "  \"n\": " + std::to_string(cfg.experts) + "\n}";
  return s;
}

MoeConfig moe_config_from_json(const std::string& text) {
  const Value doc = Parser(text).parse_document();
  if (!doc.is_obj()) throw_error(Errc::parse_error, "[json] a MoE config is an object");
  const Object& o = doc.obj();
  MoeConfig cfg;
  cfg.experts = as_integer<std::int64_t>(member(o, "n"), "n");
  cfg.active_per_example = as_integer<std::int64_t>(member(o, "k"), "k");
  if (o.count("b")) cfg.batch = as_integer<std::int64_t>(o.at("b"), "b");
  if (o.count("data_dim")) cfg.data_dim = as_integer<std::int64_t>(o.at("data_dim"), "data_dim");
  if (o.count("hidden")) cfg.hidden = as_integer<std::int64_t>(o.at("hidden"), "hidden");
  if (o.count("m")) cfg.examples_per_expert = as_double(o.at("m"), "m");
  cfg.check();  // validated on parse (k ≤ n, positive sizes)
  return cfg;
}

}  // namespace dynbatch
