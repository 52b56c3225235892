// embcomm_gpu.hpp -- the reference's C++ API (namespace embcomm,
// /root/reference/proj/core/include/embcomm/*.hpp) as a header-only layer over
// the C-ABI of libembcomm_gpu.so (embcomm_gpu.h).
//
// A reference caller switches by putting include/ (whose embcomm/*.hpp
// forward here) ahead of the reference headers and linking
// libembcomm_gpu.so: same names, value types, argument meaning and
// exceptions.  The reference's own unit tests (proj/tests/test_*.cpp) build
// unchanged against it (tests/cpp/Makefile, tests/test_ref_unit_tests.py).
// The simulator, sampler, skew table and hot/normal partition run on the GPU;
// cost model and planner stay on the host in the reference's summation order.
// Text trace and distribution-spec JSON I/O, scaling_study and
// portion_usage are host conveniences here (SURVEY.md §2 marks them out of
// the hot path); they exist so reference callers relink unchanged.
#pragma once

#include <bit>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <istream>
#include <optional>
#include <ostream>
#include <span>
#include <sstream>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "embcomm_gpu.h"

namespace embcomm {

// ------------------------------------------------------------------ errors
// error.hpp:10-19; DeviceError is this layer's own (CUDA / NCCL failures).
class ValidationError : public std::runtime_error {
 public:
  explicit ValidationError(const std::string& w) : std::runtime_error(w) {}
};
class InvariantError : public std::logic_error {
 public:
  explicit InvariantError(const std::string& w) : std::logic_error(w) {}
};
class DeviceError : public std::runtime_error {
 public:
  explicit DeviceError(const std::string& w) : std::runtime_error(w) {}
};

namespace detail {
inline void check(int rc) {
  if (rc == EC_OK) return;
  const std::string m = ec_last_error();
  if (rc == EC_EINVAL) throw ValidationError(m);
  if (rc == EC_EINVARIANT) throw InvariantError(m);
  throw DeviceError(m);
}
}  // namespace detail

// -------------------------------------------------------------------- rng
// rng.hpp:12-43.  Draws for sampling happen on the GPU (closed form of the
// stream position); this class carries the state they advance.
inline constexpr const char* kRngAlgorithm = "splitmix64";

inline std::uint64_t substream_seed(std::uint64_t master, std::uint64_t index) {
  return ec_substream_seed(master, index);
}

class SplitMix64 {
 public:
  explicit SplitMix64(std::uint64_t seed) : state_(seed) {}
  std::uint64_t next() {
    state_ += 0x9E3779B97F4A7C15ull;
    std::uint64_t z = state_;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  double next_double() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  std::uint64_t& state() { return state_; }

 private:
  std::uint64_t state_;
};

// ---------------------------------------------------------- distribution
// distribution.hpp:11-49.  A handle to the library's distribution; copies
// are independent (ec_dist_clone), as the reference's value type.
inline constexpr double kProbabilitySumTolerance = 1e-9;

class DiscreteSampler;

class EmbeddingDistribution {
 public:
  static EmbeddingDistribution from_probabilities(std::vector<double> probs) {
    ec_dist h = nullptr;
    detail::check(ec_dist_from_probabilities(probs.data(), probs.size(), &h));
    return EmbeddingDistribution(h);
  }
  static EmbeddingDistribution uniform(std::size_t size) {
    ec_dist h = nullptr;
    detail::check(ec_dist_uniform(size, &h));
    return EmbeddingDistribution(h);
  }
  static EmbeddingDistribution adopt(ec_dist h) { return EmbeddingDistribution(h); }

  EmbeddingDistribution(const EmbeddingDistribution& o) { detail::check(ec_dist_clone(o.h_, &h_)); }
  EmbeddingDistribution(EmbeddingDistribution&& o) noexcept
      : h_(std::exchange(o.h_, nullptr)), s_(std::exchange(o.s_, nullptr)) {}
  EmbeddingDistribution& operator=(EmbeddingDistribution o) noexcept {
    std::swap(h_, o.h_);
    std::swap(s_, o.s_);
    return *this;
  }
  ~EmbeddingDistribution() {
    if (s_) ec_sampler_destroy(s_);
    if (h_) ec_dist_destroy(h_);
  }

  std::size_t size() const noexcept { return ec_dist_size(h_); }
  double prob(std::uint32_t id) const { return get<double>(ec_dist_prob, id); }
  double prob_at_rank(std::size_t rank) const { return get<double>(ec_dist_prob_at_rank, rank); }
  std::uint32_t id_at_rank(std::size_t rank) const { return get<std::uint32_t>(ec_dist_id_at_rank, rank); }
  std::size_t rank_of(std::uint32_t id) const { return get<std::uint64_t>(ec_dist_rank_of, id); }
  std::span<const double> ranked_probs() const noexcept {
    const double* p = nullptr;
    if (ec_dist_ranked_view(h_, &p) != EC_OK) return {};
    return {p, size()};
  }
  std::vector<std::uint32_t> top_ids(std::size_t k) const {
    if (k > size())
      throw ValidationError("cannot take top " + std::to_string(k) + " of " + std::to_string(size()) +
                            " embeddings");
    std::vector<std::uint32_t> v(k);
    detail::check(ec_dist_top_ids(h_, k, v.data()));
    return v;
  }
  double mass_of(std::span<const std::uint32_t> ids) const {
    double v = 0.0;
    detail::check(ec_dist_mass_of(h_, ids.data(), ids.size(), &v));
    return v;
  }

  ec_dist handle() const { return h_; }
  // the GPU sampler of this distribution (built on first use, device 0)
  ec_sampler sampler() const {
    if (!s_) detail::check(ec_sampler_create(h_, 0, &s_));
    return s_;
  }

 private:
  explicit EmbeddingDistribution(ec_dist h) : h_(h) {}
  template <class T, class F, class A>
  T get(F fn, A arg) const {
    T v{};
    detail::check(fn(h_, arg, &v));
    return v;
  }
  ec_dist h_ = nullptr;
  mutable ec_sampler s_ = nullptr;
};

// ------------------------------------------------------ distribution spec
// distribution_spec.hpp:14-67.
enum class DistributionKind { zipf = EC_ZIPF, exponential = EC_EXPONENTIAL, half_normal = EC_HALF_NORMAL,
                              empirical = EC_EMPIRICAL };

inline constexpr double kDefaultZipfExponent = 2.5;
inline constexpr double kDefaultExponentialRate = 100.0;
inline constexpr double kDefaultHalfNormalSigma = 0.05;

inline std::string to_string(DistributionKind kind) {
  switch (kind) {
    case DistributionKind::zipf: return "zipf";
    case DistributionKind::exponential: return "exponential";
    case DistributionKind::half_normal: return "half_normal";
    case DistributionKind::empirical: return "empirical";
  }
  return "?";
}

inline std::optional<DistributionKind> kind_from_string(std::string_view name) {
  for (auto k : {DistributionKind::zipf, DistributionKind::exponential, DistributionKind::half_normal,
                 DistributionKind::empirical})
    if (name == to_string(k)) return k;
  return std::nullopt;
}

inline double default_shape(DistributionKind kind) {
  double v = 0.0;
  detail::check(ec_default_shape(static_cast<int>(kind), &v));
  return v;
}

namespace detail {
// Just enough JSON for a distribution spec document: an object of string,
// number, array-of-number and (ignored, nested) object values.
class SpecJson {
 public:
  explicit SpecJson(const std::string& text) : s_(text) {}

  struct Value {
    enum Kind { kString, kNumber, kArray, kObject, kOther } kind = kOther;
    std::string str;
    double num = 0.0;
    bool integral = false, negative = false;
    std::uint64_t uint = 0;
    std::vector<double> arr;
  };

  std::vector<std::pair<std::string, Value>> object() {
    std::vector<std::pair<std::string, Value>> out;
    ws();
    expect('{');
    ws();
    if (peek() == '}') {
      ++i_;
      return finish(out);
    }
    for (;;) {
      ws();
      std::string key = string_lit();
      ws();
      expect(':');
      out.emplace_back(std::move(key), value());
      ws();
      if (peek() == ',') {
        ++i_;
        continue;
      }
      expect('}');
      return finish(out);
    }
  }

 private:
  [[noreturn]] void fail(const std::string& what) const {
    throw ValidationError("invalid distribution JSON: " + what + " at offset " + std::to_string(i_));
  }
  char peek() const { return i_ < s_.size() ? s_[i_] : '\0'; }
  void ws() {
    while (i_ < s_.size() && (s_[i_] == ' ' || s_[i_] == '\n' || s_[i_] == '\t' || s_[i_] == '\r')) ++i_;
  }
  void expect(char c) {
    if (peek() != c) fail(std::string("expected '") + c + "'");
    ++i_;
  }
  std::vector<std::pair<std::string, Value>> finish(std::vector<std::pair<std::string, Value>>& out) {
    ws();
    if (depth_ == 0 && i_ != s_.size()) fail("trailing characters");
    return std::move(out);
  }
  std::string string_lit() {
    expect('"');
    std::string r;
    while (peek() != '"') {
      if (i_ >= s_.size()) fail("unterminated string");
      if (s_[i_] == '\\') {
        ++i_;
        if (i_ >= s_.size()) fail("unterminated string");
      }
      r.push_back(s_[i_++]);
    }
    ++i_;
    return r;
  }
  Value number() {
    Value v;
    v.kind = Value::kNumber;
    const std::size_t b = i_;
    if (peek() == '-') {
      v.negative = true;
      ++i_;
    }
    bool frac = false;
    while (i_ < s_.size() && (std::isdigit(static_cast<unsigned char>(s_[i_])) || s_[i_] == '.' || s_[i_] == 'e' ||
                              s_[i_] == 'E' || s_[i_] == '+' || s_[i_] == '-')) {
      if (!std::isdigit(static_cast<unsigned char>(s_[i_]))) frac = true;
      ++i_;
    }
    const std::string tok = s_.substr(b, i_ - b);
    if (tok.empty() || tok == "-") fail("bad number");
    std::size_t used = 0;
    try {
      v.num = std::stod(tok, &used);
    } catch (const std::exception&) {
      fail("bad number");
    }
    if (used != tok.size()) fail("bad number");
    v.integral = !frac;
    if (v.integral && !v.negative) v.uint = std::stoull(tok);
    return v;
  }
  Value value() {
    ws();
    Value v;
    const char c = peek();
    if (c == '"') {
      v.kind = Value::kString;
      v.str = string_lit();
    } else if (c == '[') {
      v.kind = Value::kArray;
      ++i_;
      ws();
      if (peek() == ']') {
        ++i_;
        return v;
      }
      for (;;) {
        ws();
        const Value e = number();
        v.arr.push_back(e.num);
        ws();
        if (peek() == ',') {
          ++i_;
          continue;
        }
        expect(']');
        break;
      }
    } else if (c == '{') {
      v.kind = Value::kObject;
      ++depth_;
      object();  // nested objects ("manifest") are parsed and ignored
      --depth_;
    } else if (c == '-' || std::isdigit(static_cast<unsigned char>(c))) {
      v = number();
    } else {
      fail("unexpected character");
    }
    return v;
  }

  const std::string& s_;
  std::size_t i_ = 0;
  int depth_ = 0;
};
}  // namespace detail

struct DistributionSpec {
  DistributionKind kind = DistributionKind::zipf;
  std::size_t size = 0;
  double shape = 0.0;
  std::vector<double> probs;

  static DistributionSpec parametric(DistributionKind kind, std::size_t size, double shape) {
    if (kind == DistributionKind::empirical)
      throw ValidationError("use DistributionSpec::empirical for explicit probabilities");
    if (size == 0) throw ValidationError("distribution size must be >= 1");
    if (!(shape > 0.0) || !std::isfinite(shape)) throw ValidationError("shape parameter must be positive and finite");
    DistributionSpec s;
    s.kind = kind;
    s.size = size;
    s.shape = shape;
    return s;
  }
  static DistributionSpec empirical(std::vector<double> probs) {
    if (probs.empty()) throw ValidationError("distribution size must be >= 1");
    DistributionSpec s;
    s.kind = DistributionKind::empirical;
    s.size = probs.size();
    s.probs = std::move(probs);
    return s;
  }

  std::string to_json() const {
    auto num = [](double x) {
      char b[32];
      std::snprintf(b, sizeof b, "%.17g", x);
      return std::string(b);
    };
    std::string j = "{\n  \"kind\": \"" + to_string(kind) + "\"";
    if (kind == DistributionKind::empirical) {
      j += ",\n  \"probs\": [";
      for (std::size_t i = 0; i < probs.size(); ++i) j += (i ? ", " : "") + num(probs[i]);
      j += "]";
    } else {
      j += ",\n  \"size\": " + std::to_string(size) + ",\n  \"shape\": " + num(shape);
    }
    return j + "\n}\n";
  }

  static DistributionSpec from_json(const std::string& text) {
    using V = detail::SpecJson::Value;
    const auto fields = detail::SpecJson(text).object();
    const V* kind = nullptr;
    const V* size = nullptr;
    const V* shape = nullptr;
    const V* probs = nullptr;
    for (const auto& [k, v] : fields) {
      if (k == "kind") kind = &v;
      else if (k == "size") size = &v;
      else if (k == "shape") shape = &v;
      else if (k == "probs") probs = &v;
      else if (k != "manifest") throw ValidationError("unknown field \"" + k + "\" in distribution JSON");
    }
    if (!kind || kind->kind != V::kString) throw ValidationError("distribution JSON needs a string \"kind\"");
    const auto kd = kind_from_string(kind->str);
    if (!kd) throw ValidationError("unknown distribution kind \"" + kind->str + "\"");
    if (*kd == DistributionKind::empirical) {
      if (!probs || probs->kind != V::kArray)
        throw ValidationError("empirical distribution JSON needs a \"probs\" array");
      if (size && (size->kind != V::kNumber || size->uint != probs->arr.size()))
        throw ValidationError("\"size\" disagrees with the length of \"probs\"");
      return empirical(probs->arr);
    }
    if (!size || size->kind != V::kNumber || !size->integral || size->negative)
      throw ValidationError("distribution JSON needs a non-negative integer \"size\"");
    if (!shape || shape->kind != V::kNumber) throw ValidationError("distribution JSON needs a numeric \"shape\"");
    if (size->uint == 0) throw ValidationError("distribution size must be >= 1");
    return parametric(*kd, static_cast<std::size_t>(size->uint), shape->num);
  }

  static DistributionSpec load(const std::filesystem::path& path) {
    std::ifstream in(path);
    if (!in) throw ValidationError("cannot open distribution file " + path.string());
    std::ostringstream b;
    b << in.rdbuf();
    return from_json(b.str());
  }
  void save(const std::filesystem::path& path) const {
    std::ofstream out(path);
    if (!out) throw ValidationError("cannot write distribution file " + path.string());
    out << to_json();
  }
};

inline EmbeddingDistribution materialize(const DistributionSpec& spec) {
  if (spec.kind == DistributionKind::empirical) return EmbeddingDistribution::from_probabilities(spec.probs);
  ec_dist h = nullptr;
  detail::check(ec_dist_materialize(static_cast<int>(spec.kind), spec.size, spec.shape, &h));
  return EmbeddingDistribution::adopt(h);
}

inline DistributionSpec scale(const DistributionSpec& spec, std::int64_t factor) {
  if (spec.kind == DistributionKind::empirical) throw ValidationError("scale requires a parametric distribution");
  if (factor < 1) throw ValidationError("scale factor must be >= 1");
  std::size_t grown = 0;
  if (__builtin_mul_overflow(spec.size, static_cast<std::size_t>(factor), &grown))
    throw ValidationError("scaled size overflows");
  return DistributionSpec::parametric(spec.kind, grown, spec.shape);
}

inline EmbeddingDistribution materialize_extended(const DistributionSpec& spec, std::int64_t factor) {
  if (spec.kind == DistributionKind::empirical)
    throw ValidationError("materialize_extended requires a parametric distribution");
  ec_dist h = nullptr;
  detail::check(ec_dist_materialize_extended(static_cast<int>(spec.kind), spec.size, spec.shape, factor, &h));
  return EmbeddingDistribution::adopt(h);
}

// ------------------------------------------------------------ cost model
// cost_model.hpp:11-64 (host, the reference's summation order).
inline constexpr const char* kCostUnitsNote = "one unit = one embedding vector = one transmitted index";

struct WorkloadSpec {
  std::int64_t num_samples;
  std::int64_t batch_size;
  std::int64_t lookups_per_sample;
  WorkloadSpec(std::int64_t q, std::int64_t b, std::int64_t d) : num_samples(q), batch_size(b), lookups_per_sample(d) {
    const ec_workload w{q, b, d};
    detail::check(ec_workload_validate(&w));
  }
  ec_workload c() const { return {num_samples, batch_size, lookups_per_sample}; }
};

struct CostBreakdown {
  double index_cost = 0.0;
  double embedding_cost = 0.0;
  double total = 0.0;
  std::string units_note = kCostUnitsNote;
};

namespace detail {
inline CostBreakdown cost(const ec_cost& c) { return {c.index_cost, c.embedding_cost, c.total, kCostUnitsNote}; }
template <class F, class... A>
double scalar(F fn, A... a) {
  double v = 0.0;
  check(fn(a..., &v));
  return v;
}
}  // namespace detail

inline double batch_presence_prob(double p, std::int64_t b) { return detail::scalar(ec_batch_presence_prob, p, b); }
inline double expected_unique_per_batch(const EmbeddingDistribution& d, std::int64_t b) {
  return detail::scalar(ec_expected_unique_per_batch, d.handle(), b);
}
inline double expected_unique_from_rank(const EmbeddingDistribution& d, std::int64_t b, std::size_t first_rank) {
  return detail::scalar(ec_expected_unique_from_rank, d.handle(), b, static_cast<std::uint64_t>(first_rank));
}
inline CostBreakdown coalesced_batch_cost(const EmbeddingDistribution& d, std::int64_t b) {
  ec_cost c{};
  detail::check(ec_coalesced_batch_cost(d.handle(), b, &c));
  return detail::cost(c);
}
inline double baseline_epoch_cost(const WorkloadSpec& s) {
  const ec_workload w = s.c();
  return detail::scalar(ec_baseline_epoch_cost, &w);
}
inline CostBreakdown coalesced_epoch_cost(const EmbeddingDistribution& d, const WorkloadSpec& s) {
  const ec_workload w = s.c();
  ec_cost c{};
  detail::check(ec_coalesced_epoch_cost(d.handle(), &w, &c));
  return detail::cost(c);
}
inline CostBreakdown cached_epoch_cost(const EmbeddingDistribution& d, const WorkloadSpec& s,
                                       std::span<const std::uint32_t> cache_ids) {
  const ec_workload w = s.c();
  ec_cost c{};
  detail::check(ec_cached_epoch_cost(d.handle(), &w, cache_ids.data(), cache_ids.size(), &c));
  return detail::cost(c);
}

// --------------------------------------------------------- cache planner
// cache_planner.hpp:16-81 (host).
struct DeviceModel {
  std::int64_t total_params;
  std::int64_t activation_params_per_sample;
  std::int64_t embedding_params;
  double memory_efficiency = 1.0;
  DeviceModel(std::int64_t m, std::int64_t a, std::int64_t e, double eff = 1.0)
      : total_params(m), activation_params_per_sample(a), embedding_params(e), memory_efficiency(eff) {
    const ec_device_model x = c();
    detail::check(ec_device_model_validate(&x));
  }
  ec_device_model c() const { return {total_params, activation_params_per_sample, embedding_params, memory_efficiency}; }
};

inline std::optional<std::int64_t> max_batch_size(const DeviceModel& device, std::int64_t cache_size) {
  const ec_device_model x = device.c();
  std::int64_t v = 0;
  detail::check(ec_max_batch_size(&x, cache_size, &v));
  if (v < 0) return std::nullopt;
  return v;
}

struct MarginalReport {
  std::uint32_t candidate_id = 0;
  double presence_gain = 0.0;
  double threshold = 0.0;
  double delta_comm = 0.0;
  bool recommend = false;
};

inline MarginalReport delta_comm(const EmbeddingDistribution& dist, const DeviceModel& device,
                                 std::int64_t num_samples, std::int64_t current_cache_size) {
  const ec_device_model x = device.c();
  ec_marginal r{};
  detail::check(ec_delta_comm(dist.handle(), &x, num_samples, current_cache_size, &r));
  return {r.candidate_id, r.presence_gain, r.threshold, r.delta_comm, r.recommend != 0};
}

struct CachePlan {
  std::size_t cache_size = 0;
  std::vector<std::uint32_t> cached_ids;
  std::int64_t batch_size = 0;
  CostBreakdown expected_epoch_cost;
  bool feasible = false;
  bool used_scan_fallback = false;
};

namespace detail {
template <class F>
CachePlan plan(F fn, const EmbeddingDistribution& d, const DeviceModel& m, const WorkloadSpec& s) {
  const ec_device_model x = m.c();
  const ec_workload w = s.c();
  ec_cache_plan p{};
  std::vector<std::uint32_t> ids(d.size());
  check(fn(d.handle(), &x, &w, &p, ids.data()));
  CachePlan out;
  out.feasible = p.feasible != 0;
  out.used_scan_fallback = p.used_scan_fallback != 0;
  if (out.feasible) {
    out.cache_size = p.cache_size;
    ids.resize(p.cache_size);
    out.cached_ids = std::move(ids);
    out.batch_size = p.batch_size;
    out.expected_epoch_cost = cost(p.expected_epoch_cost);
  }
  return out;
}
}  // namespace detail

inline CachePlan optimal_cache_size_scan(const EmbeddingDistribution& d, const DeviceModel& m, const WorkloadSpec& s) {
  return detail::plan(ec_optimal_cache_size_scan, d, m, s);
}
inline CachePlan optimal_cache_size_search(const EmbeddingDistribution& d, const DeviceModel& m,
                                           const WorkloadSpec& s) {
  return detail::plan(ec_optimal_cache_size_search, d, m, s);
}
inline double memory_io_proxy(const EmbeddingDistribution& d, const WorkloadSpec& s,
                              std::span<const std::uint32_t> cache_ids) {
  const ec_workload w = s.c();
  return detail::scalar(ec_memory_io_proxy, d.handle(), &w, cache_ids.data(), static_cast<std::uint64_t>(cache_ids.size()));
}

// ----------------------------------------------------------------- traces
// trace.hpp:14-88.
struct Trace {
  std::int64_t num_features = 0;
  std::size_t vocab_size = 0;
  std::vector<std::uint32_t> ids;

  std::size_t num_samples() const {
    return num_features > 0 ? ids.size() / static_cast<std::size_t>(num_features) : 0;
  }
  std::span<const std::uint32_t> sample(std::size_t i) const {
    const auto d = static_cast<std::size_t>(num_features);
    return {ids.data() + i * d, d};
  }
};

namespace detail {
[[noreturn]] inline void at_line(std::size_t line, const std::string& what) {
  throw ValidationError("line " + std::to_string(line) + ": " + what);
}
// one decimal field of a trace line; advances p past it
inline std::uint64_t trace_field(const std::string& ln, std::size_t& p, std::size_t line) {
  std::uint64_t v = 0;
  const std::size_t b = p;
  while (p < ln.size() && ln[p] >= '0' && ln[p] <= '9') {
    const std::uint64_t d = static_cast<std::uint64_t>(ln[p] - '0');
    if (v > (UINT64_MAX - d) / 10) at_line(line, "malformed id near \"" + ln.substr(b, 12) + "\"");
    v = v * 10 + d;
    ++p;
  }
  if (p == b || (p < ln.size() && ln[p] != ' ')) at_line(line, "malformed id near \"" + ln.substr(b, 12) + "\"");
  return v;
}
}  // namespace detail

inline Trace parse_trace(std::istream& in) {
  std::string ln;
  if (!std::getline(in, ln)) throw ValidationError("empty trace");
  if (!ln.empty() && ln.back() == '\r') ln.pop_back();
  const std::string bad_header = "malformed header, expected \"d=<int> E=<int>\"";
  long long d = 0;
  unsigned long long e = 0;
  int used = 0;
  if (std::sscanf(ln.c_str(), "d=%lld E=%llu%n", &d, &e, &used) != 2 || used != static_cast<int>(ln.size()) ||
      ln.rfind("d=", 0) != 0 || ln.find(" E=") == std::string::npos)
    detail::at_line(1, bad_header);
  if (d < 1) detail::at_line(1, "lookups per sample must be >= 1");
  if (e < 1) detail::at_line(1, "vocabulary size must be >= 1");
  if (e > 0xFFFFFFFFull) detail::at_line(1, "vocabulary too large for 32-bit ids");
  Trace t;
  t.num_features = d;
  t.vocab_size = static_cast<std::size_t>(e);
  std::size_t line = 1;
  while (std::getline(in, ln)) {
    ++line;
    if (!ln.empty() && ln.back() == '\r') ln.pop_back();
    std::size_t p = 0, fields = 0;
    for (;;) {
      while (p < ln.size() && ln[p] == ' ') ++p;
      if (p >= ln.size()) break;
      const std::uint64_t id = detail::trace_field(ln, p, line);
      if (id >= t.vocab_size)
        detail::at_line(line, "id " + std::to_string(id) + " out of range [0, " + std::to_string(t.vocab_size) + ")");
      t.ids.push_back(static_cast<std::uint32_t>(id));
      ++fields;
    }
    if (fields != static_cast<std::size_t>(d))
      detail::at_line(line, "expected " + std::to_string(d) + " ids, found " + std::to_string(fields));
  }
  if (t.ids.empty()) throw ValidationError("empty trace");
  return t;
}

inline Trace load_trace(const std::filesystem::path& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw ValidationError("cannot open trace file " + path.string());
  return parse_trace(in);
}

inline void write_trace(std::ostream& out, const Trace& t) {
  out << "d=" << t.num_features << " E=" << t.vocab_size << "\n";
  for (std::size_t s = 0; s < t.num_samples(); ++s) {
    const auto row = t.sample(s);
    for (std::size_t j = 0; j < row.size(); ++j) out << (j ? " " : "") << row[j];
    out << "\n";
  }
}

inline void save_trace(const std::filesystem::path& path, const Trace& t) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw ValidationError("cannot write trace file " + path.string());
  write_trace(out, t);
}

struct SkewEntry {
  std::uint32_t id = 0;
  std::uint64_t count = 0;
  double cum_fraction = 0.0;
};
struct SkewTable {
  std::vector<SkewEntry> entries;
  std::uint64_t total_accesses = 0;
};

// access counts histogrammed on the GPU (device 0), ranked on the host
inline SkewTable build_skew_table(const Trace& t) {
  if (t.ids.empty()) throw ValidationError("empty trace");
  const std::size_t cap = std::min<std::size_t>(t.ids.size(), t.vocab_size);
  std::vector<std::uint32_t> ids(cap);
  std::vector<std::uint64_t> counts(cap);
  std::vector<double> cum(cap);
  std::uint64_t n = 0;
  detail::check(ec_build_skew_table(t.ids.data(), t.ids.size(), t.vocab_size, 0, ids.data(), counts.data(),
                                    cum.data(), &n));
  SkewTable s;
  s.total_accesses = t.ids.size();
  s.entries.resize(n);
  for (std::uint64_t i = 0; i < n; ++i) s.entries[i] = {ids[i], counts[i], cum[i]};
  return s;
}

inline void write_skew_csv(std::ostream& out, const SkewTable& s) {
  out << "id,count,cum_fraction\n";
  for (const auto& e : s.entries) {
    char b[32];
    std::snprintf(b, sizeof b, "%.17g", e.cum_fraction);
    // shortest text that reads back to the same double
    for (int prec = 1; prec <= 17; ++prec) {
      char c[32];
      std::snprintf(c, sizeof c, "%.*g", prec, e.cum_fraction);
      if (std::strtod(c, nullptr) == e.cum_fraction) {
        std::snprintf(b, sizeof b, "%s", c);
        break;
      }
    }
    out << e.id << "," << e.count << "," << b << "\n";
  }
}

inline EmbeddingDistribution estimate_distribution(const SkewTable& s, std::size_t vocab_size, double smoothing = 0.0) {
  std::vector<std::uint32_t> ids(s.entries.size());
  std::vector<std::uint64_t> counts(s.entries.size());
  for (std::size_t i = 0; i < ids.size(); ++i) {
    ids[i] = s.entries[i].id;
    counts[i] = s.entries[i].count;
  }
  ec_dist h = nullptr;
  detail::check(ec_estimate_distribution(ids.data(), counts.data(), ids.size(), s.total_accesses, vocab_size,
                                         smoothing, &h));
  return EmbeddingDistribution::adopt(h);
}

struct SampleClasses {
  std::vector<std::uint32_t> hot;
  std::vector<std::uint32_t> normal;
};

inline SampleClasses classify_samples(const Trace& t, std::span<const std::uint32_t> cache_ids) {
  const std::size_t q = t.num_samples();
  std::vector<std::uint8_t> hot(q);
  detail::check(ec_classify_samples(t.ids.data(), q, t.num_features, t.vocab_size, cache_ids.data(),
                                    cache_ids.size(), 0, hot.data()));
  SampleClasses c;
  for (std::size_t s = 0; s < q; ++s) (hot[s] ? c.hot : c.normal).push_back(static_cast<std::uint32_t>(s));
  return c;
}

struct BatchSchedule {
  std::vector<std::vector<std::uint32_t>> hot_batches;
  std::vector<std::vector<std::uint32_t>> normal_batches;
  std::int64_t batch_size = 0;
};

inline BatchSchedule build_schedule(const Trace& t, std::span<const std::uint32_t> cache_ids, std::int64_t batch_size,
                                    std::optional<std::uint64_t> shuffle_seed = std::nullopt) {
  if (batch_size < 1) throw ValidationError("batch size must be >= 1");
  const std::size_t q = t.num_samples();
  std::vector<std::uint32_t> order(q);
  std::uint64_t nh = 0;
  detail::check(ec_build_schedule(t.ids.data(), q, t.num_features, t.vocab_size, cache_ids.data(), cache_ids.size(), 0,
                                  shuffle_seed ? 1 : 0, shuffle_seed.value_or(0), order.data(), &nh));
  auto pack = [&](std::size_t lo, std::size_t hi) {
    std::vector<std::vector<std::uint32_t>> out;
    for (std::size_t p = lo; p < hi; p += static_cast<std::size_t>(batch_size))
      out.emplace_back(order.begin() + static_cast<std::ptrdiff_t>(p),
                       order.begin() + static_cast<std::ptrdiff_t>(std::min<std::size_t>(hi, p + batch_size)));
    return out;
  };
  BatchSchedule s;
  s.batch_size = batch_size;
  s.hot_batches = pack(0, nh);
  s.normal_batches = pack(nh, q);
  return s;
}

// -------------------------------------------------------------- simulator
// simulator.hpp:19-127.  Monte Carlo on the GPU; every SimResult field is
// bit-identical to the reference's.
class DiscreteSampler {
 public:
  explicit DiscreteSampler(const EmbeddingDistribution& dist) : dist_(&dist) { dist.sampler(); }
  // one draw (a kernel launch per call: batch draws go through sample_batch)
  std::uint32_t draw(SplitMix64& rng) const {
    std::uint32_t id = 0;
    detail::check(ec_sample_batch(dist_->sampler(), 1, 1, &rng.state(), &id));
    return id;
  }

 private:
  const EmbeddingDistribution* dist_;
};

struct Stat {
  double mean = 0.0;
  double std_error = 0.0;
};

struct SimResult {
  Stat unique_per_batch;
  Stat non_cached_unique;
  CostBreakdown measured_epoch_cost;
  double hot_batch_fraction = 0.0;
  std::vector<double> portion_usage;
};

namespace detail {
inline SimResult sim(const ec_sim_result& r) {
  SimResult s;
  s.unique_per_batch = {r.unique_mean, r.unique_std_error};
  s.non_cached_unique = {r.non_cached_mean, r.non_cached_std_error};
  s.measured_epoch_cost = cost(r.measured_epoch_cost);
  s.hot_batch_fraction = r.hot_batch_fraction;
  return s;
}
}  // namespace detail

inline std::vector<std::uint32_t> sample_batch(const EmbeddingDistribution& d, std::int64_t batch_size,
                                               std::int64_t lookups_per_sample, SplitMix64& rng) {
  if (batch_size < 1) throw ValidationError("batch size must be >= 1");
  if (lookups_per_sample < 1) throw ValidationError("lookups per sample must be >= 1");
  std::vector<std::uint32_t> out(static_cast<std::size_t>(batch_size * lookups_per_sample));
  detail::check(ec_sample_batch(d.sampler(), batch_size, lookups_per_sample, &rng.state(), out.data()));
  return out;
}

inline SimResult measure_unique(const EmbeddingDistribution& d, std::int64_t batch_size, std::int64_t trials,
                                std::uint64_t seed) {
  ec_sim_result r{};
  detail::check(ec_measure_unique(d.sampler(), batch_size, trials, seed, &r));
  return detail::sim(r);
}

inline SimResult simulate_epoch(const EmbeddingDistribution& d, const WorkloadSpec& spec,
                                std::span<const std::uint32_t> cache_ids, std::int64_t epochs, std::uint64_t seed) {
  const ec_workload w = spec.c();
  ec_sim_result r{};
  detail::check(ec_simulate_epoch(d.sampler(), &w, cache_ids.data(), cache_ids.size(), epochs, seed, &r));
  return detail::sim(r);
}

inline SimResult simulate_epoch(const Trace& t, std::int64_t batch_size, std::span<const std::uint32_t> cache_ids) {
  ec_sim_result r{};
  detail::check(ec_simulate_trace(t.ids.data(), t.num_samples(), t.num_features, t.vocab_size, batch_size,
                                  cache_ids.data(), cache_ids.size(), 0, &r));
  return detail::sim(r);
}

struct ScalingRow {
  DistributionKind kind = DistributionKind::zipf;
  double shape = 0.0;
  std::int64_t base_size = 0;
  std::int64_t scaled_size = 0;
  std::int64_t base_batch = 0;
  std::int64_t scaled_batch = 0;
  double baseline_ratio = 0.0;
  double embedding_ratio = 0.0;
  double total_ratio = 0.0;
  double growth_bound = 0.0;
  bool within_bound = false;
};

struct ScalingReport {
  std::int64_t factor = 0;
  std::int64_t base_batch = 0;
  std::int64_t lookups_per_sample = 0;
  std::vector<ScalingRow> rows;
  bool all_within_bounds = false;
  std::string calibration_note;
};

inline double scaling_growth_bound(DistributionKind kind) {
  if (kind == DistributionKind::zipf) return 2.0;
  if (kind == DistributionKind::exponential || kind == DistributionKind::half_normal) return 1.5;
  throw ValidationError("no growth bound for empirical distributions");
}

// simulator.hpp:99-104: catalog-extension growth of the per-batch coalesced
// cost, from the host cost model (purely analytical)
inline ScalingReport scaling_study(std::span<const DistributionSpec> specs, std::int64_t base_batch,
                                   std::int64_t lookups_per_sample, std::int64_t factor = 5) {
  if (base_batch < 1) throw ValidationError("batch size must be >= 1");
  if (lookups_per_sample < 1) throw ValidationError("lookups per sample must be >= 1");
  if (factor < 2) throw ValidationError("scale factor must be >= 2");
  ScalingReport rep;
  rep.factor = factor;
  rep.base_batch = base_batch;
  rep.lookups_per_sample = lookups_per_sample;
  rep.calibration_note =
      "default shapes zipf=2.5, exponential=100, half_normal=0.05 keep the embedding-cost growth under the bound "
      "when catalog and batch grow together; the earlier defaults (1, 5, 0.3) do not";
  rep.all_within_bounds = true;
  for (const DistributionSpec& spec : specs) {
    const auto base = materialize(spec);
    const auto grown = materialize_extended(spec, factor);
    const CostBreakdown c0 = coalesced_batch_cost(base, base_batch);
    const CostBreakdown c1 = coalesced_batch_cost(grown, factor * base_batch);
    ScalingRow r;
    r.kind = spec.kind;
    r.shape = spec.shape;
    r.base_size = static_cast<std::int64_t>(spec.size);
    r.scaled_size = static_cast<std::int64_t>(grown.size());
    r.base_batch = base_batch;
    r.scaled_batch = factor * base_batch;
    const double d = static_cast<double>(lookups_per_sample);
    r.baseline_ratio = (static_cast<double>(r.scaled_batch) * d) / (static_cast<double>(base_batch) * d);
    r.embedding_ratio = c1.embedding_cost / c0.embedding_cost;
    r.total_ratio = c1.total / c0.total;
    r.growth_bound = scaling_growth_bound(spec.kind);
    r.within_bound = r.embedding_ratio < r.growth_bound;
    rep.all_within_bounds = rep.all_within_bounds && r.within_bound;
    rep.rows.push_back(r);
  }
  return rep;
}

namespace detail {
// cached ids split by rank into `portions` near-equal contiguous chunks,
// hottest first (the first size % portions chunks one longer); -1 = uncached
inline std::vector<int> portion_of(const EmbeddingDistribution& d, std::span<const std::uint32_t> cache, int portions) {
  if (portions < 1) throw ValidationError("portions must be >= 1");
  if (portions > 64) throw ValidationError("at most 64 portions supported");
  if (cache.empty()) throw ValidationError("portion analysis needs a non-empty cache");
  if (static_cast<std::size_t>(portions) > cache.size()) throw ValidationError("more portions than cached embeddings");
  std::vector<std::size_t> ranks;
  for (std::uint32_t id : cache) ranks.push_back(d.rank_of(id));
  std::sort(ranks.begin(), ranks.end());
  std::vector<int> of(d.size(), -1);
  const std::size_t k = ranks.size(), per = k / portions, extra = k % portions;
  std::size_t at = 0;
  for (int p = 0; p < portions; ++p)
    for (std::size_t i = 0; i < per + (static_cast<std::size_t>(p) < extra ? 1 : 0); ++i) of[d.id_at_rank(ranks[at++])] = p;
  return of;
}
// add one per portion the sample touches
inline void touch(const std::vector<int>& of, std::span<const std::uint32_t> sample, std::vector<double>& sums) {
  std::uint64_t m = 0;
  for (std::uint32_t id : sample)
    if (of[id] >= 0) m |= std::uint64_t{1} << of[id];
  for (; m; m &= m - 1) sums[static_cast<std::size_t>(std::countr_zero(m))] += 1.0;
}
}  // namespace detail

// simulator.hpp:110-126.  Draws on the GPU (the same stream positions as the
// reference's per-trial SplitMix64), touch counting on the host.
inline std::vector<double> portion_usage(const EmbeddingDistribution& d, std::span<const std::uint32_t> cache_ids,
                                         int portions, std::int64_t batch_size, std::int64_t lookups_per_sample,
                                         std::int64_t trials, std::uint64_t seed) {
  if (batch_size < 1) throw ValidationError("batch size must be >= 1");
  if (lookups_per_sample < 1) throw ValidationError("lookups per sample must be >= 1");
  if (trials < 1) throw ValidationError("trials must be >= 1");
  const std::vector<int> of = detail::portion_of(d, cache_ids, portions);
  std::vector<double> sums(static_cast<std::size_t>(portions), 0.0);
  const auto f = static_cast<std::size_t>(lookups_per_sample);
  for (std::int64_t tr = 0; tr < trials; ++tr) {
    SplitMix64 rng(substream_seed(seed, static_cast<std::uint64_t>(tr)));
    const auto ids = sample_batch(d, batch_size, lookups_per_sample, rng);
    for (std::size_t s = 0; s < static_cast<std::size_t>(batch_size); ++s)
      detail::touch(of, std::span<const std::uint32_t>(ids.data() + s * f, f), sums);
  }
  for (double& v : sums) v /= static_cast<double>(trials);
  return sums;
}

inline std::vector<double> portion_usage(const Trace& t, std::span<const std::uint32_t> cache_ids, int portions,
                                         std::int64_t batch_size) {
  if (batch_size < 1) throw ValidationError("batch size must be >= 1");
  const auto dist = estimate_distribution(build_skew_table(t), t.vocab_size);
  const std::vector<int> of = detail::portion_of(dist, cache_ids, portions);
  const std::size_t b = static_cast<std::size_t>(batch_size), full = t.num_samples() / b;
  if (full == 0) throw ValidationError("trace shorter than one batch of " + std::to_string(batch_size));
  std::vector<double> sums(static_cast<std::size_t>(portions), 0.0);
  for (std::size_t s = 0; s < full * b; ++s) detail::touch(of, t.sample(s), sums);
  for (double& v : sums) v /= static_cast<double>(full);
  return sums;
}

}  // namespace embcomm
