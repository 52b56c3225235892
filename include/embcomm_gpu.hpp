// embcomm_gpu.hpp — header-only C++ mirror of the reference's core/ hot-path
// API (namespace embcomm, /root/reference/proj/core/include/embcomm/*.hpp)
// over the C-ABI of libembcomm_gpu.so (embcomm_gpu.h).
//
// A reference caller switches by including this header instead of the
// reference headers and linking libembcomm_gpu.so: the same names, argument
// meaning and exceptions (ValidationError / InvariantError), with the
// simulator and the lookup engine running on the GPU.  Value types mirror the
// reference's (WorkloadSpec, CostBreakdown, DeviceModel, CachePlan, SimResult,
// Trace).  std::span inputs become (pointer, size) internally.
#pragma once

#include <cstdint>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "embcomm_gpu.h"

namespace embcomm {

// error.hpp:10-19
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

inline constexpr const char* kCostUnitsNote = "one unit = one embedding vector = one transmitted index";
inline constexpr const char* kRngAlgorithm = "splitmix64";

inline std::uint64_t substream_seed(std::uint64_t master, std::uint64_t index) {
  return ec_substream_seed(master, index);
}

// SplitMix64 state holder (rng.hpp:12-27); draws happen on the GPU in
// sample_batch, which advances state_ exactly as the reference does.
class SplitMix64 {
 public:
  explicit SplitMix64(std::uint64_t seed) : state_(seed) {}
  std::uint64_t next() {
    std::uint64_t z = (state_ += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  double next_double() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  std::uint64_t& state() { return state_; }

 private:
  std::uint64_t state_;
};

// EmbeddingDistribution (distribution.hpp:19-49).
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
  EmbeddingDistribution(EmbeddingDistribution&& o) noexcept : h_(std::exchange(o.h_, nullptr)),
                                                             s_(std::exchange(o.s_, nullptr)) {}
  EmbeddingDistribution& operator=(EmbeddingDistribution&& o) noexcept {
    std::swap(h_, o.h_);
    std::swap(s_, o.s_);
    return *this;
  }
  EmbeddingDistribution(const EmbeddingDistribution&) = delete;
  ~EmbeddingDistribution() {
    if (s_) ec_sampler_destroy(s_);
    if (h_) ec_dist_destroy(h_);
  }

  std::size_t size() const noexcept { return ec_dist_size(h_); }
  double prob(std::uint32_t id) const { double v; detail::check(ec_dist_prob(h_, id, &v)); return v; }
  double prob_at_rank(std::size_t r) const { double v; detail::check(ec_dist_prob_at_rank(h_, r, &v)); return v; }
  std::uint32_t id_at_rank(std::size_t r) const { std::uint32_t v; detail::check(ec_dist_id_at_rank(h_, r, &v)); return v; }
  std::size_t rank_of(std::uint32_t id) const { std::uint64_t v; detail::check(ec_dist_rank_of(h_, id, &v)); return v; }
  std::vector<double> ranked_probs() const {
    std::vector<double> p(size());
    detail::check(ec_dist_export(h_, p.data(), nullptr));
    return p;
  }
  std::vector<std::uint32_t> top_ids(std::size_t k) const {
    std::vector<std::uint32_t> v(k);
    detail::check(ec_dist_top_ids(h_, k, v.data()));
    return v;
  }
  double mass_of(std::span<const std::uint32_t> ids) const {
    double v;
    detail::check(ec_dist_mass_of(h_, ids.data(), ids.size(), &v));
    return v;
  }

  ec_dist handle() const { return h_; }
  static EmbeddingDistribution adopt(ec_dist h) { return EmbeddingDistribution(h); }
  // GPU sampler bound to this distribution (built on first use, device 0).
  ec_sampler sampler(int device = 0) const {
    if (!s_) detail::check(ec_sampler_create(h_, device, &s_));
    return s_;
  }

 private:
  explicit EmbeddingDistribution(ec_dist h) : h_(h) {}
  ec_dist h_ = nullptr;
  mutable ec_sampler s_ = nullptr;
};

// distribution_spec.hpp:14-67 (parametric kinds)
enum class DistributionKind { zipf = EC_ZIPF, exponential = EC_EXPONENTIAL, half_normal = EC_HALF_NORMAL,
                              empirical = EC_EMPIRICAL };

inline EmbeddingDistribution materialize_parametric(DistributionKind kind, std::size_t size, double shape) {
  ec_dist h = nullptr;
  detail::check(ec_dist_materialize(static_cast<int>(kind), size, shape, &h));
  return EmbeddingDistribution::adopt(h);
}

// cost_model.hpp:17-64
struct WorkloadSpec {
  std::int64_t num_samples, batch_size, lookups_per_sample;
  WorkloadSpec(std::int64_t q, std::int64_t b, std::int64_t d) : num_samples(q), batch_size(b), lookups_per_sample(d) {
    const ec_workload w{q, b, d};
    detail::check(ec_workload_validate(&w));
  }
  ec_workload c() const { return {num_samples, batch_size, lookups_per_sample}; }
};

struct CostBreakdown {
  double index_cost = 0.0, embedding_cost = 0.0, total = 0.0;
  std::string units_note = kCostUnitsNote;
};

namespace detail {
inline CostBreakdown cost(const ec_cost& c) { return {c.index_cost, c.embedding_cost, c.total, kCostUnitsNote}; }
}  // namespace detail

inline double batch_presence_prob(double p, std::int64_t b) {
  double v;
  detail::check(ec_batch_presence_prob(p, b, &v));
  return v;
}
inline double expected_unique_per_batch(const EmbeddingDistribution& d, std::int64_t b) {
  double v;
  detail::check(ec_expected_unique_per_batch(d.handle(), b, &v));
  return v;
}
inline double expected_unique_from_rank(const EmbeddingDistribution& d, std::int64_t b, std::size_t first) {
  double v;
  detail::check(ec_expected_unique_from_rank(d.handle(), b, first, &v));
  return v;
}
inline CostBreakdown coalesced_batch_cost(const EmbeddingDistribution& d, std::int64_t b) {
  ec_cost c;
  detail::check(ec_coalesced_batch_cost(d.handle(), b, &c));
  return detail::cost(c);
}
inline double baseline_epoch_cost(const WorkloadSpec& s) {
  const ec_workload w = s.c();
  double v;
  detail::check(ec_baseline_epoch_cost(&w, &v));
  return v;
}
inline CostBreakdown coalesced_epoch_cost(const EmbeddingDistribution& d, const WorkloadSpec& s) {
  const ec_workload w = s.c();
  ec_cost c;
  detail::check(ec_coalesced_epoch_cost(d.handle(), &w, &c));
  return detail::cost(c);
}
inline CostBreakdown cached_epoch_cost(const EmbeddingDistribution& d, const WorkloadSpec& s,
                                       std::span<const std::uint32_t> cache) {
  const ec_workload w = s.c();
  ec_cost c;
  detail::check(ec_cached_epoch_cost(d.handle(), &w, cache.data(), cache.size(), &c));
  return detail::cost(c);
}

// cache_planner.hpp:16-81
struct DeviceModel {
  std::int64_t total_params, activation_params_per_sample, embedding_params;
  double memory_efficiency = 1.0;
  DeviceModel(std::int64_t m, std::int64_t a, std::int64_t e, double eff = 1.0)
      : total_params(m), activation_params_per_sample(a), embedding_params(e), memory_efficiency(eff) {
    const ec_device_model x = c();
    detail::check(ec_device_model_validate(&x));
  }
  ec_device_model c() const { return {total_params, activation_params_per_sample, embedding_params, memory_efficiency}; }
};

inline std::optional<std::int64_t> max_batch_size(const DeviceModel& m, std::int64_t k) {
  const ec_device_model x = m.c();
  std::int64_t v;
  detail::check(ec_max_batch_size(&x, k, &v));
  if (v < 0) return std::nullopt;
  return v;
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
  ec_cache_plan p;
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
inline CachePlan optimal_cache_size_search(const EmbeddingDistribution& d, const DeviceModel& m, const WorkloadSpec& s) {
  return detail::plan(ec_optimal_cache_size_search, d, m, s);
}
inline double memory_io_proxy(const EmbeddingDistribution& d, const WorkloadSpec& s,
                              std::span<const std::uint32_t> cache) {
  const ec_workload w = s.c();
  double v;
  detail::check(ec_memory_io_proxy(d.handle(), &w, cache.data(), cache.size(), &v));
  return v;
}

// simulator.hpp:29-74 — Monte Carlo on the GPU, bit-identical SimResult
struct Stat {
  double mean = 0.0, std_error = 0.0;
};
struct SimResult {
  Stat unique_per_batch, non_cached_unique;
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

inline std::vector<std::uint32_t> sample_batch(const EmbeddingDistribution& d, std::int64_t b, std::int64_t lookups,
                                               SplitMix64& rng) {
  if (b < 1) throw ValidationError("batch size must be >= 1");
  if (lookups < 1) throw ValidationError("lookups per sample must be >= 1");
  std::vector<std::uint32_t> out(static_cast<std::size_t>(b * lookups));
  detail::check(ec_sample_batch(d.sampler(), b, lookups, &rng.state(), out.data()));
  return out;
}
inline SimResult measure_unique(const EmbeddingDistribution& d, std::int64_t b, std::int64_t trials,
                                std::uint64_t seed) {
  ec_sim_result r;
  detail::check(ec_measure_unique(d.sampler(), b, trials, seed, &r));
  return detail::sim(r);
}
inline SimResult simulate_epoch(const EmbeddingDistribution& d, const WorkloadSpec& s,
                                std::span<const std::uint32_t> cache, std::int64_t epochs, std::uint64_t seed) {
  const ec_workload w = s.c();
  ec_sim_result r;
  detail::check(ec_simulate_epoch(d.sampler(), &w, cache.data(), cache.size(), epochs, seed, &r));
  return detail::sim(r);
}

// trace.hpp:18-30
struct Trace {
  std::int64_t num_features = 0;
  std::size_t vocab_size = 0;
  std::vector<std::uint32_t> ids;
  std::size_t num_samples() const {
    return num_features > 0 ? ids.size() / static_cast<std::size_t>(num_features) : 0;
  }
};

inline SimResult simulate_epoch(const Trace& t, std::int64_t b, std::span<const std::uint32_t> cache, int device = 0) {
  ec_sim_result r;
  detail::check(ec_simulate_trace(t.ids.data(), t.num_samples(), t.num_features, t.vocab_size, b, cache.data(),
                                  cache.size(), device, &r));
  return detail::sim(r);
}

}  // namespace embcomm
