// Host side of the reference's core/ API surface: access distributions,
// expected-communication-cost model and the cache-placement planner.
//
// These stay on the host on purpose: every result is an fp64
// value the reference computes with a specific summation order, and the
// drop-in promise is bit-identical numbers.  The formulas below restate the
// reference's (file:line cited per function); they are evaluated in the same
// order with the same libm calls.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <optional>
#include <queue>
#include <unordered_map>
#include <vector>

#include "common.hpp"
#include "host_model.hpp"

using ec::invalid;

namespace ec {

namespace {
thread_local std::string g_last_error;

// Compensated sum (core/src/detail/accumulate.hpp:10-20).
double compensated_sum(const double* v, size_t n) {
  double s = 0.0, c = 0.0;
  for (size_t i = 0; i < n; ++i) {
    const double y = v[i] - c;
    const double t = s + y;
    c = (t - s) - y;
    s = t;
  }
  return s;
}
}  // namespace

void set_last_error(const std::string& m) { g_last_error = m; }
const char* last_error() { return g_last_error.c_str(); }

// ------------------------------------------------------------ Distribution
// EmbeddingDistribution::from_probabilities, core/src/distribution.cpp:13-55.
Dist Dist::from_probabilities(std::vector<double> p) {
  if (p.empty()) invalid("distribution needs at least one embedding");
  if (p.size() > static_cast<size_t>(UINT32_MAX)) invalid("vocabulary too large for 32-bit embedding ids");
  for (size_t i = 0; i < p.size(); ++i) {
    if (!(p[i] >= 0.0 && p[i] <= 1.0))
      invalid("probability out of [0,1] at id " + std::to_string(i) + ": " + std::to_string(p[i]));
  }
  const double total = compensated_sum(p.data(), p.size());
  if (std::abs(total - 1.0) > 1e-9)
    invalid("probabilities sum to " + std::to_string(total) + ", expected 1 within 1e-9");

  Dist d;
  const size_t n = p.size();
  d.rank_to_id.resize(n);
  std::iota(d.rank_to_id.begin(), d.rank_to_id.end(), 0u);
  bool non_increasing = true;
  for (size_t i = 1; i < n && non_increasing; ++i) non_increasing = !(p[i] > p[i - 1]);
  if (!non_increasing) {
    // Probability descending, ties to the smaller id (distribution.cpp:41-45).
    std::sort(d.rank_to_id.begin(), d.rank_to_id.end(), [&p](uint32_t a, uint32_t b) {
      return p[a] != p[b] ? p[a] > p[b] : a < b;
    });
  }
  d.ranked.resize(n);
  d.id_to_rank.resize(n);
  for (size_t r = 0; r < n; ++r) {
    d.ranked[r] = p[d.rank_to_id[r]];
    d.id_to_rank[d.rank_to_id[r]] = static_cast<uint32_t>(r);
  }
  return d;
}

// Parametric weight profiles (core/src/distribution_spec.cpp:19-57): rank
// x = i+1, Kahan-normalised.  rank_scale = base size (catalog extension) or
// the size itself.
Dist Dist::parametric(int kind, uint64_t count, double shape, double rank_scale) {
  std::vector<double> w(count);
  switch (kind) {
    case EC_ZIPF:
      for (uint64_t i = 0; i < count; ++i) w[i] = std::pow(static_cast<double>(i + 1), -shape);
      break;
    case EC_EXPONENTIAL:
      for (uint64_t i = 0; i < count; ++i)
        w[i] = std::exp(-shape * static_cast<double>(i + 1) / rank_scale);
      break;
    case EC_HALF_NORMAL: {
      const double two_s2 = 2.0 * shape * shape;
      for (uint64_t i = 0; i < count; ++i) {
        const double x = static_cast<double>(i + 1) / rank_scale;
        w[i] = std::exp(-(x * x) / two_s2);
      }
      break;
    }
    default:
      invalid("empirical specs carry explicit probabilities");
  }
  const double total = compensated_sum(w.data(), w.size());
  if (!(total > 0.0) || !std::isfinite(total))
    invalid("shape parameter " + std::to_string(shape) + " too extreme: weights vanish");
  for (double& v : w) v /= total;
  return from_probabilities(std::move(w));
}

void Dist::check_id(uint32_t id) const {
  if (id >= size())
    invalid("embedding id " + std::to_string(id) + " out of range [0, " + std::to_string(size()) + ")");
}
void Dist::check_rank(uint64_t r) const {
  if (r >= size()) invalid("rank " + std::to_string(r) + " out of range");
}

// ------------------------------------------------------------- cost model
// batch_presence_prob, core/src/cost_model.cpp:36-46.
double presence(double p, int64_t b) {
  if (!(p >= 0.0 && p <= 1.0))
    invalid("presence probability needs p in [0,1], got " + std::to_string(p));
  if (b < 1) invalid("presence probability needs b >= 1");
  if (b == 1) return p;
  if (p == 1.0) return 1.0;
  return -std::expm1(static_cast<double>(b) * std::log1p(-p));
}

// expected_unique_from_rank, cost_model.cpp:48-59: naive sum, rank order.
double unique_from_rank(const Dist& d, int64_t b, uint64_t first) {
  if (first > d.size()) invalid("rank offset " + std::to_string(first) + " out of range");
  double s = 0.0;
  for (size_t r = first; r < d.ranked.size(); ++r) s += presence(d.ranked[r], b);
  return s;
}

void validate(const ec_workload& w) {
  if (w.batch_size < 1) invalid("batch size must be >= 1");
  if (w.num_samples < w.batch_size)
    invalid("batch size " + std::to_string(w.batch_size) + " exceeds dataset size " +
            std::to_string(w.num_samples));
  if (w.lookups_per_sample < 1) invalid("lookups per sample must be >= 1");
}

// (Q/b) batches x distinct sum x d, cost_model.cpp:12-18.
static double epoch_embedding(double unique_sum, const ec_workload& w) {
  const double batches = static_cast<double>(w.num_samples) / static_cast<double>(w.batch_size);
  return batches * unique_sum * static_cast<double>(w.lookups_per_sample);
}

static ec_cost make_cost(double index, double emb) { return ec_cost{index, emb, index + emb}; }

// cached_epoch_cost, cost_model.cpp:88-111: rank-order walk skipping cached ids.
ec_cost cached_cost(const Dist& d, const ec_workload& w, const uint32_t* cache, uint64_t k) {
  validate(w);
  std::vector<char> cached(d.size(), 0);
  for (uint64_t i = 0; i < k; ++i) {
    if (cache[i] >= d.size())
      invalid("cache id " + std::to_string(cache[i]) + " out of range [0, " + std::to_string(d.size()) + ")");
    cached[cache[i]] = 1;
  }
  double s = 0.0;
  for (size_t r = 0; r < d.size(); ++r) {
    if (cached[d.rank_to_id[r]]) continue;
    s += presence(d.ranked[r], w.batch_size);
  }
  return make_cost(static_cast<double>(w.num_samples), epoch_embedding(s, w));
}

// ---------------------------------------------------------------- planner
void validate(const ec_device_model& m) {  // cache_planner.cpp:90-112
  if (m.activation_params_per_sample < 1) invalid("activation footprint must be >= 1 parameter");
  if (m.total_params < m.activation_params_per_sample)
    invalid("no feasible batch: device memory " + std::to_string(m.total_params) +
            " cannot hold one sample's activations (" +
            std::to_string(m.activation_params_per_sample) + ")");
  if (m.embedding_params < 1) invalid("embedding footprint must be >= 1 parameter");
  if (!(m.memory_efficiency > 0.0 && m.memory_efficiency <= 1.0))
    invalid("memory efficiency must be in (0, 1]");
}

// Eq. 7, max_batch_size (cache_planner.cpp:114-136).
std::optional<int64_t> batch_fit(const ec_device_model& m, int64_t k) {
  if (k < 0) invalid("cache size must be >= 0");
  if (m.memory_efficiency == 1.0) {
    int64_t held = 0;
    if (__builtin_mul_overflow(k, m.embedding_params, &held)) return std::nullopt;
    const int64_t left = m.total_params - held;
    if (left < m.activation_params_per_sample) return std::nullopt;
    return left / m.activation_params_per_sample;
  }
  const long double usable = static_cast<long double>(m.memory_efficiency) *
                             static_cast<long double>(m.total_params);
  const long double left =
      usable - static_cast<long double>(k) * static_cast<long double>(m.embedding_params);
  const long double slots = left / static_cast<long double>(m.activation_params_per_sample);
  if (slots < 1.0L) return std::nullopt;
  return static_cast<int64_t>(std::floor(slots));
}

namespace {
// The cache-size optimisation problem: cache = top-k prefix, batch from Eq. 7
// clamped to Q, cost = Eq. 6 on the prefix (cache_planner.cpp:24-80).
struct Problem {
  const Dist& d;
  const ec_device_model& m;
  int64_t q, lookups;

  std::optional<int64_t> batch(int64_t k) const {
    auto b = batch_fit(m, k);
    if (!b) return b;
    return std::min(*b, q);
  }
  ec_cost cost(int64_t k) const {
    const int64_t b = *batch(k);
    validate(ec_workload{q, b, lookups});
    const double s = unique_from_rank(d, b, static_cast<uint64_t>(k));
    const double emb = (static_cast<double>(q) / static_cast<double>(b)) * s * static_cast<double>(lookups);
    return make_cost(static_cast<double>(q), emb);
  }
  int64_t largest_feasible() const {  // batch() is non-increasing in k
    if (!batch(0)) return -1;
    int64_t lo = 0, hi = static_cast<int64_t>(d.size());
    while (lo < hi) {
      const int64_t mid = lo + (hi - lo + 1) / 2;
      if (batch(mid)) lo = mid; else hi = mid - 1;
    }
    return lo;
  }
  Plan plan(int64_t k) const {
    Plan p;
    p.head.cache_size = static_cast<uint64_t>(k);
    p.head.batch_size = *batch(k);
    p.head.expected_epoch_cost = cost(k);
    p.head.feasible = 1;
    p.head.used_scan_fallback = 0;
    p.k = k;
    return p;
  }
};
}  // namespace

Plan plan_scan(const Dist& d, const ec_device_model& m, const ec_workload& w) {
  validate(m);
  validate(w);
  const Problem pr{d, m, w.num_samples, w.lookups_per_sample};
  const int64_t kmax = pr.largest_feasible();
  if (kmax < 0) return Plan{};
  int64_t best = 0;
  double best_total = pr.cost(0).total;
  for (int64_t k = 1; k <= kmax; ++k) {
    const double t = pr.cost(k).total;
    if (t < best_total) { best_total = t; best = k; }
  }
  return pr.plan(best);
}

// optimal_cache_size_search, cache_planner.cpp:206-289: probe marginal signs
// (all k up to 1024, else 64 evenly spaced), fall back to the scan when the
// sign pattern is not monotone, otherwise binary-search the first
// non-negative marginal and return the cheapest point evaluated.
Plan plan_search(const Dist& d, const ec_device_model& m, const ec_workload& w) {
  validate(m);
  validate(w);
  const Problem pr{d, m, w.num_samples, w.lookups_per_sample};
  const int64_t kmax = pr.largest_feasible();
  if (kmax < 0) return Plan{};
  if (kmax == 0) return pr.plan(0);

  std::unordered_map<int64_t, double> seen;
  auto total = [&](int64_t k) {
    auto it = seen.find(k);
    if (it != seen.end()) return it->second;
    const double t = pr.cost(k).total;
    seen.emplace(k, t);
    return t;
  };
  auto stops_paying = [&](int64_t k) { return total(k + 1) >= total(k); };

  std::vector<int64_t> probe;
  if (kmax <= 1024) {
    for (int64_t i = 0; i < kmax; ++i) probe.push_back(i);
  } else {
    for (int64_t i = 0; i < 64; ++i) probe.push_back(i * (kmax - 1) / 63);
    probe.erase(std::unique(probe.begin(), probe.end()), probe.end());
  }
  bool any_nonneg = false;
  int64_t last_neg = -1, first_nonneg = kmax;
  for (const int64_t k : probe) {
    if (stops_paying(k)) {
      if (!any_nonneg) first_nonneg = k;
      any_nonneg = true;
    } else if (any_nonneg) {
      Plan p = plan_scan(d, m, w);
      p.head.used_scan_fallback = 1;
      return p;
    } else {
      last_neg = k;
    }
  }
  int64_t lo = last_neg + 1, hi = first_nonneg;
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (stops_paying(mid)) hi = mid; else lo = mid + 1;
  }
  int64_t best = lo;
  double best_total = total(best);
  std::vector<std::pair<int64_t, double>> pts(seen.begin(), seen.end());
  std::sort(pts.begin(), pts.end());
  for (const auto& [k, t] : pts)
    if (t < best_total) { best_total = t; best = k; }
  return pr.plan(best);
}

// delta_comm, cache_planner.cpp:138-186 (Eqs. 8-12).
ec_marginal marginal(const Dist& d, const ec_device_model& m, int64_t q, int64_t k) {
  validate(m);
  if (q < 1) invalid("dataset size must be >= 1");
  if (k < 0 || static_cast<uint64_t>(k) >= d.size())
    invalid("no candidate embedding beyond cache size " + std::to_string(k));
  const auto b = batch_fit(m, k);
  const auto b1 = batch_fit(m, k + 1);
  if (!b || !b1) invalid("cache of size " + std::to_string(k + 1) + " leaves no room for a batch");
  auto traffic = [&](int64_t bb, int64_t kk) {  // (Q/b) * sum, no lookup multiplier
    return unique_from_rank(d, bb, static_cast<uint64_t>(kk)) * static_cast<double>(q) /
           static_cast<double>(bb);
  };
  const double with = traffic(*b1, k + 1);
  const double without = traffic(*b, k);
  ec_marginal r{};
  r.candidate_id = d.rank_to_id[static_cast<size_t>(k)];
  r.delta_comm = with - without;
  r.recommend = r.delta_comm < 0.0;
  r.presence_gain = presence(d.ranked[static_cast<size_t>(k)], *b);
  double thr = 0.0;
  const double bd = static_cast<double>(*b), bn = static_cast<double>(*b1);
  for (size_t rr = static_cast<size_t>(k) + 1; rr < d.size(); ++rr) {
    const double p = d.ranked[rr];
    thr += (bd * presence(p, *b1) - bn * presence(p, *b)) / bn;
  }
  r.threshold = thr;
  const bool rearranged = r.presence_gain > thr;
  const double scale = std::max({std::abs(with), std::abs(without), 1.0});
  if (std::abs(r.delta_comm) > 1e-9 * scale && rearranged != static_cast<bool>(r.recommend))
    invariant("marginal caching test: direct and rearranged forms disagree");
  return r;
}

}  // namespace ec

// ===================================================================== ABI
using namespace ec;

struct ec_dist_s {
  Dist d;
};

static const Dist& D(ec_dist h) {
  if (!h) invalid("null distribution handle");
  return h->d;
}

extern "C" {

const char* ec_last_error(void) { return ec::last_error(); }
const char* ec_version(void) { return "embcomm-b200 0.1.0 (sm_100a)"; }
const char* ec_cost_units_note(void) { return "one unit = one embedding vector = one transmitted index"; }
const char* ec_rng_algorithm(void) { return "splitmix64"; }
uint64_t ec_substream_seed(uint64_t master, uint64_t index) { return substream(master, index); }

int ec_dist_from_probabilities(const double* p, uint64_t n, ec_dist* out) {
  return guard([&] {
    if (n && !p) invalid("null probabilities");
    *out = new ec_dist_s{Dist::from_probabilities(std::vector<double>(p, p + n))};
  });
}
int ec_dist_uniform(uint64_t n, ec_dist* out) {
  return guard([&] {
    if (n == 0) invalid("distribution needs at least one embedding");
    *out = new ec_dist_s{Dist::from_probabilities(std::vector<double>(n, 1.0 / static_cast<double>(n)))};
  });
}
static void check_spec(int kind, uint64_t size, double shape) {
  if (kind == EC_EMPIRICAL) invalid("use ec_dist_from_probabilities for explicit probabilities");
  if (kind < 0 || kind > EC_EMPIRICAL) invalid("unknown distribution kind");
  if (size == 0) invalid("distribution size must be >= 1");
  if (!(shape > 0.0) || !std::isfinite(shape)) invalid("shape parameter must be positive and finite");
}
int ec_dist_materialize(int kind, uint64_t size, double shape, ec_dist* out) {
  return guard([&] {
    check_spec(kind, size, shape);
    *out = new ec_dist_s{Dist::parametric(kind, size, shape, static_cast<double>(size))};
  });
}
int ec_dist_materialize_extended(int kind, uint64_t size, double shape, int64_t factor, ec_dist* out) {
  return guard([&] {
    if (kind == EC_EMPIRICAL) invalid("materialize_extended requires a parametric distribution");
    check_spec(kind, size, shape);
    if (factor < 1) invalid("scale factor must be >= 1");
    uint64_t count = 0;
    if (__builtin_mul_overflow(size, static_cast<uint64_t>(factor), &count)) invalid("scaled size overflows");
    *out = new ec_dist_s{Dist::parametric(kind, count, shape, static_cast<double>(size))};
  });
}
int ec_default_shape(int kind, double* out) {
  return guard([&] {
    switch (kind) {  // distribution_spec.hpp:22-24
      case EC_ZIPF: *out = 2.5; break;
      case EC_EXPONENTIAL: *out = 100.0; break;
      case EC_HALF_NORMAL: *out = 0.05; break;
      default: invalid("empirical distributions have no shape parameter");
    }
  });
}
void ec_dist_destroy(ec_dist d) { delete d; }
uint64_t ec_dist_size(ec_dist d) { return d ? d->d.size() : 0; }
int ec_dist_prob(ec_dist h, uint32_t id, double* out) {
  return guard([&] { D(h).check_id(id); *out = h->d.ranked[h->d.id_to_rank[id]]; });
}
int ec_dist_prob_at_rank(ec_dist h, uint64_t r, double* out) {
  return guard([&] { D(h).check_rank(r); *out = h->d.ranked[r]; });
}
int ec_dist_id_at_rank(ec_dist h, uint64_t r, uint32_t* out) {
  return guard([&] { D(h).check_rank(r); *out = h->d.rank_to_id[r]; });
}
int ec_dist_rank_of(ec_dist h, uint32_t id, uint64_t* out) {
  return guard([&] { D(h).check_id(id); *out = h->d.id_to_rank[id]; });
}
int ec_dist_top_ids(ec_dist h, uint64_t k, uint32_t* out) {
  return guard([&] {
    if (k > D(h).size())
      invalid("cannot take top " + std::to_string(k) + " of " + std::to_string(h->d.size()) + " embeddings");
    std::memcpy(out, h->d.rank_to_id.data(), k * sizeof(uint32_t));
  });
}
int ec_dist_mass_of(ec_dist h, const uint32_t* ids, uint64_t n, double* out) {
  return guard([&] {
    double m = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
      D(h).check_id(ids[i]);
      m += h->d.ranked[h->d.id_to_rank[ids[i]]];
    }
    *out = m;
  });
}
int ec_dist_export(ec_dist h, double* p, uint32_t* r2i) {
  return guard([&] {
    const Dist& d = D(h);
    if (p) std::memcpy(p, d.ranked.data(), d.size() * sizeof(double));
    if (r2i) std::memcpy(r2i, d.rank_to_id.data(), d.size() * sizeof(uint32_t));
  });
}

int ec_dist_clone(ec_dist h, ec_dist* out) {
  return guard([&] {
    if (!out) invalid("null output");
    *out = new ec_dist_s{D(h)};
  });
}
int ec_dist_ranked_view(ec_dist h, const double** ranked) {
  return guard([&] {
    if (!ranked) invalid("null output");
    *ranked = D(h).ranked.data();
  });
}

int ec_workload_validate(const ec_workload* w) { return guard([&] { validate(*w); }); }
int ec_batch_presence_prob(double p, int64_t b, double* out) {
  return guard([&] { *out = presence(p, b); });
}
int ec_expected_unique_per_batch(ec_dist h, int64_t b, double* out) {
  return guard([&] { *out = unique_from_rank(D(h), b, 0); });
}
int ec_expected_unique_from_rank(ec_dist h, int64_t b, uint64_t first, double* out) {
  return guard([&] { *out = unique_from_rank(D(h), b, first); });
}
int ec_coalesced_batch_cost(ec_dist h, int64_t b, ec_cost* out) {
  return guard([&] { *out = make_cost(static_cast<double>(b), unique_from_rank(D(h), b, 0)); });
}
int ec_baseline_epoch_cost(const ec_workload* w, double* out) {
  return guard([&] {
    validate(*w);
    *out = static_cast<double>(w->num_samples) * static_cast<double>(w->lookups_per_sample);
  });
}
int ec_coalesced_epoch_cost(ec_dist h, const ec_workload* w, ec_cost* out) {
  return guard([&] {
    validate(*w);
    *out = make_cost(static_cast<double>(w->num_samples),
                     epoch_embedding(unique_from_rank(D(h), w->batch_size, 0), *w));
  });
}
int ec_cached_epoch_cost(ec_dist h, const ec_workload* w, const uint32_t* c, uint64_t k, ec_cost* out) {
  return guard([&] { *out = cached_cost(D(h), *w, c, k); });
}

int ec_device_model_validate(const ec_device_model* m) { return guard([&] { validate(*m); }); }
int ec_max_batch_size(const ec_device_model* m, int64_t k, int64_t* out) {
  return guard([&] {
    const auto b = batch_fit(*m, k);
    *out = b ? *b : -1;
  });
}
int ec_delta_comm(ec_dist h, const ec_device_model* m, int64_t q, int64_t k, ec_marginal* out) {
  return guard([&] { *out = marginal(D(h), *m, q, k); });
}
static void emit_plan(const Dist& d, const Plan& p, ec_cache_plan* out, uint32_t* ids) {
  *out = p.head;
  if (ids && p.head.feasible)
    std::memcpy(ids, d.rank_to_id.data(), p.head.cache_size * sizeof(uint32_t));
}
int ec_optimal_cache_size_scan(ec_dist h, const ec_device_model* m, const ec_workload* w,
                               ec_cache_plan* out, uint32_t* ids) {
  return guard([&] { emit_plan(D(h), plan_scan(h->d, *m, *w), out, ids); });
}
int ec_optimal_cache_size_search(ec_dist h, const ec_device_model* m, const ec_workload* w,
                                 ec_cache_plan* out, uint32_t* ids) {
  return guard([&] { emit_plan(D(h), plan_search(h->d, *m, *w), out, ids); });
}
int ec_memory_io_proxy(ec_dist h, const ec_workload* w, const uint32_t* c, uint64_t k, double* out) {
  return guard([&] { *out = cached_cost(D(h), *w, c, k).embedding_cost; });
}

int ec_place_topk_global(const ec_dist* dists, uint32_t T, uint64_t budget, uint64_t* k_out) {
  return guard([&] {
    uint64_t total_rows = 0;
    for (uint32_t t = 0; t < T; ++t) {
      total_rows += D(dists[t]).size();
      k_out[t] = 0;
    }
    budget = std::min(budget, total_rows);
    // k-way merge over the tables' ranked (non-increasing) probabilities.
    using Item = std::pair<double, uint32_t>;  // (p, table); max-heap, ties -> lower table
    auto cmp = [](const Item& a, const Item& b) {
      return a.first != b.first ? a.first < b.first : a.second > b.second;
    };
    std::priority_queue<Item, std::vector<Item>, decltype(cmp)> heap(cmp);
    for (uint32_t t = 0; t < T; ++t) heap.emplace(dists[t]->d.ranked[0], t);
    for (uint64_t taken = 0; taken < budget; ++taken) {
      const auto [p, t] = heap.top();
      heap.pop();
      const uint64_t next = ++k_out[t];
      if (next < dists[t]->d.size()) heap.emplace(dists[t]->d.ranked[next], t);
    }
  });
}

}  // extern "C"

namespace ec {
const Dist& dist_of(ec_dist h) { return D(h); }
ec_dist make_dist(Dist&& d) { return new ec_dist_s{std::move(d)}; }
}  // namespace ec
