// TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.
//
// extern "C" wrapper around the *unmodified* reference library (embcomm
// core, compiled from /root/reference/proj/core/src by oracle/Makefile into
// oracle/_ref/libembcomm_ref.so).  It exists so Python tests, the parity
// checker in __graft_entry__.smoke() and bench.py's reference arm can call the
// reference's own functions.  Nothing here is reachable from the product
// library (paper_2411_01611_b200/csrc); the product must never link it.
//
// Each wrapper names the reference function it forwards to (file:line into
// /root/reference/proj).  Exceptions never cross the ABI: ValidationError maps
// to 2, InvariantError to 3 (core/include/embcomm/error.hpp:10-19, CLI
// exit-code convention tools/src/main.cpp:220-229), anything else to 4.

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <exception>
#include <optional>
#include <string>
#include <thread>
#include <vector>

#include "embcomm/cache_planner.hpp"
#include "embcomm/cost_model.hpp"
#include "embcomm/distribution.hpp"
#include "embcomm/distribution_spec.hpp"
#include "embcomm/error.hpp"
#include "embcomm/rng.hpp"
#include "embcomm/simulator.hpp"
#include "embcomm/trace.hpp"

using namespace embcomm;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const ValidationError& e) {
    g_err = e.what();
    return 2;
  } catch (const InvariantError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

struct RefSim {
  double unique_mean, unique_se, nc_mean, nc_se;
  double index_cost, embedding_cost, total, hot_batch_fraction;
};

void fill(RefSim* out, const SimResult& r) {
  out->unique_mean = r.unique_per_batch.mean;
  out->unique_se = r.unique_per_batch.std_error;
  out->nc_mean = r.non_cached_unique.mean;
  out->nc_se = r.non_cached_unique.std_error;
  out->index_cost = r.measured_epoch_cost.index_cost;
  out->embedding_cost = r.measured_epoch_cost.embedding_cost;
  out->total = r.measured_epoch_cost.total;
  out->hot_batch_fraction = r.hot_batch_fraction;
}

void fill_cost(double* out3, const CostBreakdown& c) {
  out3[0] = c.index_cost;
  out3[1] = c.embedding_cost;
  out3[2] = c.total;
}

DistributionKind kind_of(int k) {
  switch (k) {
    case 0: return DistributionKind::zipf;
    case 1: return DistributionKind::exponential;
    case 2: return DistributionKind::half_normal;
    default: return DistributionKind::empirical;
  }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// --- distributions (core/src/distribution.cpp:13-104, distribution_spec.cpp:195-226)
int ref_dist_parametric(int kind, uint64_t size, double shape, void** out) {
  return guard([&] {
    *out = new EmbeddingDistribution(
        materialize(DistributionSpec::parametric(kind_of(kind), size, shape)));
  });
}
int ref_dist_extended(int kind, uint64_t size, double shape, int64_t factor, void** out) {
  return guard([&] {
    *out = new EmbeddingDistribution(materialize_extended(
        DistributionSpec::parametric(kind_of(kind), size, shape), factor));
  });
}
int ref_dist_from_probs(const double* p, uint64_t n, void** out) {
  return guard([&] {
    *out = new EmbeddingDistribution(
        EmbeddingDistribution::from_probabilities(std::vector<double>(p, p + n)));
  });
}
int ref_dist_uniform(uint64_t n, void** out) {
  return guard([&] { *out = new EmbeddingDistribution(EmbeddingDistribution::uniform(n)); });
}
void ref_dist_free(void* h) { delete static_cast<EmbeddingDistribution*>(h); }
uint64_t ref_dist_size(void* h) { return static_cast<EmbeddingDistribution*>(h)->size(); }
// ranked probabilities and the rank -> id map
void ref_dist_export(void* h, double* ranked_probs, uint32_t* rank_to_id) {
  auto* d = static_cast<EmbeddingDistribution*>(h);
  const auto p = d->ranked_probs();
  for (std::size_t r = 0; r < p.size(); ++r) {
    if (ranked_probs) ranked_probs[r] = p[r];
    if (rank_to_id) rank_to_id[r] = d->id_at_rank(r);
  }
}
int ref_dist_top_ids(void* h, uint64_t k, uint32_t* out) {
  return guard([&] {
    const auto v = static_cast<EmbeddingDistribution*>(h)->top_ids(k);
    std::memcpy(out, v.data(), v.size() * sizeof(uint32_t));
  });
}
int ref_dist_mass_of(void* h, const uint32_t* ids, uint64_t n, double* out) {
  return guard([&] {
    *out = static_cast<EmbeddingDistribution*>(h)->mass_of({ids, n});
  });
}

// --- sampler (core/src/simulator.cpp:110-143; rng core/include/embcomm/rng.hpp:12-41)
int ref_sample_batch(void* h, int64_t b, int64_t d, uint64_t rng_seed, uint32_t* out) {
  return guard([&] {
    SplitMix64 rng(rng_seed);
    const auto v = sample_batch(*static_cast<EmbeddingDistribution*>(h), b, d, rng);
    std::memcpy(out, v.data(), v.size() * sizeof(uint32_t));
  });
}
uint64_t ref_substream_seed(uint64_t master, uint64_t index) {
  return substream_seed(master, index);
}

// --- simulator (core/src/simulator.cpp:145-273)
int ref_measure_unique(void* h, int64_t b, int64_t trials, uint64_t seed, RefSim* out) {
  return guard([&] {
    fill(out, measure_unique(*static_cast<EmbeddingDistribution*>(h), b, trials, seed));
  });
}
int ref_simulate_epoch(void* h, int64_t q, int64_t b, int64_t d, const uint32_t* cache,
                       uint64_t k, int64_t epochs, uint64_t seed, RefSim* out) {
  return guard([&] {
    fill(out, simulate_epoch(*static_cast<EmbeddingDistribution*>(h), WorkloadSpec(q, b, d),
                             {cache, k}, epochs, seed));
  });
}
int ref_simulate_trace(const uint32_t* ids, uint64_t n_samples, int64_t d, uint64_t vocab,
                       int64_t b, const uint32_t* cache, uint64_t k, RefSim* out) {
  return guard([&] {
    Trace t;
    t.num_features = d;
    t.vocab_size = vocab;
    t.ids.assign(ids, ids + n_samples * static_cast<uint64_t>(d));
    fill(out, simulate_epoch(t, b, {cache, k}));
  });
}

// Many independent (table, batch) dedup+hit/miss counts, the SURVEY §8(c) M1
// protocol: segment j is replayed as a one-column trace of n_j lookups with
// batch size n_j through simulate_epoch(Trace, …) (simulator.cpp:222-273);
// its measured embedding_cost is the non-cached distinct count and
// unique_per_batch.mean the distinct count.  `threads` > 1 runs segments in
// parallel (the reference's functions are pure).
int ref_segment_counts(const uint32_t* ids, const uint64_t* seg_off, uint64_t n_seg,
                       const uint64_t* seg_vocab, const uint32_t* const* seg_cache,
                       const uint64_t* seg_cache_len, int threads, int64_t* out_all,
                       int64_t* out_nc) {
  return guard([&] {
    std::vector<std::exception_ptr> errs(n_seg);
    auto work = [&](uint64_t lo, uint64_t hi) {
      for (uint64_t j = lo; j < hi; ++j) {
        try {
          const uint64_t n = seg_off[j + 1] - seg_off[j];
          if (n == 0) {
            if (out_all) out_all[j] = 0;
            out_nc[j] = 0;
            continue;
          }
          Trace t;
          t.num_features = 1;
          t.vocab_size = seg_vocab[j];
          t.ids.assign(ids + seg_off[j], ids + seg_off[j + 1]);
          const auto r = simulate_epoch(t, static_cast<int64_t>(n),
                                        {seg_cache[j], seg_cache_len[j]});
          out_nc[j] = static_cast<int64_t>(r.measured_epoch_cost.embedding_cost);
          // With a non-empty cache the schedule splits the segment into a hot
          // and a normal batch, neither full, so unique_per_batch stays 0; the
          // distinct count then needs a second, cache-free replay.
          if (seg_cache_len[j] == 0) {
            if (out_all) out_all[j] = static_cast<int64_t>(r.unique_per_batch.mean);
          } else if (out_all) {
            const auto r0 = simulate_epoch(t, static_cast<int64_t>(n), {});
            out_all[j] = static_cast<int64_t>(r0.unique_per_batch.mean);
          }
        } catch (...) {
          errs[j] = std::current_exception();
        }
      }
    };
    if (threads <= 1 || n_seg <= 1) {
      work(0, n_seg);
    } else {
      std::vector<std::thread> pool;
      const uint64_t nt = std::min<uint64_t>(threads, n_seg);
      for (uint64_t w = 0; w < nt; ++w) {
        pool.emplace_back([&, w] {
          for (uint64_t j = w; j < n_seg; j += nt) work(j, j + 1);
        });
      }
      for (auto& th : pool) th.join();
    }
    for (auto& e : errs)
      if (e) std::rethrow_exception(e);
  });
}

// --- cost model (core/src/cost_model.cpp:36-111)
int ref_batch_presence_prob(double p, int64_t b, double* out) {
  return guard([&] { *out = batch_presence_prob(p, b); });
}
int ref_expected_unique_from_rank(void* h, int64_t b, uint64_t first, double* out) {
  return guard([&] {
    *out = expected_unique_from_rank(*static_cast<EmbeddingDistribution*>(h), b, first);
  });
}
int ref_coalesced_batch_cost(void* h, int64_t b, double* out3) {
  return guard([&] { fill_cost(out3, coalesced_batch_cost(*static_cast<EmbeddingDistribution*>(h), b)); });
}
int ref_baseline_epoch_cost(int64_t q, int64_t b, int64_t d, double* out) {
  return guard([&] { *out = baseline_epoch_cost(WorkloadSpec(q, b, d)); });
}
int ref_coalesced_epoch_cost(void* h, int64_t q, int64_t b, int64_t d, double* out3) {
  return guard([&] {
    fill_cost(out3, coalesced_epoch_cost(*static_cast<EmbeddingDistribution*>(h), WorkloadSpec(q, b, d)));
  });
}
int ref_cached_epoch_cost(void* h, int64_t q, int64_t b, int64_t d, const uint32_t* cache,
                          uint64_t k, double* out3) {
  return guard([&] {
    fill_cost(out3, cached_epoch_cost(*static_cast<EmbeddingDistribution*>(h),
                                      WorkloadSpec(q, b, d), {cache, k}));
  });
}

// --- planner (core/src/cache_planner.cpp:114-294)
int ref_max_batch_size(int64_t m, int64_t a, int64_t d_emb, double eff, int64_t k,
                       int64_t* out) {
  return guard([&] {
    const auto b = max_batch_size(DeviceModel(m, a, d_emb, eff), k);
    *out = b ? *b : -1;
  });
}
// plan_out: [cache_size, batch_size, feasible, used_scan_fallback]; cost3; ids (cap E)
int ref_plan(void* h, int64_t m, int64_t a, int64_t d_emb, double eff, int64_t q, int64_t d,
             int search, int64_t* plan_out, double* cost3, uint32_t* ids) {
  return guard([&] {
    const auto& dist = *static_cast<EmbeddingDistribution*>(h);
    const DeviceModel dev(m, a, d_emb, eff);
    const WorkloadSpec spec(q, 1, d);
    const CachePlan p = search ? optimal_cache_size_search(dist, dev, spec)
                               : optimal_cache_size_scan(dist, dev, spec);
    plan_out[0] = static_cast<int64_t>(p.cache_size);
    plan_out[1] = p.batch_size;
    plan_out[2] = p.feasible;
    plan_out[3] = p.used_scan_fallback;
    fill_cost(cost3, p.expected_epoch_cost);
    if (ids) std::memcpy(ids, p.cached_ids.data(), p.cached_ids.size() * sizeof(uint32_t));
  });
}
// out: [candidate_id, presence_gain, threshold, delta_comm, recommend]
int ref_delta_comm(void* h, int64_t m, int64_t a, int64_t d_emb, double eff, int64_t q,
                   int64_t k, double* out5) {
  return guard([&] {
    const auto r = delta_comm(*static_cast<EmbeddingDistribution*>(h),
                              DeviceModel(m, a, d_emb, eff), q, k);
    out5[0] = r.candidate_id;
    out5[1] = r.presence_gain;
    out5[2] = r.threshold;
    out5[3] = r.delta_comm;
    out5[4] = r.recommend;
  });
}
int ref_memory_io_proxy(void* h, int64_t q, int64_t b, int64_t d, const uint32_t* cache,
                        uint64_t k, double* out) {
  return guard([&] {
    *out = memory_io_proxy(*static_cast<EmbeddingDistribution*>(h), WorkloadSpec(q, b, d),
                           {cache, k});
  });
}

// --- traces (core/src/trace.cpp:51-240)
// parse_trace of a text file: *d, *vocab, *n_ids; ids copied when cap allows
int ref_load_trace(const char* path, int64_t* d, uint64_t* vocab, uint32_t* ids, uint64_t cap, uint64_t* n_ids) {
  return guard([&] {
    const Trace t = load_trace(path);
    *d = t.num_features;
    *vocab = t.vocab_size;
    *n_ids = t.ids.size();
    if (ids && cap >= t.ids.size()) std::copy(t.ids.begin(), t.ids.end(), ids);
  });
}

// entries out: ids, counts, cum (cap = vocab); returns number of entries in *n_out
int ref_build_skew_table(const uint32_t* ids, uint64_t n_samples, int64_t d, uint64_t vocab,
                         uint32_t* out_ids, uint64_t* out_counts, double* out_cum,
                         uint64_t* n_out) {
  return guard([&] {
    Trace t;
    t.num_features = d;
    t.vocab_size = vocab;
    t.ids.assign(ids, ids + n_samples * static_cast<uint64_t>(d));
    const SkewTable s = build_skew_table(t);
    *n_out = s.entries.size();
    for (std::size_t i = 0; i < s.entries.size(); ++i) {
      out_ids[i] = s.entries[i].id;
      out_counts[i] = s.entries[i].count;
      out_cum[i] = s.entries[i].cum_fraction;
    }
  });
}
int ref_estimate_distribution(const uint32_t* ids, uint64_t n_samples, int64_t d,
                              uint64_t vocab, double smoothing, void** out) {
  return guard([&] {
    Trace t;
    t.num_features = d;
    t.vocab_size = vocab;
    t.ids.assign(ids, ids + n_samples * static_cast<uint64_t>(d));
    *out = new EmbeddingDistribution(estimate_distribution(build_skew_table(t), vocab, smoothing));
  });
}
// hot flags per sample (1 = hot)
int ref_classify_samples(const uint32_t* ids, uint64_t n_samples, int64_t d, uint64_t vocab,
                         const uint32_t* cache, uint64_t k, uint8_t* hot) {
  return guard([&] {
    Trace t;
    t.num_features = d;
    t.vocab_size = vocab;
    t.ids.assign(ids, ids + n_samples * static_cast<uint64_t>(d));
    const auto c = classify_samples(t, {cache, k});
    std::memset(hot, 0, n_samples);
    for (auto s : c.hot) hot[s] = 1;
  });
}
// schedule as a flat sample order (hot batches first) + batch sizes; shuffle<0: none
int ref_build_schedule(const uint32_t* ids, uint64_t n_samples, int64_t d, uint64_t vocab,
                       const uint32_t* cache, uint64_t k, int64_t b, int64_t shuffle_seed,
                       uint32_t* order, uint64_t* batch_sizes, uint64_t* n_hot_batches,
                       uint64_t* n_batches) {
  return guard([&] {
    Trace t;
    t.num_features = d;
    t.vocab_size = vocab;
    t.ids.assign(ids, ids + n_samples * static_cast<uint64_t>(d));
    std::optional<uint64_t> seed;
    if (shuffle_seed >= 0) seed = static_cast<uint64_t>(shuffle_seed);
    const auto s = build_schedule(t, {cache, k}, b, seed);
    uint64_t pos = 0, nb = 0;
    for (const auto* group : {&s.hot_batches, &s.normal_batches})
      for (const auto& batch : *group) {
        for (auto x : batch) order[pos++] = x;
        batch_sizes[nb++] = batch.size();
      }
    *n_hot_batches = s.hot_batches.size();
    *n_batches = nb;
  });
}

}  // extern "C"
