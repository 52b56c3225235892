// C++ callers of the reference API, relinked against libembcomm_gpu.so through
// include/embcomm_gpu.hpp.  Cases mirror the reference's own unit tests
// (tests/test_cost_model.cpp, test_simulator.cpp, test_cache_planner.cpp);
// GPU cases need a device.  Exit code 0 = all checks passed.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "embcomm_gpu.hpp"

using namespace embcomm;

static int failures = 0;
#define CHECK(c)                                                    \
  do {                                                              \
    if (!(c)) {                                                     \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);      \
      ++failures;                                                   \
    }                                                               \
  } while (0)
#define CHECK_THROWS_AS(expr, E) \
  do {                           \
    bool t = false;              \
    try {                        \
      (void)(expr);              \
    } catch (const E&) {         \
      t = true;                  \
    }                            \
    CHECK(t);                    \
  } while (0)

static void host_cases() {
  CHECK(batch_presence_prob(0.0, 100) == 0.0);
  CHECK(batch_presence_prob(1.0, 1) == 1.0);
  CHECK(std::abs(batch_presence_prob(0.5, 2) - 0.75) < 1e-12);
  CHECK_THROWS_AS(batch_presence_prob(-0.1, 1), ValidationError);
  const auto u4 = EmbeddingDistribution::uniform(4);
  CHECK(std::abs(expected_unique_per_batch(u4, 2) - 1.75) < 1e-12);
  CHECK(baseline_epoch_cost(WorkloadSpec(5000, 256, 26)) == 130000.0);
  const std::vector<std::uint32_t> one{0};
  CHECK(std::abs(cached_epoch_cost(u4, WorkloadSpec(40, 4, 1), one).total - 60.5078125) < 1e-9);
  CHECK_THROWS_AS(WorkloadSpec(10, 11, 1), ValidationError);
  const auto d = EmbeddingDistribution::from_probabilities({0.2, 0.4, 0.2, 0.2});
  CHECK(d.id_at_rank(0) == 1 && d.id_at_rank(1) == 0);
  const auto z32 = materialize_parametric(DistributionKind::zipf, 32, 1.0);
  const auto plan = optimal_cache_size_scan(z32, DeviceModel(2048, 2, 8), WorkloadSpec(10000, 1, 4));
  CHECK(plan.cache_size == 32 && plan.batch_size == 896 && plan.feasible);
  CHECK(*max_batch_size(DeviceModel(1000, 10, 5, 0.5), 12) == 44);
}

static void gpu_cases() {
  // tests/test_simulator.cpp:156-172 known answer
  Trace t;
  t.num_features = 2;
  t.vocab_size = 4;
  t.ids = {0, 1, 0, 2, 1, 1, 3, 3};
  const std::vector<std::uint32_t> cache{0, 1};
  const auto r = simulate_epoch(t, 2, cache);
  CHECK(r.measured_epoch_cost.index_cost == 4.0);
  CHECK(r.measured_epoch_cost.embedding_cost == 3.0);
  CHECK(r.hot_batch_fraction == 0.5);
  // full cache leaves only index traffic (test_simulator.cpp:89-96)
  const auto z16 = materialize_parametric(DistributionKind::zipf, 16, 1.0);
  const auto r2 = simulate_epoch(z16, WorkloadSpec(100, 10, 2), z16.top_ids(16), 3, 1);
  CHECK(r2.measured_epoch_cost.embedding_cost == 0.0 && r2.hot_batch_fraction == 1.0);
  // substream replay == measure_unique mean (test_simulator.cpp:66-85)
  const auto z32 = materialize_parametric(DistributionKind::zipf, 32, 1.0);
  const auto mu = measure_unique(z32, 16, 4, 1234);
  double total = 0.0;
  for (std::uint64_t k = 0; k < 4; ++k) {
    SplitMix64 rng(substream_seed(1234, k));
    const auto ids = sample_batch(z32, 16, 1, rng);
    std::vector<bool> seen(32, false);
    for (auto id : ids)
      if (!seen[id]) seen[id] = true, total += 1.0;
  }
  CHECK(mu.unique_per_batch.mean == total / 4.0);
}

int main(int argc, char** argv) {
  host_cases();
  if (argc > 1 && std::string(argv[1]) == "--gpu") gpu_cases();
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
