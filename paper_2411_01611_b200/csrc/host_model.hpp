// Host model types shared by the C-ABI translation units.
#pragma once

#include <cstdint>
#include <optional>
#include <string>
#include <vector>

#include "embcomm_gpu.h"

namespace ec {

// EmbeddingDistribution (core/include/embcomm/distribution.hpp:19-49).
struct Dist {
  std::vector<double> ranked;       // probabilities, non-increasing
  std::vector<uint32_t> rank_to_id;
  std::vector<uint32_t> id_to_rank;

  static Dist from_probabilities(std::vector<double> p);
  static Dist parametric(int kind, uint64_t count, double shape, double rank_scale);
  size_t size() const { return ranked.size(); }
  void check_id(uint32_t id) const;
  void check_rank(uint64_t r) const;
};

struct Plan {
  ec_cache_plan head{};  // feasible = 0 when default-constructed
  int64_t k = 0;
};

const char* last_error();
const Dist& dist_of(ec_dist h);
ec_dist make_dist(Dist&& d);

double presence(double p, int64_t b);
double unique_from_rank(const Dist& d, int64_t b, uint64_t first);
void validate(const ec_workload& w);
void validate(const ec_device_model& m);
std::optional<int64_t> batch_fit(const ec_device_model& m, int64_t k);
ec_cost cached_cost(const Dist& d, const ec_workload& w, const uint32_t* cache, uint64_t k);
Plan plan_scan(const Dist& d, const ec_device_model& m, const ec_workload& w);
Plan plan_search(const Dist& d, const ec_device_model& m, const ec_workload& w);
ec_marginal marginal(const Dist& d, const ec_device_model& m, int64_t q, int64_t k);

}  // namespace ec
