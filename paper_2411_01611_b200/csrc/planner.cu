// GPU planner sweeps.
//
// The planner's unit of work is expected_unique_from_rank(dist, b, k)
// (core/src/cost_model.cpp:48-59): an O(E) sum of presence terms
// 1-(1-p)^b = -expm1(b*log1p(-p)) over the ranks >= k.  The host restatement
// (host_model.cpp) keeps the reference's sequential order and is bit-exact;
// this file evaluates MANY (b, k) pairs at once on the GPU — fp64 terms,
// block tree sums, one fp64 atomic per block — for dense cost curves and
// sweeps.  Summation order differs from the reference, so results agree to
// ~1e-12 relative, not bitwise; the bit-exact planner remains
// ec_optimal_cache_size_search.
#include <algorithm>
#include <cmath>
#include <vector>

#include "common.hpp"
#include "device_util.cuh"
#include "host_model.hpp"

namespace ec {
namespace {

constexpr int kPThreads = 256;
constexpr int kPItems = 16;  // ranks per thread per block

// cost_model.cpp:36-46 on the device (exact at b == 1 and p == 1)
__device__ __forceinline__ double presence_d(double p, int64_t b) {
  if (b == 1) return p;
  if (p == 1.0) return 1.0;
  return -expm1(static_cast<double>(b) * log1p(-p));
}

// sums[j] += sum over ranks r >= first[j] of presence(ranked[r], b[j]);
// blockIdx.y = j, blockIdx.x = chunk of kPThreads*kPItems ranks.
__global__ void __launch_bounds__(kPThreads) k_presence_sums(const double* __restrict__ ranked, uint64_t E,
                                                            const int64_t* __restrict__ b,
                                                            const uint64_t* __restrict__ first,
                                                            double* __restrict__ sums) {
  const int j = blockIdx.y;
  const uint64_t r0 = static_cast<uint64_t>(blockIdx.x) * kPThreads * kPItems;
  const uint64_t lo = max(r0, first[j]);
  const int64_t bj = b[j];
  double acc = 0.0;
#pragma unroll 4
  for (int i = 0; i < kPItems; ++i) {
    const uint64_t r = r0 + static_cast<uint64_t>(i) * kPThreads + threadIdx.x;
    if (r < E && r >= lo) acc += presence_d(__ldg(ranked + r), bj);
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
  __shared__ double w[kPThreads / 32];
  if (lane_id() == 0) w[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < kPThreads / 32; ++k) t += w[k];
    if (t != 0.0) atomicAdd(sums + j, t);
  }
}

// Evaluate the presence sums of n (b, first) pairs (chunks of <= 65535).
void presence_sums(const Dist& d, const std::vector<int64_t>& b, const std::vector<uint64_t>& first, int device,
                   std::vector<double>& out) {
  use_device(device);
  const uint64_t E = d.size();
  const size_t n = b.size();
  out.assign(n, 0.0);
  if (!n) return;
  cudaStream_t st;
  EC_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  try {
    DevBuf<double> dp(E), ds(n);
    DevBuf<int64_t> db(n);
    DevBuf<uint64_t> df(n);
    EC_CUDA(cudaMemcpyAsync(dp.p, d.ranked.data(), E * sizeof(double), cudaMemcpyHostToDevice, st));
    EC_CUDA(cudaMemcpyAsync(db.p, b.data(), n * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    EC_CUDA(cudaMemcpyAsync(df.p, first.data(), n * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
    EC_CUDA(cudaMemsetAsync(ds.p, 0, n * sizeof(double), st));
    const uint64_t chunks = (E + kPThreads * kPItems - 1) / (kPThreads * kPItems);
    for (size_t j0 = 0; j0 < n; j0 += 65535) {
      const unsigned ny = static_cast<unsigned>(std::min<size_t>(65535, n - j0));
      k_presence_sums<<<dim3(static_cast<unsigned>(chunks), ny), kPThreads, 0, st>>>(dp.p, E, db.p + j0, df.p + j0,
                                                                                      ds.p + j0);
      EC_LAUNCH();
    }
    EC_CUDA(cudaMemcpyAsync(out.data(), ds.p, n * sizeof(double), cudaMemcpyDeviceToHost, st));
    EC_CUDA(cudaStreamSynchronize(st));
  } catch (...) {
    cudaStreamDestroy(st);
    throw;
  }
  cudaStreamDestroy(st);
}

}  // namespace
}  // namespace ec

using namespace ec;

extern "C" {

int ec_expected_unique_many(ec_dist h, const int64_t* batch_sizes, const uint64_t* first_ranks, uint64_t n,
                            int device, double* out) {
  return guard([&] {
    const Dist& d = dist_of(h);
    std::vector<int64_t> b(batch_sizes, batch_sizes + n);
    std::vector<uint64_t> f(n, 0);
    for (uint64_t i = 0; i < n; ++i) {
      if (b[i] < 1) invalid("presence probability needs b >= 1");
      if (first_ranks) {
        if (first_ranks[i] > d.size()) invalid("rank offset " + std::to_string(first_ranks[i]) + " out of range");
        f[i] = first_ranks[i];
      }
    }
    std::vector<double> s;
    presence_sums(d, b, f, device, s);
    std::copy(s.begin(), s.end(), out);
  });
}

// Cached epoch cost of the top-k prefix at the memory-derived batch size,
// for every k in ks (cache_planner.cpp:24-53 cost_at); infeasible k get
// batch -1 and NaN costs.
int ec_cost_curve(ec_dist h, const ec_device_model* m, const ec_workload* w, const int64_t* ks, uint64_t n,
                  int device, ec_cost* out, int64_t* batch_out) {
  return guard([&] {
    const Dist& d = dist_of(h);
    validate(*m);
    if (w->num_samples < 1) invalid("dataset size must be >= 1");
    if (w->lookups_per_sample < 1) invalid("lookups per sample must be >= 1");
    std::vector<int64_t> b;
    std::vector<uint64_t> f;
    std::vector<uint64_t> idx;
    for (uint64_t i = 0; i < n; ++i) {
      if (ks[i] < 0 || static_cast<uint64_t>(ks[i]) > d.size()) invalid("cache size out of [0, E]");
      const auto bb = batch_fit(*m, ks[i]);
      if (!bb) {
        batch_out[i] = -1;
        out[i] = ec_cost{NAN, NAN, NAN};
        continue;
      }
      batch_out[i] = std::min(*bb, w->num_samples);
      b.push_back(batch_out[i]);
      f.push_back(static_cast<uint64_t>(ks[i]));
      idx.push_back(i);
    }
    std::vector<double> s;
    presence_sums(d, b, f, device, s);
    for (size_t j = 0; j < idx.size(); ++j) {
      const double q = static_cast<double>(w->num_samples);
      const double emb = (q / static_cast<double>(b[j])) * s[j] * static_cast<double>(w->lookups_per_sample);
      out[idx[j]] = ec_cost{q, emb, q + emb};
    }
  });
}

}  // extern "C"
