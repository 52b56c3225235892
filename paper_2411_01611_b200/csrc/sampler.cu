// K0 (synthetic id generator) and the GPU Monte Carlo simulator.
//
// K0 restates DiscreteSampler (core/src/simulator.cpp:110-130) over the
// SplitMix64 stream (core/include/embcomm/rng.hpp:16-24) as a closed form:
// draw m of a generator seeded with s is mix64(s + (m+1)*golden), so every
// draw is independent and the device generates exactly the reference's ids.
// The CDF is built on the host in the reference's Kahan order (fp64 compares
// on the device are exact).  A 4096-entry guide table of the CDF sits in
// shared memory: the smem search narrows the range to ceil(E/4096) entries,
// so a draw costs ~log2(E/4096) dependent global loads instead of log2(E).
//
// The simulator counts distinct and non-cached distinct ids per
// (batch, feature column) on the device (count_batch_unique,
// simulator.cpp:85-106, as a hash-set insert per id with warp match-any
// collapse) and folds the integer counts on the host in the reference's
// fixed order (StatAccumulator, simulator.cpp:39-63), so every SimResult
// field is bit-identical.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "common.hpp"
#include "device_util.cuh"
#include "host_model.hpp"
#include "scan.cuh"

namespace ec {

constexpr int kGuide = 4096;

struct SamplerDev {
  const double* cdf;
  const uint32_t* rank_to_id;  // nullptr: identity (parametric kinds are pre-sorted)
  const double* guide;
  uint64_t E;
  uint64_t stride;  // guide[j] = cdf[j*stride]
  uint32_t guide_n;
};

__device__ __forceinline__ double unit_draw(uint64_t seed, uint64_t m) {
  return static_cast<double>(mix64(seed + (m + 1) * kGolden) >> 11) * 0x1.0p-53;
}

// upper_bound(cdf, u), clamped to the last rank, mapped rank -> id.
__device__ __forceinline__ uint32_t draw_id(const SamplerDev& s, const double* g, double u) {
  uint32_t lo = 0, hi = s.guide_n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (g[mid] > u) hi = mid; else lo = mid + 1;
  }
  uint64_t a = lo == 0 ? 0 : (static_cast<uint64_t>(lo) - 1) * s.stride + 1;
  uint64_t b = lo < s.guide_n ? static_cast<uint64_t>(lo) * s.stride : s.E;
  while (a < b) {
    const uint64_t mid = (a + b) >> 1;
    if (__ldg(s.cdf + mid) > u) b = mid; else a = mid + 1;
  }
  if (a == s.E) a = s.E - 1;
  return s.rank_to_id ? __ldg(s.rank_to_id + a) : static_cast<uint32_t>(a);
}

__device__ __forceinline__ void load_guide(const SamplerDev& s, double* g) {
  for (uint32_t j = threadIdx.x; j < s.guide_n; j += blockDim.x) g[j] = s.guide[j];
  __syncthreads();
}

// Draws #start.. of one stream.
__global__ void k_sample_stream(SamplerDev s, uint64_t seed, uint64_t start, uint64_t count,
                                uint32_t* __restrict__ out) {
  __shared__ double g[kGuide];
  load_guide(s, g);
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = draw_id(s, g, unit_draw(seed, start + i));
}

// measure_unique trials t0..: trial t draws `b` ids from substream(master, t)
// (simulator.cpp:153-159).
__global__ void k_sample_trials(SamplerDev s, uint64_t master, uint64_t t0, uint64_t b,
                                uint64_t count, uint32_t* __restrict__ out) {
  __shared__ double g[kGuide];
  load_guide(s, g);
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t t = i / b;
    out[i] = draw_id(s, g, unit_draw(substream(master, t0 + t), i - t * b));
  }
}

// simulate_epoch batches: the epoch stream is consumed sample-major
// (simulator.cpp:191-192); draw m belongs to batch m/(b*d), sample (m%(b*d))/d,
// column m%d.  Written column-major per batch so each (batch, column) is a
// contiguous segment.  m0 is a batch boundary; the last batch may be short.
__global__ void k_sample_epoch(SamplerDev s, uint64_t seed, uint64_t q, uint64_t b, uint64_t d,
                               uint64_t m0, uint64_t count, uint32_t* __restrict__ out) {
  __shared__ double g[kGuide];
  load_guide(s, g);
  const uint64_t bd = b * d;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t m = m0 + i;
    const uint64_t jb = m / bd;
    const uint64_t bi = min(b, q - jb * b);
    const uint64_t r = m - jb * bd;
    const uint64_t smp = r / d, f = r - smp * d;
    out[(i - r) + f * bi + smp] = draw_id(s, g, unit_draw(seed, m));
  }
}

// Distinct / non-cached distinct count per segment.  Batch j covers elements
// [boff[j], boff[j+1]) laid out column-major (d columns of bi = size/d);
// segment g = j*d + f owns hash keys[g*cap, (g+1)*cap), cap = 2^(32-shift).
__global__ void k_count_segments(const uint32_t* __restrict__ ids, uint64_t n,
                                 const uint64_t* __restrict__ boff, uint32_t nb, uint32_t d,
                                 uint32_t* __restrict__ keys, uint32_t shift,
                                 const uint8_t* __restrict__ cached, int* __restrict__ cnt_all,
                                 int* __restrict__ cnt_nc) {
  const uint64_t cap = 1ull << (32 - shift);
  for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x; base < n;
       base += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t p = base + threadIdx.x;
    const bool live = p < n;
    uint64_t gseg = ~0ull;
    uint32_t id = 0;
    if (live) {
      uint32_t lo = 0, hi = nb;  // batch: last j with boff[j] <= p
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (boff[mid] <= p) lo = mid; else hi = mid;
      }
      const uint64_t bi = (boff[lo + 1] - boff[lo]) / d;
      gseg = static_cast<uint64_t>(lo) * d + (p - boff[lo]) / bi;
      id = ids[p];
    }
    // collapse equal (segment, id) lanes; the leader inserts
    const unsigned long long key = (gseg << 32) | id;
    const unsigned peers = __match_any_sync(kFull, key);
    const bool leader = live && (__ffs(peers) - 1) == lane_id();
    bool fresh = false;
    if (leader) {
      uint32_t* tab = keys + gseg * cap;
      uint32_t h = hash_slot(id, shift);
      for (;;) {
        uint32_t cur = tab[h];
        if (cur == kEmptyKey) {
          cur = atomicCAS(tab + h, kEmptyKey, id);
          if (cur == kEmptyKey) { fresh = true; break; }
        }
        if (cur == id) break;
        h = (h + 1) & static_cast<uint32_t>(cap - 1);
      }
    }
    const bool nc = fresh && !(cached && cached[id]);
    const unsigned seg_peers = __match_any_sync(kFull, gseg);
    const int na = group_count(seg_peers, fresh), nn = group_count(seg_peers, nc);
    if (live && (__ffs(seg_peers) - 1) == lane_id()) {
      if (na) atomicAdd(cnt_all + gseg, na);
      if (nn) atomicAdd(cnt_nc + gseg, nn);
    }
  }
}

// classify_samples (core/src/trace.cpp:185-204): hot iff all d ids cached.
__global__ void k_classify(const uint32_t* __restrict__ ids, uint64_t q, uint32_t d, uint64_t vocab,
                           const uint8_t* __restrict__ cached, int* __restrict__ hot,
                           int* __restrict__ bad) {
  for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < q;
       s += (uint64_t)gridDim.x * blockDim.x) {
    int h = 1;
    for (uint32_t f = 0; f < d; ++f) {
      const uint32_t id = ids[s * d + f];
      if (id >= vocab) { atomicExch(bad, 1); h = 0; break; }
      h &= cached ? cached[id] : 0;
    }
    hot[s] = h;
  }
}

// build_schedule order (trace.cpp:206-240, no shuffle): stable partition,
// hot samples first.
__global__ void k_partition_order(const int* __restrict__ hot, const int* __restrict__ excl,
                                  const int* __restrict__ n_hot, uint64_t q,
                                  uint32_t* __restrict__ order) {
  const int H = *n_hot;
  for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < q;
       s += (uint64_t)gridDim.x * blockDim.x) {
    const int e = excl[s];
    order[hot[s] ? e : H + static_cast<int>(s) - e] = static_cast<uint32_t>(s);
  }
}

// Replay layout: batch j = schedule positions [p0_j, p0_j + bi), written
// column-major at element offset boff[j].
__global__ void k_gather_schedule(const uint32_t* __restrict__ ids, const uint32_t* __restrict__ order,
                                  const uint64_t* __restrict__ boff, const uint64_t* __restrict__ pos0,
                                  uint32_t nb, uint32_t d, uint64_t n, uint32_t* __restrict__ out) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n;
       e += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t lo = 0, hi = nb;
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (boff[mid] <= e) lo = mid; else hi = mid;
    }
    const uint64_t bi = (boff[lo + 1] - boff[lo]) / d;
    const uint64_t r = e - boff[lo];
    const uint64_t f = r / bi, k = r - f * bi;
    out[e] = ids[static_cast<uint64_t>(order[pos0[lo] + k]) * d + f];
  }
}

// ------------------------------------------------------------ host side
static int grid_for(uint64_t n, int device, int threads = 256) {
  const uint64_t want = (n + threads - 1) / threads;
  const uint64_t cap = static_cast<uint64_t>(sm_count(device)) * 16;
  return static_cast<int>(std::max<uint64_t>(1, std::min(want, cap)));
}

static uint32_t log2_ceil(uint64_t x) {
  uint32_t l = 0;
  while ((1ull << l) < x) ++l;
  return l;
}

// Host-side fixed-order accumulation (StatAccumulator, simulator.cpp:39-63).
struct Stat {
  uint64_t n = 0;
  double s = 0.0, sq = 0.0;
  void add(double x) { ++n; s += x; sq += x * x; }
  void finish(double* mean, double* se) const {
    *mean = 0.0;
    *se = 0.0;
    if (!n) return;
    const double dn = static_cast<double>(n);
    *mean = s / dn;
    if (n > 1) *se = std::sqrt(std::max(0.0, (sq - dn * *mean * *mean) / (dn - 1.0)) / dn);
  }
};

// Device workspace for segment counting, grown on demand.
struct CountWork {
  DevBuf<uint32_t> ids, keys;
  DevBuf<int> cnt_all, cnt_nc;
  DevBuf<uint64_t> boff;
  void ensure(uint64_t n_ids, uint64_t n_keys, uint64_t n_seg, uint64_t n_batches) {
    if (ids.n < n_ids) ids.alloc(n_ids);
    if (keys.n < n_keys) keys.alloc(n_keys);
    if (cnt_all.n < n_seg) { cnt_all.alloc(n_seg); cnt_nc.alloc(n_seg); }
    if (boff.n < n_batches + 1) boff.alloc(n_batches + 1);
  }
};

// Count distinct ids per (batch, column) for batches already laid out in
// w.ids; batch sizes bi[j] (samples), d columns; returns per-segment counts.
static void count_batches(CountWork& w, int device, uint64_t n, const std::vector<uint64_t>& bsz,
                          uint32_t d, uint64_t max_bi, const uint8_t* cached_dev,
                          std::vector<int>& all, std::vector<int>& nc, cudaStream_t st) {
  const uint64_t nb = bsz.size();
  const uint32_t lg = std::max<uint32_t>(4, log2_ceil(2 * max_bi));
  const uint64_t cap = 1ull << lg;
  const uint64_t nseg = nb * d;
  w.ensure(n, nseg * cap, nseg, nb);
  std::vector<uint64_t> boff(nb + 1, 0);
  for (uint64_t j = 0; j < nb; ++j) boff[j + 1] = boff[j] + bsz[j] * d;
  EC_CUDA(cudaMemcpyAsync(w.boff.p, boff.data(), (nb + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
  EC_CUDA(cudaMemsetAsync(w.keys.p, 0xFF, nseg * cap * sizeof(uint32_t), st));
  EC_CUDA(cudaMemsetAsync(w.cnt_all.p, 0, nseg * sizeof(int), st));
  EC_CUDA(cudaMemsetAsync(w.cnt_nc.p, 0, nseg * sizeof(int), st));
  k_count_segments<<<grid_for(n, device), 256, 0, st>>>(w.ids.p, n, w.boff.p, static_cast<uint32_t>(nb), d,
                                                         w.keys.p, 32 - lg, cached_dev, w.cnt_all.p, w.cnt_nc.p);
  EC_LAUNCH();
  all.resize(nseg);
  nc.resize(nseg);
  EC_CUDA(cudaMemcpyAsync(all.data(), w.cnt_all.p, nseg * sizeof(int), cudaMemcpyDeviceToHost, st));
  EC_CUDA(cudaMemcpyAsync(nc.data(), w.cnt_nc.p, nseg * sizeof(int), cudaMemcpyDeviceToHost, st));
  EC_CUDA(cudaStreamSynchronize(st));
}

// cache_mask (simulator.cpp:65-75) uploaded as a byte mask.
static void upload_mask(DevBuf<uint8_t>& m, uint64_t vocab, const uint32_t* ids, uint64_t k,
                        cudaStream_t st) {
  std::vector<uint8_t> h(vocab, 0);
  for (uint64_t i = 0; i < k; ++i) {
    if (ids[i] >= vocab)
      invalid("cache id " + std::to_string(ids[i]) + " out of range [0, " + std::to_string(vocab) + ")");
    h[ids[i]] = 1;
  }
  m.alloc(vocab);
  EC_CUDA(cudaMemcpyAsync(m.p, h.data(), vocab, cudaMemcpyHostToDevice, st));
  EC_CUDA(cudaStreamSynchronize(st));
}

}  // namespace ec

using namespace ec;

struct ec_sampler_s {
  int device = 0;
  uint64_t E = 0;
  DevBuf<double> cdf, guide;
  DevBuf<uint32_t> r2i;
  uint64_t stride = 1;
  uint32_t guide_n = 0;
  bool identity = true;
  cudaStream_t st = nullptr;
  CountWork work;
  SamplerDev dev() const {
    return SamplerDev{cdf.p, identity ? nullptr : r2i.p, guide.p, E, stride, guide_n};
  }
  ~ec_sampler_s() {
    if (st) cudaStreamDestroy(st);
  }
};

static void launch_stream(ec_sampler s, uint64_t seed, uint64_t start, uint64_t count, uint32_t* out,
                          cudaStream_t st) {
  if (!count) return;
  k_sample_stream<<<grid_for(count, s->device), 256, 0, st>>>(s->dev(), seed, start, count, out);
  EC_LAUNCH();
}

// Per-chunk draw budget for the simulator's device workspace.
constexpr uint64_t kChunkDraws = 1ull << 24;

extern "C" {

int ec_sampler_create(ec_dist h, int device, ec_sampler* out) {
  return guard([&] {
    const Dist& d = dist_of(h);
    use_device(device);
    auto s = new ec_sampler_s;
    try {
      s->device = device;
      s->E = d.size();
      // DiscreteSampler ctor (simulator.cpp:110-123): Kahan running CDF, last = 1.0
      std::vector<double> cdf(d.size());
      double run = 0.0, carry = 0.0;
      for (size_t r = 0; r < d.size(); ++r) {
        const double y = d.ranked[r] - carry;
        const double t = run + y;
        carry = (t - run) - y;
        run = t;
        cdf[r] = run;
      }
      cdf.back() = 1.0;
      s->stride = std::max<uint64_t>(1, (s->E + kGuide - 1) / kGuide);
      s->guide_n = static_cast<uint32_t>((s->E + s->stride - 1) / s->stride);
      std::vector<double> g(s->guide_n);
      for (uint32_t j = 0; j < s->guide_n; ++j) g[j] = cdf[j * s->stride];
      s->identity = true;
      for (size_t r = 0; r < d.size() && s->identity; ++r) s->identity = d.rank_to_id[r] == r;
      EC_CUDA(cudaStreamCreateWithFlags(&s->st, cudaStreamNonBlocking));
      s->cdf.alloc(s->E);
      s->guide.alloc(s->guide_n);
      EC_CUDA(cudaMemcpy(s->cdf.p, cdf.data(), s->E * sizeof(double), cudaMemcpyHostToDevice));
      EC_CUDA(cudaMemcpy(s->guide.p, g.data(), s->guide_n * sizeof(double), cudaMemcpyHostToDevice));
      if (!s->identity) {
        s->r2i.alloc(s->E);
        EC_CUDA(cudaMemcpy(s->r2i.p, d.rank_to_id.data(), s->E * sizeof(uint32_t), cudaMemcpyHostToDevice));
      }
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
  });
}

void ec_sampler_destroy(ec_sampler s) { delete s; }

int ec_sample_stream(ec_sampler s, uint64_t seed, uint64_t start, uint64_t count, uint32_t* ids_dev,
                     void* stream) {
  return guard([&] {
    if (!s) invalid("null sampler");
    use_device(s->device);
    launch_stream(s, seed, start, count, ids_dev, as_stream(stream));
  });
}

int ec_sample_batch(ec_sampler s, int64_t b, int64_t d, uint64_t* rng_state, uint32_t* out_host) {
  return guard([&] {
    if (!s) invalid("null sampler");
    if (b < 1) invalid("batch size must be >= 1");
    if (d < 1) invalid("lookups per sample must be >= 1");
    use_device(s->device);
    const uint64_t n = static_cast<uint64_t>(b) * static_cast<uint64_t>(d);
    s->work.ensure(n, 0, 0, 0);
    launch_stream(s, *rng_state, 0, n, s->work.ids.p, s->st);
    EC_CUDA(cudaMemcpyAsync(out_host, s->work.ids.p, n * sizeof(uint32_t), cudaMemcpyDeviceToHost, s->st));
    EC_CUDA(cudaStreamSynchronize(s->st));
    *rng_state += n * kGolden;  // the generator advanced by n steps (rng.hpp:17)
  });
}

int ec_measure_unique(ec_sampler s, int64_t b, int64_t trials, uint64_t seed, ec_sim_result* out) {
  return guard([&] {
    if (!s) invalid("null sampler");
    if (b < 1) invalid("batch size must be >= 1");
    if (trials < 1) invalid("trials must be >= 1");
    use_device(s->device);
    const uint64_t per_chunk = std::max<uint64_t>(1, kChunkDraws / static_cast<uint64_t>(b));
    Stat acc;
    std::vector<int> all, nc;
    for (uint64_t t0 = 0; t0 < static_cast<uint64_t>(trials); t0 += per_chunk) {
      const uint64_t nt = std::min<uint64_t>(per_chunk, trials - t0);
      const uint64_t n = nt * b;
      s->work.ensure(n, 0, 0, 0);
      k_sample_trials<<<grid_for(n, s->device), 256, 0, s->st>>>(s->dev(), seed, t0, b, n, s->work.ids.p);
      EC_LAUNCH();
      count_batches(s->work, s->device, n, std::vector<uint64_t>(nt, b), 1, b, nullptr, all, nc, s->st);
      for (uint64_t t = 0; t < nt; ++t) acc.add(static_cast<double>(all[t]));
    }
    ec_sim_result r{};
    acc.finish(&r.unique_mean, &r.unique_std_error);
    r.non_cached_mean = r.unique_mean;  // simulator.cpp:165
    r.non_cached_std_error = r.unique_std_error;
    *out = r;
  });
}

int ec_simulate_epoch(ec_sampler s, const ec_workload* w, const uint32_t* cache, uint64_t k,
                      int64_t epochs, uint64_t seed, ec_sim_result* out) {
  return guard([&] {
    if (!s) invalid("null sampler");
    validate(*w);
    if (epochs < 1) invalid("epochs must be >= 1");
    use_device(s->device);
    DevBuf<uint8_t> mask;
    upload_mask(mask, s->E, cache, k, s->st);
    const uint64_t q = w->num_samples, b = w->batch_size, d = w->lookups_per_sample;
    const uint64_t n_batches = (q + b - 1) / b;
    const uint64_t per_chunk = std::max<uint64_t>(1, kChunkDraws / (b * d));
    Stat st_all, st_nc;
    double emb_units = 0.0;
    int64_t hot = 0, total = 0;
    std::vector<int> all, nc;
    for (int64_t e = 0; e < epochs; ++e) {
      const uint64_t seed_e = substream(seed, static_cast<uint64_t>(e));  // simulator.cpp:186
      for (uint64_t j0 = 0; j0 < n_batches; j0 += per_chunk) {
        const uint64_t nbj = std::min(per_chunk, n_batches - j0);
        std::vector<uint64_t> bsz(nbj);
        uint64_t n = 0;
        for (uint64_t j = 0; j < nbj; ++j) {
          bsz[j] = std::min(b, q - (j0 + j) * b);
          n += bsz[j] * d;
        }
        s->work.ensure(n, 0, 0, 0);
        k_sample_epoch<<<grid_for(n, s->device), 256, 0, s->st>>>(s->dev(), seed_e, q, b, d, j0 * b * d, n,
                                                                   s->work.ids.p);
        EC_LAUNCH();
        count_batches(s->work, s->device, n, bsz, static_cast<uint32_t>(d), b, k ? mask.p : nullptr, all, nc,
                      s->st);
        for (uint64_t j = 0; j < nbj; ++j) {  // simulator.cpp:194-205, batch then column order
          int64_t batch_nc = 0;
          for (uint64_t f = 0; f < d; ++f) {
            if (bsz[j] == b) {
              st_all.add(static_cast<double>(all[j * d + f]));
              st_nc.add(static_cast<double>(nc[j * d + f]));
            }
            batch_nc += nc[j * d + f];
          }
          emb_units += static_cast<double>(batch_nc);
          hot += batch_nc == 0;
          ++total;
        }
      }
    }
    ec_sim_result r{};
    st_all.finish(&r.unique_mean, &r.unique_std_error);
    st_nc.finish(&r.non_cached_mean, &r.non_cached_std_error);
    r.measured_epoch_cost.index_cost = static_cast<double>(q);
    r.measured_epoch_cost.embedding_cost = emb_units / static_cast<double>(epochs);
    r.measured_epoch_cost.total = r.measured_epoch_cost.index_cost + r.measured_epoch_cost.embedding_cost;
    r.hot_batch_fraction = static_cast<double>(hot) / static_cast<double>(total);
    *out = r;
  });
}

}  // extern "C"

// ------------------------------------------------------------ trace paths
namespace {
struct TraceOnDevice {
  DevBuf<uint32_t> ids, order;
  DevBuf<uint8_t> mask;
  DevBuf<int> hot, excl, part, scal;  // scal[0] = #hot, scal[1] = bad-id flag
  uint64_t q = 0, nhot = 0;
};

// Upload, classify and stably partition a trace (trace.cpp:185-240).
void classify_and_order(TraceOnDevice& t, const uint32_t* ids, uint64_t q, int64_t d, uint64_t vocab,
                        const uint32_t* cache, uint64_t k, int device, cudaStream_t st, bool want_order) {
  if (d < 1) invalid("lookups per sample must be >= 1");
  if (vocab < 1) invalid("vocabulary size must be >= 1");
  if (q == 0) invalid("empty trace");
  use_device(device);
  t.q = q;
  const uint64_t n = q * static_cast<uint64_t>(d);
  t.ids.alloc(n);
  EC_CUDA(cudaMemcpyAsync(t.ids.p, ids, n * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
  upload_mask(t.mask, vocab, cache, k, st);
  t.hot.alloc(q);
  t.scal.alloc(2);
  EC_CUDA(cudaMemsetAsync(t.scal.p, 0, 2 * sizeof(int), st));
  k_classify<<<grid_for(q, device), 256, 0, st>>>(t.ids.p, q, static_cast<uint32_t>(d), vocab, t.mask.p, t.hot.p,
                                                   t.scal.p + 1);
  EC_LAUNCH();
  if (want_order) {
    t.excl.alloc(q);
    t.part.alloc(scan_parts(q));
    t.order.alloc(q);
    exclusive_scan(t.hot.p, static_cast<int64_t>(q), t.excl.p, t.part.p, t.scal.p, st);
    k_partition_order<<<grid_for(q, device), 256, 0, st>>>(t.hot.p, t.excl.p, t.scal.p, q, t.order.p);
    EC_LAUNCH();
  }
  int h[2];
  EC_CUDA(cudaMemcpyAsync(h, t.scal.p, sizeof(h), cudaMemcpyDeviceToHost, st));
  EC_CUDA(cudaStreamSynchronize(st));
  if (h[1]) invalid("trace id out of range [0, " + std::to_string(vocab) + ")");
  t.nhot = static_cast<uint64_t>(h[0]);
}

struct Stream {
  cudaStream_t s = nullptr;
  Stream() { EC_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }
  ~Stream() { cudaStreamDestroy(s); }
};
}  // namespace

extern "C" {

int ec_classify_samples(const uint32_t* ids, uint64_t q, int64_t d, uint64_t vocab, const uint32_t* cache,
                        uint64_t k, int device, uint8_t* hot_host) {
  return guard([&] {
    use_device(device);
    Stream st;
    TraceOnDevice t;
    classify_and_order(t, ids, q, d, vocab, cache, k, device, st.s, false);
    std::vector<int> h(q);
    EC_CUDA(cudaMemcpy(h.data(), t.hot.p, q * sizeof(int), cudaMemcpyDeviceToHost));
    for (uint64_t s = 0; s < q; ++s) hot_host[s] = static_cast<uint8_t>(h[s]);
  });
}

int ec_schedule_order(const uint32_t* ids, uint64_t q, int64_t d, uint64_t vocab, const uint32_t* cache,
                      uint64_t k, int device, uint32_t* order_host, uint64_t* num_hot) {
  return guard([&] {
    use_device(device);
    Stream st;
    TraceOnDevice t;
    classify_and_order(t, ids, q, d, vocab, cache, k, device, st.s, true);
    EC_CUDA(cudaMemcpy(order_host, t.order.p, q * sizeof(uint32_t), cudaMemcpyDeviceToHost));
    *num_hot = t.nhot;
  });
}

// build_schedule with a shuffle seed (core/src/trace.cpp:206-240): the GPU's
// stable hot/normal partition, then each class permuted on the host by a
// Fisher-Yates walk from the top index down, drawing j = next() % (i + 1) from
// SplitMix64(substream_seed(seed, class)) -- class 0 hot, 1 normal
// (trace.cpp:211-222).  The permutation is a serial chain of 64-bit draws, so it
// stays on the host; the partition (the O(Q*d) part) runs on the device.
int ec_build_schedule(const uint32_t* ids, uint64_t q, int64_t d, uint64_t vocab, const uint32_t* cache, uint64_t k,
                      int device, int shuffle, uint64_t seed, uint32_t* order_host, uint64_t* num_hot) {
  return guard([&] {
    use_device(device);
    Stream st;
    TraceOnDevice t;
    classify_and_order(t, ids, q, d, vocab, cache, k, device, st.s, true);
    EC_CUDA(cudaMemcpy(order_host, t.order.p, q * sizeof(uint32_t), cudaMemcpyDeviceToHost));
    *num_hot = t.nhot;
    if (!shuffle) return;
    const uint64_t lo[2] = {0, t.nhot}, hi[2] = {t.nhot, q};
    for (int cls = 0; cls < 2; ++cls) {
      uint64_t state = substream(seed, static_cast<uint64_t>(cls));
      uint32_t* v = order_host + lo[cls];
      for (uint64_t len = hi[cls] - lo[cls]; len > 1; --len) {
        state += kGolden;
        const uint64_t j = mix64(state) % len;
        std::swap(v[len - 1], v[j]);
      }
    }
  });
}

// simulate_epoch(Trace, b, C), core/src/simulator.cpp:222-273.
int ec_simulate_trace(const uint32_t* ids, uint64_t q, int64_t d, uint64_t vocab, int64_t b,
                      const uint32_t* cache, uint64_t k, int device, ec_sim_result* out) {
  return guard([&] {
    if (b < 1) invalid("batch size must be >= 1");
    use_device(device);
    Stream st;
    TraceOnDevice t;
    classify_and_order(t, ids, q, d, vocab, cache, k, device, st.s, true);
    // batches: hot class packed by b, then the normal class (trace.cpp:314-328)
    std::vector<uint64_t> bsz, pos0;
    for (uint64_t cls_lo : {uint64_t{0}, t.nhot}) {
      const uint64_t cls_hi = cls_lo == 0 ? t.nhot : q;
      for (uint64_t p = cls_lo; p < cls_hi; p += b) {
        pos0.push_back(p);
        bsz.push_back(std::min<uint64_t>(b, cls_hi - p));
      }
    }
    const uint64_t nb = bsz.size(), n = q * static_cast<uint64_t>(d);
    std::vector<uint64_t> boff(nb + 1, 0);
    for (uint64_t j = 0; j < nb; ++j) boff[j + 1] = boff[j] + bsz[j] * d;
    CountWork w;
    w.ensure(n, 0, 0, nb);
    DevBuf<uint64_t> dpos(nb);
    EC_CUDA(cudaMemcpyAsync(w.boff.p, boff.data(), (nb + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, st.s));
    EC_CUDA(cudaMemcpyAsync(dpos.p, pos0.data(), nb * sizeof(uint64_t), cudaMemcpyHostToDevice, st.s));
    k_gather_schedule<<<grid_for(n, device), 256, 0, st.s>>>(t.ids.p, t.order.p, w.boff.p, dpos.p,
                                                              static_cast<uint32_t>(nb), static_cast<uint32_t>(d),
                                                              n, w.ids.p);
    EC_LAUNCH();
    std::vector<int> all, nc;
    count_batches(w, device, n, bsz, static_cast<uint32_t>(d), static_cast<uint64_t>(b), k ? t.mask.p : nullptr,
                  all, nc, st.s);
    Stat st_all, st_nc;
    double emb = 0.0;
    int64_t hot = 0;
    for (uint64_t j = 0; j < nb; ++j) {
      int64_t batch_nc = 0;
      for (int64_t f = 0; f < d; ++f) {
        if (bsz[j] == static_cast<uint64_t>(b)) {
          st_all.add(static_cast<double>(all[j * d + f]));
          st_nc.add(static_cast<double>(nc[j * d + f]));
        }
        batch_nc += nc[j * d + f];
      }
      emb += static_cast<double>(batch_nc);
      hot += batch_nc == 0;
    }
    ec_sim_result r{};
    st_all.finish(&r.unique_mean, &r.unique_std_error);
    st_nc.finish(&r.non_cached_mean, &r.non_cached_std_error);
    r.measured_epoch_cost.index_cost = static_cast<double>(q);
    r.measured_epoch_cost.embedding_cost = emb;
    r.measured_epoch_cost.total = r.measured_epoch_cost.index_cost + emb;
    r.hot_batch_fraction = nb ? static_cast<double>(hot) / static_cast<double>(nb) : 0.0;
    *out = r;
  });
}

}  // extern "C"

// ------------------------------------------------ frequency placement (a17)
// build_skew_table (core/src/trace.cpp:128-150): exact access counts — the
// O(Q*d) histogram runs on the GPU — then the observed ids ordered by (count
// desc, id asc) with the running fraction, on the host (O(S log S) over the S
// observed ids).  estimate_distribution (trace.cpp:161-183) restated on the
// host so probabilities and ranks are bit-identical.
namespace {
__global__ void k_histogram(const uint32_t* __restrict__ ids, uint64_t n, uint64_t vocab,
                            unsigned long long* __restrict__ counts, int* __restrict__ bad) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t id = ids[i];
    if (id >= vocab) {
      atomicExch(bad, 1);
      continue;
    }
    // hot ids repeat inside a warp: one atomic per distinct id
    const unsigned peers = __match_any_sync(__activemask(), id);
    if ((__ffs(peers) - 1) == lane_id()) atomicAdd(counts + id, static_cast<unsigned long long>(__popc(peers)));
  }
}
}  // namespace

extern "C" {

int ec_build_skew_table(const uint32_t* ids_host, uint64_t n, uint64_t vocab, int device, uint32_t* out_ids,
                        uint64_t* out_counts, double* out_cum, uint64_t* n_entries) {
  return guard([&] {
    if (n == 0) invalid("empty trace");
    if (vocab < 1) invalid("vocabulary size must be >= 1");
    use_device(device);
    Stream st;
    DevBuf<uint32_t> d_ids(n);
    DevBuf<unsigned long long> d_cnt(vocab);
    DevBuf<int> d_bad(1);
    EC_CUDA(cudaMemcpyAsync(d_ids.p, ids_host, n * sizeof(uint32_t), cudaMemcpyHostToDevice, st.s));
    EC_CUDA(cudaMemsetAsync(d_cnt.p, 0, vocab * sizeof(unsigned long long), st.s));
    EC_CUDA(cudaMemsetAsync(d_bad.p, 0, sizeof(int), st.s));
    k_histogram<<<grid_for(n, device), 256, 0, st.s>>>(d_ids.p, n, vocab, d_cnt.p, d_bad.p);
    EC_LAUNCH();
    std::vector<unsigned long long> cnt(vocab);
    int bad = 0;
    EC_CUDA(cudaMemcpyAsync(cnt.data(), d_cnt.p, vocab * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st.s));
    EC_CUDA(cudaMemcpyAsync(&bad, d_bad.p, sizeof(int), cudaMemcpyDeviceToHost, st.s));
    EC_CUDA(cudaStreamSynchronize(st.s));
    if (bad) invalid("trace id out of range [0, " + std::to_string(vocab) + ")");
    std::vector<uint32_t> obs;
    for (uint64_t id = 0; id < vocab; ++id)
      if (cnt[id]) obs.push_back(static_cast<uint32_t>(id));
    std::sort(obs.begin(), obs.end(), [&](uint32_t a, uint32_t b) { return cnt[a] != cnt[b] ? cnt[a] > cnt[b] : a < b; });
    uint64_t run = 0;
    for (size_t k = 0; k < obs.size(); ++k) {
      run += cnt[obs[k]];
      if (out_ids) out_ids[k] = obs[k];
      if (out_counts) out_counts[k] = cnt[obs[k]];
      if (out_cum) out_cum[k] = static_cast<double>(run) / static_cast<double>(n);
    }
    *n_entries = obs.size();
  });
}

int ec_estimate_distribution(const uint32_t* entry_ids, const uint64_t* entry_counts, uint64_t n_entries,
                             uint64_t total_accesses, uint64_t vocab, double smoothing, ec_dist* out) {
  return guard([&] {
    if (smoothing < 0.0) invalid("smoothing must be >= 0");
    uint32_t max_id = 0;
    for (uint64_t k = 0; k < n_entries; ++k) max_id = std::max(max_id, entry_ids[k]);
    if (n_entries && vocab < static_cast<uint64_t>(max_id) + 1)
      invalid("vocabulary size " + std::to_string(vocab) + " smaller than max observed id " + std::to_string(max_id));
    if (vocab == 0) invalid("vocabulary size must be >= 1");
    const double denom = static_cast<double>(total_accesses) + smoothing * static_cast<double>(vocab);
    if (!(denom > 0.0)) invalid("cannot estimate a distribution from zero observations without smoothing");
    std::vector<double> p(vocab, smoothing / denom);
    for (uint64_t k = 0; k < n_entries; ++k) p[entry_ids[k]] = (static_cast<double>(entry_counts[k]) + smoothing) / denom;
    *out = make_dist(Dist::from_probabilities(std::move(p)));
  });
}

}  // extern "C"
