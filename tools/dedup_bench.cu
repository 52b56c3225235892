// Standalone microbenchmark of the K1+K2 cluster dedup kernel with per-phase
// timestamps (EC_TRACE).  Not part of the product; built by tools/Makefile.
//
//   ./dedup_bench [kaggle|tb] [iters] [zipf|uniform] [tag 0|1]
//
// Zipf(1.05) ids per table (host inverse-CDF sampler, not the reference
// stream: only the shape matters here), a top-k cache remap, one L2 hash per
// table.  Prints the kernel time (CUDA events, mean over iters) and, from the
// last launch, per-table phase times (max over the cluster's CTAs).
#define EC_TRACE 1
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <unordered_set>
#include <vector>

#include "lookup_kernels.cuh"

using namespace ec;

static const std::vector<uint64_t> kKaggle = {1460, 583, 10131227, 2202608, 305, 24, 12517, 633, 3, 93145, 5683, 8351593, 3194,
                                              27, 14992, 5461306, 10, 5652, 2173, 4, 7046547, 18, 15, 286181, 105, 142572};
static const std::vector<uint64_t> kTb = {39884406, 39043, 17289, 7420, 20263, 3, 7120, 1543, 63, 38532951, 2953546, 403346, 10,
                                          2208, 11938, 155, 4, 976, 14, 39979771, 25641295, 39664984, 585935, 12972, 108, 36};

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) {                                                               \
      std::fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      std::exit(1);                                                                        \
    }                                                                                      \
  } while (0)

template <int ITEMS>
static void launch(const TableDev* td, int T, const uint32_t* idx, unsigned long long* tstat, int* ctr, uint32_t* uniq,
                   uint32_t* uslot, uint16_t* utab, uint32_t* inv, int32_t* usrc, uint32_t* missq, int* ucount, int tag) {
  constexpr size_t smem = cluster_smem_bytes(ITEMS);
  if (kClusterCtas > 8) CK(cudaFuncSetAttribute(k_dedup_cluster<ITEMS>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute(k_dedup_cluster<ITEMS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_dedup_cluster<ITEMS><<<kClusterCtas * T, kClusterThreads, smem>>>(td, T, idx, tstat, ctr, uniq, uslot, utab, inv, usrc,
                                                                       missq, ucount, tag);
}

int main(int argc, char** argv) {
  const bool tb = argc > 1 && !std::strcmp(argv[1], "tb");
  const int iters = argc > 2 ? std::atoi(argv[2]) : 20;
  const bool uniform = argc > 3 && !std::strcmp(argv[3], "uniform");
  const int tag = argc > 4 ? std::atoi(argv[4]) : 1;
  const std::vector<uint64_t>& rows = tb ? kTb : kKaggle;
  const int T = static_cast<int>(rows.size());
  const int64_t n = tb ? 65536 : 16384;
  const uint64_t cache_rows = tb ? (1ull << 30) / 256 : (256ull << 20) / 64;
  std::mt19937_64 rng(12345);
  std::vector<uint32_t> ids(static_cast<size_t>(n) * T);
  std::vector<TableDev> td(T);
  std::vector<void*> allocs;
  std::vector<uint64_t> hslots;
  std::vector<std::vector<unsigned long long>> hinit;  // each table's set as laid out before a launch
  uint64_t expect_u = 0;
  for (int t = 0; t < T; ++t) {
    const uint64_t E = rows[t];
    std::vector<double> cdf(E);
    double s = 0;
    for (uint64_t i = 0; i < E; ++i) cdf[i] = (s += uniform ? 1.0 : std::pow(static_cast<double>(i + 1), -1.05));
    std::uniform_real_distribution<double> u(0.0, s);
    std::unordered_set<uint32_t> seen;
    for (int64_t i = 0; i < n; ++i) {
      const uint64_t r = std::upper_bound(cdf.begin(), cdf.end(), u(rng)) - cdf.begin();
      ids[t * n + i] = static_cast<uint32_t>(std::min<uint64_t>(r, E - 1));
      seen.insert(ids[t * n + i]);
    }
    expect_u += seen.size();
    const uint64_t k = std::min<uint64_t>(E, cache_rows / T);
    std::vector<int32_t> remap(E);
    for (uint64_t i = 0; i < E; ++i) remap[i] = i < k ? static_cast<int32_t>(i) : -1;
    uint64_t cap = 2;
    while (cap < 2 * std::min<uint64_t>(n, E)) cap <<= 1;
    int bits = 0;
    while ((1ull << bits) < cap) ++bits;
    const uint32_t direct = 1;  // the cluster kernel needs direct-mapped sets
    const uint64_t slots = direct ? E : cap;
    hslots.push_back(slots);
    unsigned long long* h;
    int32_t* rm;
    // direct sets interleave (set word, remap copy) per id (lookup_kernels.cuh:set_word)
    std::vector<unsigned long long> init(2 * slots, ~0ull);
    for (uint64_t i = 0; i < E; ++i) init[2 * i + 1] = static_cast<uint32_t>(remap[i]);
    hinit.push_back(init);
    CK(cudaMalloc(&h, 2 * slots * 8));
    CK(cudaMemcpy(h, init.data(), 2 * slots * 8, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&rm, E * 4));
    CK(cudaMemcpy(rm, remap.data(), E * 4, cudaMemcpyHostToDevice));
    allocs.push_back(h);
    allocs.push_back(rm);
    td[t] = TableDev{h, static_cast<uint32_t>(32 - bits), static_cast<uint32_t>(cap - 1), rm, nullptr, E, t * n, n, direct, 0, nullptr};
  }
  const size_t N = ids.size();
  TableDev* dtd;
  uint32_t *didx, *uniq, *uslot, *inv, *missq;
  int32_t* usrc;
  uint16_t* utab;
  unsigned long long *tstat, *trace;
  int* ctr;
  CK(cudaMalloc(&dtd, T * sizeof(TableDev)));
  CK(cudaMemcpy(dtd, td.data(), T * sizeof(TableDev), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&didx, N * 4));
  CK(cudaMemcpy(didx, ids.data(), N * 4, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&uniq, N * 4));
  CK(cudaMalloc(&uslot, N * 4));
  CK(cudaMalloc(&inv, N * 4));
  CK(cudaMalloc(&missq, N * 4));
  CK(cudaMalloc(&usrc, N * 4));
  int* ucount;
  CK(cudaMalloc(&ucount, N * 4));
  CK(cudaMemset(ucount, 0, N * 4));
  CK(cudaMalloc(&utab, N * 2));
  CK(cudaMalloc(&tstat, T * 8));
  CK(cudaMalloc(&ctr, counters_size(T) * 4));
  CK(cudaMemset(ctr, 0, counters_size(T) * 4));
  const int nblk = kClusterCtas * T;
  CK(cudaMalloc(&trace, nblk * 8 * 8));
  int items = 1;
  while (static_cast<int64_t>(kClusterCtas) * kClusterThreads * items < n) items *= 2;
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  double tot = 0;
  for (int it = 0; it < iters + 3; ++it) {
    CK(cudaMemset(ctr, 0, (counters_size(T) - 1) * 4));
    CK(cudaMemset(tstat, 0, T * 8));
    for (int t = 0; t < T; ++t) CK(cudaMemcpy(td[t].hash, hinit[t].data(), hinit[t].size() * 8, cudaMemcpyHostToDevice));
    unsigned long long* tp = it == iters + 2 ? trace : nullptr;
    CK(cudaMemcpyToSymbol(g_trace, &tp, sizeof(tp)));
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(a));
    switch (items) {
      case 1: launch<1>(dtd, T, didx, tstat, ctr, uniq, uslot, utab, inv, usrc, missq, ucount, tag); break;
      case 2: launch<2>(dtd, T, didx, tstat, ctr, uniq, uslot, utab, inv, usrc, missq, ucount, tag); break;
      case 4: launch<4>(dtd, T, didx, tstat, ctr, uniq, uslot, utab, inv, usrc, missq, ucount, tag); break;
      case 8: launch<8>(dtd, T, didx, tstat, ctr, uniq, uslot, utab, inv, usrc, missq, ucount, tag); break;
      default: launch<16>(dtd, T, didx, tstat, ctr, uniq, uslot, utab, inv, usrc, missq, ucount, tag); break;
    }
    CK(cudaGetLastError());
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (it >= 3 && it < iters + 2) tot += ms;
  }
  std::vector<int> hc(counters_size(T));
  CK(cudaMemcpy(hc.data(), ctr, hc.size() * 4, cudaMemcpyDeviceToHost));
  std::printf("%s: T=%d n=%lld items=%d smem=%zu  kernel %.2f us  U=%d (host %llu) misses=%d err=%d\n", tb ? "tb" : "kaggle", T,
              (long long)n, items, cluster_smem_bytes(items), 1e3 * tot / iters, hc[2 * T], (unsigned long long)expect_u,
              hc[2 * T + 1], hc[2 * T + 3]);
  {  // validate the last launch: uniq[inv[p]] == ids[p], usrc[g] == remap[uniq[g]]
    const int U = hc[2 * T];
    std::vector<uint32_t> hinv(N), huniq(U);
    std::vector<int32_t> husrc(U);
    std::vector<uint16_t> hutab(U);
    CK(cudaMemcpy(hinv.data(), inv, N * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(huniq.data(), uniq, U * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(husrc.data(), usrc, U * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hutab.data(), utab, U * 2, cudaMemcpyDeviceToHost));
    long bad_inv = 0, bad_src = 0, miss = 0;
    for (size_t p = 0; p < N; ++p)
      if (hinv[p] >= static_cast<uint32_t>(U) || huniq[hinv[p]] != ids[p]) ++bad_inv;
    for (int g = 0; g < U; ++g) {
      const uint64_t k = std::min<uint64_t>(rows[hutab[g]], cache_rows / T);
      const int32_t want = huniq[g] < k ? static_cast<int32_t>(huniq[g]) : -1;
      if (husrc[g] != want) ++bad_src;
      miss += want < 0;
    }
    // the L2 set after the kernel: the tagged misses (tag) or nothing
    long left = 0, bad_tag = 0;
    for (int t = 0; t < T; ++t) {
      std::vector<unsigned long long> hw(2 * hslots[t]);
      CK(cudaMemcpy(hw.data(), td[t].hash, hw.size() * 8, cudaMemcpyDeviceToHost));
      for (uint64_t i = 0; i < hslots[t]; ++i) {
        if (hw[2 * i + 1] != hinit[t][2 * i + 1]) ++bad_tag;  // remap copies untouched
      }
      std::vector<unsigned long long> hs(hslots[t]);
      for (uint64_t i = 0; i < hslots[t]; ++i) hs[i] = hw[2 * i];
      for (uint64_t i = 0; i < hslots[t]; ++i)
        if (hs[i] != ~0ull) {
          ++left;
          const uint32_t g = static_cast<uint32_t>(hs[i]) & ~kRankTag;
          if ((hs[i] >> 32) != i || g >= static_cast<uint32_t>(U) || huniq[g] != i || husrc[g] >= 0) ++bad_tag;
        }
    }
    std::printf("validate: bad inverse %ld, bad usrc %ld, expected misses %ld, L2 slots left %ld (want %ld), bad tags %ld\n",
                bad_inv, bad_src, miss, left, tag ? miss : 0L, bad_tag);
  }
  std::vector<unsigned long long> tr(nblk * 8);
  CK(cudaMemcpy(tr.data(), trace, tr.size() * 8, cudaMemcpyDeviceToHost));
  unsigned long long t0 = ~0ull;
  for (int i = 0; i < nblk; ++i) t0 = std::min(t0, tr[i * 8]);
  const char* names[] = {"start", "loaded", "local", "global", "flags", "base", "emit", "inverse"};
  std::printf("per cluster (blockIdx order), us since first CTA start, max over its 8 CTAs:\n%6s", "clus");
  for (int p = 0; p < 8; ++p) std::printf("%9s", names[p]);
  std::printf("\n");
  for (int c = 0; c < T; ++c) {
    std::printf("%6d", c);
    for (int p = 0; p < 8; ++p) {
      unsigned long long m = 0;
      for (int r = 0; r < kClusterCtas; ++r) m = std::max(m, tr[(c * kClusterCtas + r) * 8 + p]);
      std::printf("%9.2f", (m - t0) * 1e-3);
    }
    std::printf("\n");
  }
  return 0;
}
