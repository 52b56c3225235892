// Probe (not shipped): can the pinned-host tier's random row traffic go
// through host threads + sequential transfers faster than GPU loads/stores of
// random 64 B rows over the link?  Built by tools/Makefile, run under gpurun.
//
//   ./hoststage_probe [rows_in_table=33800000] [misses=7187] [threads=8]
//
// Prints, for M random 64 B rows of a host table:
//   gpu_gather   : SM loads of the random rows through the mapped table (k_gather_host's pattern)
//   gpu_scatter  : SM stores of the random rows into the mapped table (k_apply_host's pattern)
//   cpu_gather   : host threads copy the rows into a contiguous pinned staging buffer
//   cpu_scatter  : host threads copy contiguous staged rows out to the table
//   pull / push  : SM loads / stores of the contiguous staging (M * 64 B)
//   hostfunc     : kernel -> cudaLaunchHostFunc(no-op) -> kernel, extra latency
//   chain_in     : kernel writes keys (mapped) -> hostfunc(cpu gather) -> pull kernel
//   chain_out    : push kernel -> hostfunc(cpu scatter)
#include <cuda_runtime.h>
#include <sys/mman.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

#define CK(x)                                                                                \
  do {                                                                                       \
    cudaError_t e_ = (x);                                                                    \
    if (e_ != cudaSuccess) {                                                                 \
      std::fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      std::exit(1);                                                                          \
    }                                                                                        \
  } while (0)

__global__ void k_rand_read(const float4* __restrict__ host, const uint32_t* __restrict__ idx, int n,
                            float4* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n * 4; i += gridDim.x * blockDim.x)
    out[i] = host[static_cast<size_t>(idx[i / 4]) * 4 + i % 4];
}
__global__ void k_rand_write(float4* __restrict__ host, const uint32_t* __restrict__ idx, int n,
                             const float4* __restrict__ in) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n * 4; i += gridDim.x * blockDim.x)
    host[static_cast<size_t>(idx[i / 4]) * 4 + i % 4] = in[i];
}
__global__ void k_copy(const int4* __restrict__ src, int4* __restrict__ dst, int n16) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += gridDim.x * blockDim.x) dst[i] = src[i];
}
__global__ void k_keys(const uint32_t* __restrict__ idx, int n, uint32_t* __restrict__ keys_host, int* __restrict__ n_host) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) keys_host[i] = idx[i];
  if (blockIdx.x == 0 && threadIdx.x == 0) *n_host = n;
}
__global__ void k_nop() {}

// persistent host worker pool: run(fn) splits [0, n) over the workers and the caller
struct Pool {
  std::vector<std::thread> th;
  std::atomic<unsigned> gen{0}, done{0};
  std::atomic<bool> stop{false};
  int nw;
  const float4* table = nullptr;
  float4* stage = nullptr;
  const uint32_t* keys = nullptr;
  int n = 0;
  bool gather = true;
  explicit Pool(int threads) : nw(threads) {
    for (int w = 1; w < nw; ++w)
      th.emplace_back([this, w] {
        unsigned seen = 0;
        while (!stop.load(std::memory_order_relaxed)) {
          const unsigned g = gen.load(std::memory_order_acquire);
          if (g == seen) continue;  // spin (the probe measures the best case)
          seen = g;
          work(w);
          done.fetch_add(1, std::memory_order_acq_rel);
        }
      });
  }
  ~Pool() {
    stop = true;
    for (auto& t : th) t.join();
  }
  void work(int w) {
    const int lo = static_cast<int>(static_cast<long>(n) * w / nw), hi = static_cast<int>(static_cast<long>(n) * (w + 1) / nw);
    if (gather)
      for (int i = lo; i < hi; ++i) {
        const float4* s = table + static_cast<size_t>(keys[i]) * 4;
        float4* d = stage + static_cast<size_t>(i) * 4;
        d[0] = s[0], d[1] = s[1], d[2] = s[2], d[3] = s[3];
      }
    else
      for (int i = lo; i < hi; ++i) {
        float4* d = const_cast<float4*>(table) + static_cast<size_t>(keys[i]) * 4;
        const float4* s = stage + static_cast<size_t>(i) * 4;
        d[0] = s[0], d[1] = s[1], d[2] = s[2], d[3] = s[3];
      }
  }
  void run(bool g) {
    gather = g;
    done.store(0);
    gen.fetch_add(1, std::memory_order_acq_rel);
    work(0);
    while (done.load(std::memory_order_acquire) != static_cast<unsigned>(nw - 1)) {
    }
  }
};

struct Job {
  Pool* pool;
  const int* n_host;
  bool gather;
};
static void CUDART_CB host_job(void* p) {
  Job* j = static_cast<Job*>(p);
  j->pool->n = *j->n_host;
  j->pool->run(j->gather);
}
static void CUDART_CB host_nop(void*) {}

int main(int argc, char** argv) {
  const size_t rows = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 33800000;
  const int M = argc > 2 ? std::atoi(argv[2]) : 7187;
  const int threads = argc > 3 ? std::atoi(argv[3]) : 8;
  const size_t bytes = rows * 64;
  void* tab = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  madvise(tab, bytes, MADV_HUGEPAGE);
  std::memset(tab, 1, bytes);
  CK(cudaHostRegister(tab, bytes, cudaHostRegisterMapped));
  float4* tab_d;
  CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&tab_d), tab, 0));
  std::mt19937_64 rng(5);
  std::vector<uint32_t> idx(M);
  for (auto& x : idx) x = static_cast<uint32_t>(rng() % rows);
  uint32_t *idx_d, *keys_h;
  float4 *rows_d, *stage_h, *stage_hd;
  int* n_h;
  CK(cudaMalloc(&idx_d, M * 4));
  CK(cudaMemcpy(idx_d, idx.data(), M * 4, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&rows_d, static_cast<size_t>(M) * 64));
  CK(cudaHostAlloc(&keys_h, M * 4, cudaHostAllocMapped));
  CK(cudaHostAlloc(&n_h, 4, cudaHostAllocMapped));
  CK(cudaHostAlloc(&stage_h, static_cast<size_t>(M) * 64, cudaHostAllocMapped));
  CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&stage_hd), stage_h, 0));
  uint32_t* keys_hd;
  int* n_hd;
  CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&keys_hd), keys_h, 0));
  CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&n_hd), n_h, 0));
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  Pool pool(threads);
  pool.table = reinterpret_cast<const float4*>(tab);
  pool.stage = stage_h;
  pool.keys = keys_h;
  std::memcpy(keys_h, idx.data(), M * 4);
  auto time_gpu = [&](const char* name, auto&& enqueue) {
    float best = 1e9f, sum = 0.f;
    for (int it = 0; it < 30; ++it) {
      CK(cudaEventRecord(a, s));
      enqueue();
      CK(cudaEventRecord(b, s));
      CK(cudaEventSynchronize(b));
      float ms;
      CK(cudaEventElapsedTime(&ms, a, b));
      if (it >= 5) best = std::min(best, ms), sum += ms;
    }
    std::printf("%-12s best %7.1f us  mean %7.1f us\n", name, best * 1e3f, sum / 25 * 1e3f);
  };
  auto time_cpu = [&](const char* name, bool g) {
    double best = 1e9, sum = 0;
    for (int it = 0; it < 30; ++it) {
      // a different random row set each time (cold host cache lines)
      for (auto& x : idx) x = static_cast<uint32_t>(rng() % rows);
      std::memcpy(keys_h, idx.data(), M * 4);
      pool.n = M;
      const auto t0 = std::chrono::steady_clock::now();
      pool.run(g);
      const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
      if (it >= 5) best = std::min(best, us), sum += us;
    }
    std::printf("%-12s best %7.1f us  mean %7.1f us  (%d threads)\n", name, best, sum / 25, threads);
  };
  std::printf("table %zu rows (%.2f GB), M = %d rows of 64 B\n", rows, bytes / 1e9, M);
  time_gpu("gpu_gather", [&] { k_rand_read<<<20, 256, 0, s>>>(tab_d, idx_d, M, rows_d); });
  time_gpu("gpu_scatter", [&] { k_rand_write<<<20, 256, 0, s>>>(tab_d, idx_d, M, rows_d); });
  {  // the same rows in ascending address order (IOMMU / page locality)
    std::vector<uint32_t> sidx(idx);
    std::sort(sidx.begin(), sidx.end());
    uint32_t* sidx_d;
    CK(cudaMalloc(&sidx_d, M * 4));
    CK(cudaMemcpy(sidx_d, sidx.data(), M * 4, cudaMemcpyHostToDevice));
    time_gpu("gpu_gather_sorted", [&] { k_rand_read<<<20, 256, 0, s>>>(tab_d, sidx_d, M, rows_d); });
    time_gpu("gpu_scatter_sorted", [&] { k_rand_write<<<20, 256, 0, s>>>(tab_d, sidx_d, M, rows_d); });
    for (int g : {40, 80}) {
      char nm[40];
      std::snprintf(nm, sizeof nm, "gpu_gather_sorted_g%d", g);
      time_gpu(nm, [&] { k_rand_read<<<g, 256, 0, s>>>(tab_d, sidx_d, M, rows_d); });
      std::snprintf(nm, sizeof nm, "gpu_gather_g%d", g);
      time_gpu(nm, [&] { k_rand_read<<<g, 256, 0, s>>>(tab_d, idx_d, M, rows_d); });
    }
  }
  time_cpu("cpu_gather", true);
  time_cpu("cpu_scatter", false);
  const int n16 = M * 4;
  for (int ctas : {4, 8, 16}) {
    char nm[32];
    std::snprintf(nm, sizeof nm, "pull%d", ctas);
    time_gpu(nm, [&] { k_copy<<<ctas, 256, 0, s>>>(reinterpret_cast<const int4*>(stage_hd), reinterpret_cast<int4*>(rows_d), n16); });
    std::snprintf(nm, sizeof nm, "push%d", ctas);
    time_gpu(nm, [&] { k_copy<<<ctas, 256, 0, s>>>(reinterpret_cast<const int4*>(rows_d), reinterpret_cast<int4*>(stage_hd), n16); });
  }
  time_gpu("memcpy_h2d", [&] { CK(cudaMemcpyAsync(rows_d, stage_h, static_cast<size_t>(M) * 64, cudaMemcpyHostToDevice, s)); });
  time_gpu("memcpy_d2h", [&] { CK(cudaMemcpyAsync(stage_h, rows_d, static_cast<size_t>(M) * 64, cudaMemcpyDeviceToHost, s)); });
  time_gpu("2kernels", [&] { k_nop<<<1, 32, 0, s>>>(); k_nop<<<1, 32, 0, s>>>(); });
  time_gpu("hostfunc", [&] { k_nop<<<1, 32, 0, s>>>(); CK(cudaLaunchHostFunc(s, host_nop, nullptr)); k_nop<<<1, 32, 0, s>>>(); });
  Job jin{&pool, n_h, true}, jout{&pool, n_h, false};
  time_gpu("chain_in", [&] {
    k_keys<<<8, 256, 0, s>>>(idx_d, M, keys_hd, n_hd);
    CK(cudaLaunchHostFunc(s, host_job, &jin));
    k_copy<<<8, 256, 0, s>>>(reinterpret_cast<const int4*>(stage_hd), reinterpret_cast<int4*>(rows_d), n16);
  });
  time_gpu("chain_out", [&] {
    k_keys<<<8, 256, 0, s>>>(idx_d, M, keys_hd, n_hd);
    k_copy<<<8, 256, 0, s>>>(reinterpret_cast<const int4*>(rows_d), reinterpret_cast<int4*>(stage_hd), n16);
    CK(cudaLaunchHostFunc(s, host_job, &jout));
  });
  // both directions at once on two streams (the step's gather and write-back overlap)
  cudaStream_t s2;
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  cudaEvent_t j2;
  CK(cudaEventCreateWithFlags(&j2, cudaEventDisableTiming));
  time_gpu("gpu_both", [&] {
    CK(cudaEventRecord(j2, s));
    CK(cudaStreamWaitEvent(s2, j2, 0));
    k_rand_read<<<20, 256, 0, s>>>(tab_d, idx_d, M, rows_d);
    k_rand_write<<<20, 256, 0, s2>>>(tab_d, idx_d, M, rows_d);
    CK(cudaEventRecord(j2, s2));
    CK(cudaStreamWaitEvent(s, j2, 0));
  });
  std::printf("threads available: %u\n", std::thread::hardware_concurrency());
  return 0;
}
