// Host-link microbenchmark (not shipped): random row reads / writes between a
// B200 and pinned host memory, the pattern of the cold tier (k_gather_host /
// k_apply_host).  Built by tools/Makefile, run under gpurun.
//
//   ./hostlink_bench [numa_node|-1] [rows] [alloc: mmap|cuda|hugetlb] [interference]
//
// Prints the GPU's NUMA node, sequential H2D/D2H copy bandwidth, and the time
// of an LSU gather / scatter of `rows` random rows at several grid sizes.
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#define CK(x)                                                                                \
  do {                                                                                       \
    cudaError_t e_ = (x);                                                                    \
    if (e_ != cudaSuccess) {                                                                 \
      std::fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      std::exit(1);                                                                          \
    }                                                                                        \
  } while (0)

// one 16-byte lane per thread, VEC lanes per row, rows grid-strided
template <int VEC>
__global__ void k_read(const float4* __restrict__ host, const uint32_t* __restrict__ idx, int n, float4* __restrict__ out) {
  const int lanes = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n * VEC; i += lanes) {
    const int r = i / VEC, c = i % VEC;
    out[i] = host[static_cast<size_t>(idx[r]) * VEC + c];
  }
}
template <int VEC>
__global__ void k_write(float4* __restrict__ host, const uint32_t* __restrict__ idx, int n, const float4* __restrict__ in) {
  const int lanes = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n * VEC; i += lanes) {
    const int r = i / VEC, c = i % VEC;
    host[static_cast<size_t>(idx[r]) * VEC + c] = in[i];
  }
}

// ids-style bulk stream (pinned host -> device) by SM loads, few CTAs
__global__ void k_stream(const int4* __restrict__ src, int4* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

// Row reads (7187 x 64 B, grid 16, as k_gather_host) alone and beside a 1.7 MB
// bulk H2D transfer: copy engine vs SM loads at several CTA counts.
static void interference(float4* host, int rows_total, void* bulk_host) {
  const int n = 7187;
  const size_t bulk = 1703936;
  std::mt19937 rng(11);
  std::vector<uint32_t> idx(n);
  for (auto& x : idx) x = rng() % rows_total;
  uint32_t* didx;
  float4* buf;
  void* dbulk;
  CK(cudaMalloc(&didx, n * 4));
  CK(cudaMalloc(&buf, static_cast<size_t>(n) * 64));
  CK(cudaMalloc(&dbulk, bulk));
  CK(cudaMemcpy(didx, idx.data(), n * 4, cudaMemcpyHostToDevice));
  int4* bulk_dev_view;
  CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&bulk_dev_view), bulk_host, 0));
  cudaStream_t s1, s2;
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  cudaEvent_t a, b, c, d;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(cudaEventCreate(&c));
  CK(cudaEventCreate(&d));
  for (int mode = 0; mode < 6; ++mode) {  // 0 alone, 1 copy engine, 2.. SM stream with 1,2,4,8 CTAs
    float best_r = 1e9f, best_t = 1e9f, best_b = 1e9f;
    for (int it = 0; it < 10; ++it) {
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(a, s1));
      CK(cudaStreamWaitEvent(s2, a, 0));
      if (mode == 1) CK(cudaMemcpyAsync(dbulk, bulk_host, bulk, cudaMemcpyHostToDevice, s2));
      if (mode >= 2)
        k_stream<<<1 << (mode - 2), 512, 0, s2>>>(bulk_dev_view, static_cast<int4*>(dbulk), bulk / 16);
      CK(cudaEventRecord(c, s2));
      k_read<4><<<16, 256, 0, s1>>>(host, didx, n, buf);
      CK(cudaEventRecord(b, s1));
      CK(cudaStreamWaitEvent(s1, c, 0));
      CK(cudaEventRecord(d, s1));
      CK(cudaEventSynchronize(d));
      float ms;
      CK(cudaEventElapsedTime(&ms, a, b));
      best_r = std::min(best_r, ms);
      CK(cudaEventElapsedTime(&ms, a, c));
      best_b = std::min(best_b, ms);
      CK(cudaEventElapsedTime(&ms, a, d));
      best_t = std::min(best_t, ms);
    }
    const char* names[] = {"rows alone", "rows + copy engine 1.7MB", "rows + SM stream 1 CTA", "rows + SM stream 2 CTAs",
                           "rows + SM stream 4 CTAs", "rows + SM stream 8 CTAs"};
    std::printf("  %-28s rows %7.1f us  bulk %7.1f us  both %7.1f us\n", names[mode], best_r * 1e3,
                mode ? best_b * 1e3 : 0.f, best_t * 1e3);
  }
}

// HBM-bound neighbour: a grid-stride copy over all SMs (what the pool/scatter
// do beside the host gather in a pipelined step)
__global__ void k_hbm_copy(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

// the engine's host gather chain: queue slot -> unique index -> id -> row
template <int VEC>
__global__ void k_read_chain(const float4* __restrict__ host, const uint32_t* __restrict__ missq,
                             const uint32_t* __restrict__ uniq, int n, float4* __restrict__ out) {
  const int lanes = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n * VEC; i += lanes) {
    const int q = i / VEC, c = i % VEC;
    const uint32_t g = missq[q];
    out[static_cast<size_t>(g) * VEC + c] = host[static_cast<size_t>(uniq[g]) * VEC + c];
  }
}

static void chain_cost(float4* host, int rows_total) {
  const int n = 7187, U = 75000;
  std::mt19937 rng(17);
  std::vector<uint32_t> uniq(U), missq(n);
  for (auto& x : uniq) x = rng() % rows_total;
  for (auto& x : missq) x = rng() % U;
  uint32_t *du, *dq, *didx;
  float4* buf;
  CK(cudaMalloc(&du, U * 4));
  CK(cudaMalloc(&dq, n * 4));
  CK(cudaMalloc(&didx, n * 4));
  CK(cudaMalloc(&buf, static_cast<size_t>(U) * 64));
  CK(cudaMemcpy(du, uniq.data(), U * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dq, missq.data(), n * 4, cudaMemcpyHostToDevice));
  std::vector<uint32_t> flat(n);
  for (int i = 0; i < n; ++i) flat[i] = uniq[missq[i]];
  CK(cudaMemcpy(didx, flat.data(), n * 4, cudaMemcpyHostToDevice));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  for (int mode = 0; mode < 2; ++mode) {
    float best = 1e9f;
    for (int it = 0; it < 10; ++it) {
      CK(cudaEventRecord(a));
      if (mode == 0) k_read<4><<<16, 256>>>(host, didx, n, buf);
      else k_read_chain<4><<<16, 256>>>(host, dq, du, n, buf);
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      float ms;
      CK(cudaEventElapsedTime(&ms, a, b));
      best = std::min(best, ms);
    }
    std::printf("  %s: %.1f us\n", mode == 0 ? "row index precomputed" : "queue -> unique -> id chain", best * 1e3);
  }
}

static void hbm_interference(float4* host, int rows_total) {
  const int n = 7187;
  std::mt19937 rng(13);
  std::vector<uint32_t> idx(n);
  for (auto& x : idx) x = rng() % rows_total;
  uint32_t* didx;
  float4* buf;
  CK(cudaMalloc(&didx, n * 4));
  CK(cudaMalloc(&buf, static_cast<size_t>(n) * 64));
  CK(cudaMemcpy(didx, idx.data(), n * 4, cudaMemcpyHostToDevice));
  const size_t hb = 1ull << 30;
  float4 *ha, *hbuf;
  CK(cudaMalloc(&ha, hb));
  CK(cudaMalloc(&hbuf, hb));
  cudaStream_t s1, s2;
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  cudaEvent_t a, b, c;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(cudaEventCreate(&c));
  for (int mode = 0; mode < 3; ++mode) {  // 0 rows alone, 1 beside an HBM copy (4 CTAs/SM), 2 beside 1 CTA/SM
    float best = 1e9f, bestc = 1e9f;
    for (int it = 0; it < 8; ++it) {
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(a, s1));
      CK(cudaStreamWaitEvent(s2, a, 0));
      if (mode) k_hbm_copy<<<148 * (mode == 1 ? 4 : 1), 256, 0, s2>>>(ha, hbuf, hb / 16 / 8);
      CK(cudaEventRecord(c, s2));
      k_read<4><<<16, 256, 0, s1>>>(host, didx, n, buf);
      CK(cudaEventRecord(b, s1));
      CK(cudaDeviceSynchronize());
      float ms;
      CK(cudaEventElapsedTime(&ms, a, b));
      best = std::min(best, ms);
      CK(cudaEventElapsedTime(&ms, a, c));
      bestc = std::min(bestc, ms);
    }
    std::printf("  rows %s: %.1f us (copy %.1f us)\n", mode == 0 ? "alone" : mode == 1 ? "+HBM copy 4 CTAs/SM" : "+HBM copy 1 CTA/SM",
                best * 1e3, mode ? bestc * 1e3 : 0.f);
  }
}

static int gpu_numa_node() {
  char bus[64];
  CK(cudaDeviceGetPCIBusId(bus, sizeof(bus), 0));
  for (char* p = bus; *p; ++p) *p = static_cast<char>(std::tolower(*p));
  std::string path = std::string("/sys/bus/pci/devices/") + bus + "/numa_node";
  FILE* f = std::fopen(path.c_str(), "r");
  if (!f) {
    // sysfs uses a 4-digit domain
    std::string b(bus);
    if (b.size() > 4 && b[8] == ':') b = b.substr(4);
    path = "/sys/bus/pci/devices/" + b + "/numa_node";
    f = std::fopen(path.c_str(), "r");
  }
  int node = -2;
  if (f) {
    if (std::fscanf(f, "%d", &node) != 1) node = -2;
    std::fclose(f);
  }
  std::printf("gpu pci %s numa_node %d\n", bus, node);
  return node;
}

template <int VEC>
static void run(float4* host, int rows_total, int n, int row_bytes) {
  std::mt19937 rng(7);
  std::vector<uint32_t> idx(n);
  for (auto& x : idx) x = rng() % rows_total;
  uint32_t* didx;
  float4* buf;
  CK(cudaMalloc(&didx, n * 4));
  CK(cudaMalloc(&buf, static_cast<size_t>(n) * row_bytes));
  CK(cudaMemcpy(didx, idx.data(), n * 4, cudaMemcpyHostToDevice));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  for (int grid : {16, 32, 74, 148, 296, 592}) {
    float best_r = 1e9f, best_w = 1e9f;
    for (int it = 0; it < 8; ++it) {
      CK(cudaEventRecord(a));
      k_read<VEC><<<grid, 256>>>(host, didx, n, buf);
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      float ms;
      CK(cudaEventElapsedTime(&ms, a, b));
      best_r = std::min(best_r, ms);
      CK(cudaEventRecord(a));
      k_write<VEC><<<grid, 256>>>(host, didx, n, buf);
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      CK(cudaEventElapsedTime(&ms, a, b));
      best_w = std::min(best_w, ms);
    }
    std::printf("  row %4d B rows %6d grid %4d: read %7.1f us (%6.1f GB/s, %6.1f Mrows/s)  write %7.1f us (%6.1f GB/s)\n",
                row_bytes, n, grid, best_r * 1e3, n * (double)row_bytes / (best_r * 1e6), n / (best_r * 1e3),
                best_w * 1e3, n * (double)row_bytes / (best_w * 1e6));
  }
  {  // reads and writes at once on two streams (disjoint rows)
    uint32_t* didx2;
    float4* buf2;
    std::vector<uint32_t> idx2(n);
    for (auto& x : idx2) x = rng() % rows_total;
    CK(cudaMalloc(&didx2, n * 4));
    CK(cudaMalloc(&buf2, static_cast<size_t>(n) * row_bytes));
    CK(cudaMemcpy(didx2, idx2.data(), n * 4, cudaMemcpyHostToDevice));
    cudaStream_t s1, s2;
    CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    float best = 1e9f;
    for (int it = 0; it < 8; ++it) {
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(a));
      CK(cudaStreamWaitEvent(s1, a, 0));
      CK(cudaStreamWaitEvent(s2, a, 0));
      k_read<VEC><<<148, 256, 0, s1>>>(host, didx, n, buf);
      k_write<VEC><<<148, 256, 0, s2>>>(host, didx2, n, buf2);
      cudaEvent_t e1, e2;
      CK(cudaEventCreate(&e1));
      CK(cudaEventCreate(&e2));
      CK(cudaEventRecord(e1, s1));
      CK(cudaEventRecord(e2, s2));
      CK(cudaStreamWaitEvent(0, e1, 0));
      CK(cudaStreamWaitEvent(0, e2, 0));
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      float ms;
      CK(cudaEventElapsedTime(&ms, a, b));
      best = std::min(best, ms);
    }
    std::printf("  row %4d B rows %6d: concurrent read+write %7.1f us\n", row_bytes, n, best * 1e3);
    CK(cudaFree(didx2));
    CK(cudaFree(buf2));
  }
  CK(cudaFree(didx));
  CK(cudaFree(buf));
}

int main(int argc, char** argv) {
  const int node = argc > 1 ? std::atoi(argv[1]) : -1;
  const int n = argc > 2 ? std::atoi(argv[2]) : 7187;
  const size_t bytes = 2ull << 30;
  gpu_numa_node();
  long nodes = 0;
  for (int i = 0; i < 64; ++i) {
    char p[64];
    std::snprintf(p, sizeof(p), "/sys/devices/system/node/node%d", i);
    if (access(p, F_OK) == 0) ++nodes;
  }
  std::printf("numa nodes %ld, host memory bound to node %d\n", nodes, node);
  const std::string mode = argc > 3 ? argv[3] : "mmap";
  void* p = nullptr;
  if (mode == "cuda") {
    CK(cudaHostAlloc(&p, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
  } else {
    p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE,
             MAP_PRIVATE | MAP_ANONYMOUS | (mode == "hugetlb" ? MAP_HUGETLB : 0), -1, 0);
    if (p == MAP_FAILED) {
      std::printf("mmap %s failed\n", mode.c_str());
      return 1;
    }
    madvise(p, bytes, MADV_HUGEPAGE);
  }
  std::printf("alloc %s\n", mode.c_str());
  if (node >= 0) {
    unsigned long mask[16] = {};
    mask[node / 64] = 1ul << (node % 64);
    const long r = syscall(SYS_mbind, p, bytes, 2 /*MPOL_BIND*/, mask, 1024, 0);
    std::printf("mbind -> %ld\n", r);
  }
  std::memset(p, 0, bytes);
  if (mode != "cuda") CK(cudaHostRegister(p, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable));
  float4* host;
  CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&host), p, 0));
  {  // sequential copy bandwidth
    void* d;
    CK(cudaMalloc(&d, 256 << 20));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    float h2d = 1e9f, d2h = 1e9f, ms;
    for (int i = 0; i < 5; ++i) {
      CK(cudaEventRecord(a));
      CK(cudaMemcpyAsync(d, p, 256 << 20, cudaMemcpyHostToDevice));
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      CK(cudaEventElapsedTime(&ms, a, b));
      h2d = std::min(h2d, ms);
      CK(cudaEventRecord(a));
      CK(cudaMemcpyAsync(p, d, 256 << 20, cudaMemcpyDeviceToHost));
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      CK(cudaEventElapsedTime(&ms, a, b));
      d2h = std::min(d2h, ms);
    }
    std::printf("sequential 256 MiB: H2D %.1f GB/s  D2H %.1f GB/s\n", 0.256 * 1.048576 / (h2d * 1e-3),
                0.256 * 1.048576 / (d2h * 1e-3));
    CK(cudaFree(d));
  }
  if (argc > 4 && std::string(argv[4]) == "chain") {
    chain_cost(host, static_cast<int>(bytes / 64));
    return 0;
  }
  if (argc > 4 && std::string(argv[4]) == "hbm") {
    hbm_interference(host, static_cast<int>(bytes / 64));
    return 0;
  }
  if (argc > 4 && std::string(argv[4]) == "interference") {
    void* bulk_host;
    CK(cudaHostAlloc(&bulk_host, 1703936, cudaHostAllocMapped));
    std::memset(bulk_host, 1, 1703936);
    interference(host, static_cast<int>(bytes / 64), bulk_host);
    return 0;
  }
  run<4>(host, static_cast<int>(bytes / 64), n, 64);
  run<4>(host, static_cast<int>(bytes / 64), n * 8, 64);
  return 0;
}
