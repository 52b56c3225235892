// Device-wide exclusive prefix sum over int32 (reduce -> scan partials ->
// apply), used where a deterministic stable order is needed (schedule
// partition, compaction).  Three short launches; inputs are small next to the
// data-path kernels.
#pragma once

#include "common.hpp"
#include "device_util.cuh"

namespace ec {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

static __global__ void k_scan_reduce(const int* __restrict__ in, int64_t n, int* __restrict__ part) {
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile;
  int s = 0;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    const int64_t i = base + j * kScanThreads + threadIdx.x;
    if (i < n) s += in[i];
  }
  const int v = __reduce_add_sync(kFull, s);
  __shared__ int w[kScanThreads / 32];
  if (lane_id() == 0) w[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int k = 0; k < kScanThreads / 32; ++k) t += w[k];
    part[blockIdx.x] = t;
  }
}

// Single block: exclusive scan of `m` partials in place; total -> *total.
static __global__ void k_scan_partials(int* __restrict__ part, int m, int* __restrict__ total) {
  __shared__ int sw[32];
  int carry = 0;
  for (int base = 0; base < m; base += 1024) {
    const int i = base + threadIdx.x;
    const int v = i < m ? part[i] : 0;
    int tot;
    const int ex = block_exclusive_scan<1024>(v, sw, &tot);
    if (i < m) part[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0 && total) *total = carry;
}

static __global__ void k_scan_apply(const int* __restrict__ in, int64_t n, const int* __restrict__ part,
                             int* __restrict__ out) {
  __shared__ int sw[kScanThreads / 32];
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile;
  int run = part[blockIdx.x];
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    const int64_t i = base + j * kScanThreads + threadIdx.x;
    const int v = i < n ? in[i] : 0;
    int tot;
    const int ex = block_exclusive_scan<kScanThreads>(v, sw, &tot);
    if (i < n) out[i] = run + ex;
    run += tot;
  }
}

// out[i] = sum(in[0..i)); *total_dev = sum(in).  `part` needs
// ceil(n / kScanTile) ints.
inline void exclusive_scan(const int* in, int64_t n, int* out, int* part, int* total_dev,
                           cudaStream_t st) {
  const int blocks = static_cast<int>((n + kScanTile - 1) / kScanTile);
  if (blocks == 0) {
    EC_CUDA(cudaMemsetAsync(total_dev, 0, sizeof(int), st));
    return;
  }
  k_scan_reduce<<<blocks, kScanThreads, 0, st>>>(in, n, part);
  EC_LAUNCH();
  k_scan_partials<<<1, 1024, 0, st>>>(part, blocks, total_dev);
  EC_LAUNCH();
  k_scan_apply<<<blocks, kScanThreads, 0, st>>>(in, n, part, out);
  EC_LAUNCH();
}

inline int64_t scan_parts(int64_t n) { return (n + kScanTile - 1) / kScanTile + 1; }

}  // namespace ec
