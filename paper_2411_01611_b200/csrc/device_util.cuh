// Device helpers shared by the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace ec {

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr unsigned long long kEmptySlot = ~0ull;  // packed (id << 32 | value); ids < 2^32-1
constexpr uint32_t kEmptyKey = 0xFFFFFFFFu;
constexpr uint32_t kRankTag = 0x80000000u;  // low word holds a (tagged) unique index
constexpr uint32_t kInvalidSlot = 0xFFFFFFFFu;  // lookup whose id is out of range

// Fibonacci hashing: top `bits` bits of id * 2^32/phi.  Consecutive ids (the
// hot ranks of a parametric distribution) land far apart.
__device__ __forceinline__ uint32_t hash_slot(uint32_t id, uint32_t shift) {
  return (id * 0x9E3779B1u) >> shift;
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// Count of `flag` over the lanes of `peers` (a __match_any group); returned on
// every lane.  Full-warp ballot, so callable from converged code only.
__device__ __forceinline__ int group_count(unsigned peers, bool flag) {
  return __popc(__ballot_sync(kFull, flag) & peers);
}

// Vectorised read-only global load (ld.global.nc.v4.f32).
__device__ __forceinline__ float4 ldg4(const float* p) {
  return __ldg(reinterpret_cast<const float4*>(p));
}
// Streaming 128-bit load for data read exactly once (evict-first).
__device__ __forceinline__ float4 ld_stream4(const float* p) {
  return __ldcs(reinterpret_cast<const float4*>(p));
}
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }

__device__ __forceinline__ float4 add4(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}

// Block-wide exclusive scan of one int per thread (blockDim.x == kThreads,
// multiple of 32).  Returns the exclusive prefix; *total gets the block sum.
template <int kThreads>
__device__ __forceinline__ int block_exclusive_scan(int v, int* smem_warp, int* total) {
  constexpr int kWarps = kThreads / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) smem_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = lane < kWarps ? smem_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, w, o);
      if (lane >= o) w += y;
    }
    if (lane < kWarps) smem_warp[lane] = w;  // inclusive warp totals
  }
  __syncthreads();
  const int warp_prefix = warp ? smem_warp[warp - 1] : 0;
  *total = smem_warp[kWarps - 1];
  __syncthreads();  // smem_warp reusable after return
  return warp_prefix + x - v;
}

}  // namespace ec
