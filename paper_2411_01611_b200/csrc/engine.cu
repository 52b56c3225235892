// Lookup engine: row-sharded fp32 tables, replicated HBM hot-row cache, and
// the per-batch forward/backward pipeline (K1..K6).
//
// Fused single-rank path (<= 32768 lookups per table, e.g. the Kaggle configs):
//   forward  K1+K2 k_dedup_cluster (one thread-block cluster per table: dedup,
//                  inverse, hit/miss, miss queue; pinned-host tier: also each
//                  lookup's row source, in slot_of), prefetched a step or two
//                  ahead on its own stream (after k_clear_miss_sums and a short
//                  wait)
//            K3h   k_gather_host (pinned-host misses, side stream)
//            K5    k_pool1 / k_pool reading each unique row where it lives
//                  (pinned-host tier: through the row sources, else inverse ->
//                  usrc); trailing blocks reset the batch's set slots
//   backward K6    k_scatter<SGD> (-lr * g straight into cache / HBM rows; rows
//                  with > 64 lookups summed in fp64) -> k_apply_g64 (one rounding
//                  for those); pinned host: k_apply_host + k_patch_prefetch
// Tile path (larger batches, TB / cfg1) and multi-rank:
//   forward  K1    k_insert -> k_compact (single-pass look-back scan + emit)
//            K2    k_inverse_partition (inverse | hit/miss per unique, miss queue)
//            K3    k_gather (cache hits and HBM misses into compact rows)
//            K4    exchange.cu (world > 1)
//            K5    k_pool1 / k_pool from the compact rows
//   backward K6    k_scatter or the transpose (k_bwd_count/fill/reduce; single
//                  rank with HBM rows: SGD of one-chunk rows inside k_bwd_reduce)
//                  -> k_apply (SGD; k_apply_host for pinned-host rows)
// Kernels live in lookup_kernels.cuh.
//
// Reference anchors: the dedup reproduces count_batch_unique's distinct and
// non-cached distinct counts (core/src/simulator.cpp:85-106) per table batch
// (mapping M1), with the unique ids kept in the order the
// reference's UniqueCounter first marks them (simulator.cpp:96-98); the cache
// is the probability-ranked prefix the planner selects
// (core/src/cache_planner.cpp:71-79) and a lookup misses iff
// !cached[id] (simulator.cpp:99).  Gather, pool, exchange and backward have no
// reference counterpart (SURVEY §2 "★ new").
//
// HBM layout (device `dev`, rank r of `world`):
//   store  : per table t, local shard rows (ids with id % world == r, local
//            row id / world), D fp32 each, tables back to back — HBM or
//            pinned host (mapped, read by the GPU over PCIe/C2C)
//   cache  : K_total rows x D fp32 (replicated top-k rows of every table)
//   remap  : per table, int32[E_t]: global cache row or -1
//   hash   : per table and buffer set, (id << 32 | value): an open-addressing
//            set of pow2 >= 2*min(max lookups, E_t) slots, or direct-mapped
//            (slot = id) where the cluster kernel runs; self-cleaning per batch
//   per-batch: slot_of (tile path: lookup -> set slot; fused pinned-host
//            path: lookup -> row source)/inverse (uint32[N]), uniq/uslot/usrc (uint32[N]),
//            utab (uint16[N]), urows (fp32[N x D]), ugrad (fp32[N x D])
#include <nvtx3/nvToolsExt.h>
#include <sys/mman.h>
#include <unistd.h>

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <vector>

#include "common.hpp"
#include "device_util.cuh"
#include "engine.hpp"
#include "scan.cuh"

namespace ec {

// ----------------------------------------------------------- runtime bits
int sm_count(int device) {
  static int cached[64] = {0};
  if (device < 0 || device >= 64) return 148;
  if (!cached[device]) {
    int n = 0;
    EC_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device));
    cached[device] = n;
  }
  return cached[device];
}

void use_device(int device) {
  int n = 0;
  const cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    throw Error(EC_ECUDA, std::string("no CUDA device available (") + cudaGetErrorString(e) +
                              "); libembcomm_gpu has no CPU fallback");
  if (device < 0 || device >= n) invalid("CUDA device " + std::to_string(device) + " out of range");
  EC_CUDA(cudaSetDevice(device));
}

}  // namespace ec

#include "lookup_kernels.cuh"

namespace ec {

// -------------------------------------------------- table maintenance
__device__ __forceinline__ float synth_value(uint64_t seed, float scale, uint32_t t, uint64_t id, uint32_t D,
                                            uint32_t c) {
  const uint64_t x = mix64(seed + kGolden * ((static_cast<uint64_t>(t) << 40) ^ (id * D + c)));
  const float f = static_cast<float>(x >> 40) * 0x1.0p-24f;
  return scale * __fsub_rn(__fmul_rn(2.0f, f), 1.0f);
}

__global__ void k_init_shard(float* __restrict__ store, uint64_t local_rows, uint32_t t, uint32_t D, int rank,
                             int world, uint64_t seed, float scale) {
  const uint64_t n = local_rows * D;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = i / D;
    const uint32_t c = static_cast<uint32_t>(i - r * D);
    store[i] = synth_value(seed, scale, t, r * world + rank, D, c);
  }
}

__global__ void k_copy_remap(unsigned long long* __restrict__ words, const int32_t* __restrict__ remap, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    words[2 * i + 1] = static_cast<uint32_t>(remap[i]);
}

__global__ void k_set_remap(int32_t* __restrict__ remap, const uint32_t* __restrict__ ids, uint64_t k, int64_t slot0) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < k; j += (uint64_t)gridDim.x * blockDim.x)
    remap[ids[j]] = static_cast<int32_t>(slot0 + j);
}

// Cache rows of a new placement, each from where its current value lives:
// the old cache replica (rows cached before and after; replicas are
// bit-identical across ranks), this rank's own shard, a peer's shard over the
// peer-memory exchange (rows never cached since the last flush, so the owner's
// copy is current), or -- before any training -- the synthetic init.  A row
// none of these can supply sets *err (the caller rejects the placement).
__global__ void k_fill_cache(float* __restrict__ cache, const uint32_t* __restrict__ ids, const uint16_t* __restrict__ tabs,
                             uint64_t k, const TableDev* __restrict__ td, uint32_t D, const float* __restrict__ old_cache,
                             const int32_t* __restrict__ old_remap, const int64_t* __restrict__ remap_off,
                             const PeerView* __restrict__ peers, const int64_t* __restrict__ shard_off, uint32_t T,
                             int synth_ok, uint64_t seed, float scale, int rank, int world, int* __restrict__ err) {
  const uint64_t n = k * D;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t j = i / D;
    const uint32_t c = static_cast<uint32_t>(i - j * D);
    const uint32_t id = ids[j];
    const uint32_t t = tabs[j];
    const int o = static_cast<int>(id % world);
    const int32_t os = old_remap ? old_remap[remap_off[t] + id] : -1;
    if (os >= 0)
      cache[i] = old_cache[static_cast<uint64_t>(os) * D + c];
    else if (o == rank)
      cache[i] = td[t].store[static_cast<uint64_t>(id / world) * D + c];
    else if (peers)
      cache[i] = peers[o].store[static_cast<uint64_t>(shard_off[static_cast<int64_t>(o) * (T + 1) + t] + id / world) * D + c];
    else if (synth_ok)
      cache[i] = synth_value(seed, scale, t, id, D, c);
    else
      atomicExch(err, 1);
  }
}

// Write back cached rows owned by this rank into the shard (placement change).
__global__ void k_flush_cache(const float* __restrict__ cache, const uint32_t* __restrict__ ids,
                              const uint16_t* __restrict__ tabs, uint64_t k, const TableDev* __restrict__ td, uint32_t D,
                              int rank, int world) {
  const uint64_t n = k * D;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t j = i / D;
    const uint32_t id = ids[j];
    if (static_cast<int>(id % world) == rank)
      td[tabs[j]].store[static_cast<uint64_t>(id / world) * D + (i - j * D)] = cache[i];
  }
}

__global__ void k_rw_rows(const TableDev* __restrict__ td, uint32_t t, const uint32_t* __restrict__ ids, uint64_t n,
                          uint32_t D, float* __restrict__ cache, float* __restrict__ buf, int write, int rank, int world,
                          int* __restrict__ err) {
  const TableDev tb = td[t];
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n * D; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t j = i / D;
    const uint32_t c = static_cast<uint32_t>(i - j * D);
    const uint32_t id = ids[j];
    if (id >= tb.rows) { atomicExch(err, 1); continue; }
    const int32_t s = tb.remap[id];
    const bool own = static_cast<int>(id % world) == rank;
    float* srow = own ? tb.store + static_cast<uint64_t>(id / world) * D : nullptr;
    if (write) {
      if (s >= 0) cache[static_cast<uint64_t>(s) * D + c] = buf[i];
      if (srow) srow[c] = buf[i];
      if (s < 0 && !srow) atomicExch(err, 2);
    } else {
      if (s >= 0) buf[i] = cache[static_cast<uint64_t>(s) * D + c];
      else if (srow) buf[i] = srow[c];
      else atomicExch(err, 2);
    }
  }
}

// One warp waiting `ns` of device time on the prefetch stream (see prefetch()).
__global__ void k_spin_ns(unsigned ns) {
  unsigned long long start;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(start));
  for (;;) {
    unsigned long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    if (now - start >= ns) break;
  }
}

#ifndef EC_HOST_R
#define EC_HOST_R 4
#endif
constexpr int kHostR = EC_HOST_R;  // rows in flight per lane group in the host-link row kernels
#ifndef EC_FUSED_POOL_R
#define EC_FUSED_POOL_R 4
#endif
#ifndef EC_FUSED_SCATTER_R
#define EC_FUSED_SCATTER_R 4
#endif
// EC_ROW_SOURCES=all: per-lookup row sources on the HBM tier too (A/B)
static bool row_sources_all() {
  static const bool v = [] {
    const char* e = std::getenv("EC_ROW_SOURCES");
    return e && !std::strcmp(e, "all");
  }();
  return v;
}
constexpr int kFusedPoolR = EC_FUSED_POOL_R;        // bags in flight per thread, fused pooling-1 pool
constexpr int kFusedScatterR = EC_FUSED_SCATTER_R;  // bag windows in flight per thread, fused SGD scatter

// ------------------------------------------------------------ host side

// Largest table (rows) whose dedup set is direct-mapped (slot = id) even when
// it exceeds the hash capacity; EC_DIRECT_ROWS overrides (read at creation).
static uint64_t direct_rows_limit() {
  const char* v = std::getenv("EC_DIRECT_ROWS");
  return v && *v ? std::strtoull(v, nullptr, 10) : Engine::kDirectRows;
}
static int persistent_grid(int device) { return sm_count(device) * 8; }
// Row kernels share the SMs with the side-stream host-link kernels: size the
// main grids so every CTA stays resident beside them.
int Engine::host_grid() const {
  static const int env = [] {
    const char* v = std::getenv("EC_HOST_CTAS");
    return v ? std::atoi(v) : 0;
  }();
  if (env > 0) return env;
  // TMA path: the copy engine holds the row reads, so CTAs are cheap -- 2 per
  // SM keep 16 KiB each in flight.
  // LSU path (default): 16 CTAs x 256 threads keep ~4k row reads in flight --
  // the host link is request-rate bound (~215 M rows/s, profiles/r01/hostlink_probe.txt)
  // and deeper queues only stall the concurrent pool/dedup/scatter.  Measured
  // on the pipelined Kaggle step: 12/16/24/32 CTAs 0.099-0.103/0.100-0.104/
  // 0.103-0.110/0.107-0.113 ms; 8 CTAs starve the link (0.109), TMA at 296
  // CTAs 0.105-0.107 with the pool slowed 14 -> 30 us.  Re-measured with the
  // final row grid and pool (gather and write-back together, interleaved):
  // 16/20/24 CTAs 0.1015-0.1034 / 0.0995-0.1001 / 0.1036-0.1047 ms.  Round 2
  // (write-back right after the scatter, prefetched dedup 10 us late), three
  // interleaved sweeps, medians: 8/10/12/16/20 CTAs 0.1049/0.1019-0.1022/
  // 0.1054/0.1032/0.1115 ms; split read/write grids and TMA at 32/64/148 CTAs
  // no better than 10 (0.1026/0.1008-0.1018/0.1065).  Fewer CTAs in flight
  // slow the gather itself (50 -> 54 us) but leave the pool and scatter beside
  // it more room, and the write-back runs faster (40 -> 33 us).
  return host_tma() ? sm_count(device) * 2 : 10;
}
// Host-link row traffic goes through SM loads/stores (k_gather_host /
// k_apply_host) unless EC_HOST_TMA=1 selects the TMA bulk-copy kernels; with
// the single-rank fused path there is no concurrent HBM gather to protect, and
// a bounded number of in-flight rows interferes least with the pipeline.
bool Engine::host_tma() {
  static const bool on = [] {
    const char* v = std::getenv("EC_HOST_TMA");
    return v && v[0] == '1';
  }();
  return on;
}
int Engine::host_write_grid() const {
  static const int env = [] {
    const char* v = std::getenv("EC_HOST_WRITE_CTAS");
    return v ? std::atoi(v) : 0;
  }();
  return env > 0 ? env : host_grid();
}
int Engine::row_grid() const {
  static const int env = [] {
    const char* v = std::getenv("EC_ROW_CTAS_PER_SM");
    return v ? std::atoi(v) : 0;
  }();
  // measured per regime: fused HBM tier 5 (Kaggle 0.0618 -> 0.0596 ms; the
  // fifth CTA per SM waits for registers and fills SMs the concurrent dedup
  // frees); pinned-host tier 4 in round 1 (Kaggle 0.1042-0.1046 at 3,
  // 0.1017-0.1020 at 4, interleaved), 3 with round 2's pipeline (10 host
  // CTAs, write-back right after the scatter: medians 0.0964-0.0967 at 3 vs
  // 0.1037-0.1038 at 4 in two interleaved sweeps); tile/transpose HBM path 4
  // (TB 0.398 vs 0.409, cfg1 0.195 vs 0.201 at 5)
  const int per = storage == EC_STORAGE_HBM ? (fused() ? 5 : 4) : (fused() ? 3 : 4);
  return sm_count(device) * (env > 0 ? env : per);
}

static uint32_t log2_ceil(uint64_t x) {
  uint32_t l = 0;
  while ((1ull << l) < x) ++l;
  return l;
}

// Pinned, GPU-mapped host tier.  Backed by 2 MiB pages where the kernel
// allows (explicit hugetlb, else transparent huge pages via madvise) and then
// registered with CUDA: random GPU reads of 64-256 B rows over the host link
// then touch far fewer page translations than with 4 KiB pages, which
// otherwise throttle the HBM kernels running beside them.  EC_HOST_ALLOC=cuda
// selects plain cudaHostAlloc.
//
// With `shared_fd` (a rank of a multi-process job on the peer-memory
// exchange) the shard is a memfd mapping instead, so that peers on this node
// can map it too (/proc/<pid>/fd/<fd>) and read its rows over their own link.
void* alloc_host_tier(uint64_t bytes, bool* mmapped, int* shared_fd) {
  const char* mode = std::getenv("EC_HOST_ALLOC");
  void* p = nullptr;
  *mmapped = false;
  if (shared_fd) {
    const uint64_t huge = 2ull << 20;
    const uint64_t len = (bytes + huge - 1) / huge * huge;
    int fd = memfd_create("embcomm_host_tier", MFD_CLOEXEC | MFD_HUGETLB);
    if (fd >= 0 && ftruncate(fd, static_cast<off_t>(len)) != 0) {
      close(fd);
      fd = -1;
    }
    if (fd >= 0) {  // hugetlb pages may still be short: try to map
      p = mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_SHARED | MAP_POPULATE, fd, 0);
      if (p == MAP_FAILED) {
        close(fd);
        fd = -1;
      }
    }
    if (fd < 0) {
      fd = memfd_create("embcomm_host_tier", MFD_CLOEXEC);
      if (fd < 0 || ftruncate(fd, static_cast<off_t>(len)) != 0) invalid("cannot create the shared host tier");
      p = mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
      if (p == MAP_FAILED) invalid("cannot map the shared host tier");
      madvise(p, len, MADV_HUGEPAGE);
    }
    EC_CUDA(cudaHostRegister(p, len, cudaHostRegisterMapped | cudaHostRegisterPortable));
    *mmapped = true;
    *shared_fd = fd;
    return p;
  }
  if (!mode || std::strcmp(mode, "cuda") != 0) {
    const uint64_t huge = 2ull << 20;
    const uint64_t len = (bytes + huge - 1) / huge * huge;
    p = mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_HUGETLB, -1, 0);
    if (p == MAP_FAILED) {
      p = mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
      if (p != MAP_FAILED) madvise(p, len, MADV_HUGEPAGE);
    }
    if (p != MAP_FAILED) {
      if (cudaHostRegister(p, len, cudaHostRegisterMapped | cudaHostRegisterPortable) == cudaSuccess) {
        *mmapped = true;
        return p;
      }
      cudaGetLastError();
      munmap(p, len);
    }
    p = nullptr;
  }
  EC_CUDA(cudaHostAlloc(&p, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
  return p;
}

void free_host_tier(void* p, uint64_t bytes, bool mmapped) {
  if (!mmapped) {
    cudaFreeHost(p);
    return;
  }
  const uint64_t huge = 2ull << 20;
  cudaHostUnregister(p);
  munmap(p, (bytes + huge - 1) / huge * huge);
}

Engine::~Engine() {
  clear_graphs();
  if (ev_part) cudaEventDestroy(ev_part);
  if (ev_side) cudaEventDestroy(ev_side);
  if (side) cudaStreamDestroy(side);
  if (pstream) cudaStreamDestroy(pstream);
  if (side2) cudaStreamDestroy(side2);
  if (ev_side2) cudaEventDestroy(ev_side2);
  if (ctr_host) cudaFreeHost(ctr_host);
  if (ring_host) cudaFreeHost(ring_host);
  for (cudaEvent_t ev : ring_ev)
    if (ev) cudaEventDestroy(ev);
  for (BatchBufs& b : bb)
    for (cudaEvent_t e : {b.ev_free, b.ev_ded, b.ev_pf})
      if (e) cudaEventDestroy(e);
  if (ev_grad) cudaEventDestroy(ev_grad);
  if (ev_patch) cudaEventDestroy(ev_patch);
  if (ev_pfcall) cudaEventDestroy(ev_pfcall);
  if (ev_gate) cudaEventDestroy(ev_gate);
  if (ev_b1) cudaEventDestroy(ev_b1);
  destroy_comm();  // (unmaps the peers' shards first)
  if (store_host) free_host_tier(store_host, store_host_bytes, store_host_mmapped);
  if (store_host_fd >= 0) close(store_host_fd);
}

void Engine::create(const ec_tables_config& c) {
  if (c.num_tables < 1) invalid("need at least one table");
  if (c.num_tables > 65535) invalid("at most 65535 tables");
  if (c.dim != 4 && c.dim != 8 && c.dim != 16 && c.dim != 32 && c.dim != 64 && c.dim != 128)
    invalid("dim must be one of 4, 8, 16, 32, 64, 128 (the row kernels' vector widths)");
  if (c.world < 1 || c.rank < 0 || c.rank >= c.world) invalid("rank/world out of range");
  if (c.storage != EC_STORAGE_HBM && c.storage != EC_STORAGE_HOST) invalid("unknown storage tier");
  if (c.max_lookups_per_table < 1 || c.max_lookups_per_table > (1ull << 30))
    invalid("max_lookups_per_table must be in [1, 2^30]");
  if (c.max_batch_size < 1) invalid("max_batch_size must be >= 1");
  if (!c.rows_host) invalid("null rows");
  use_device(c.device);
  device = c.device;
  T = c.num_tables;
  D = c.dim;
  storage = c.storage;
  rank = c.rank;
  world = c.world;
  max_n = c.max_lookups_per_table;
  max_b = c.max_batch_size;
  rows.assign(c.rows_host, c.rows_host + T);
  local_rows.resize(T);
  store_off.assign(T + 1, 0);
  remap_off.assign(T + 1, 0);
  for (uint32_t t = 0; t < T; ++t) {
    if (rows[t] < 1 || rows[t] > 0xFFFFFFFFull) invalid("table " + std::to_string(t) + " rows out of [1, 2^32-1]");
    local_rows[t] = rows[t] > static_cast<uint64_t>(rank) ? (rows[t] - rank + world - 1) / world : 0;
    store_off[t + 1] = store_off[t] + local_rows[t];
    remap_off[t + 1] = remap_off[t] + rows[t];
  }
  // large tables get direct-mapped sets where the cluster dedup kernel will run
  // (it needs them; batches of <= kAutoClusterN lookups per table), hashed ones
  // where the tile path will (TB shape 0.395 -> 0.379 ms, cfg1 0.200 -> 0.187:
  // a 2^17-slot set stays in L2, a 40M-row direct one costs a DRAM sector per
  // probe in each of k_insert, k_compact, k_inverse_partition)
  // (the auto choice of set_geometry: cluster kernel iff every table's batch
  // fits 8 items per thread and the tables alone fill the GPU)
  plan_sets(max_n <= kAutoClusterN && static_cast<int64_t>(T) * kClusterCtas >= sm_count(device));
  const uint64_t store_elems = store_off[T] * D;
  if (storage == EC_STORAGE_HBM) {
    store_dev.alloc(store_elems);
    store_base = store_dev.p;
  } else {
    store_host_bytes = std::max<uint64_t>(store_elems, 1) * sizeof(float);
    store_host = static_cast<float*>(
        alloc_host_tier(store_host_bytes, &store_host_mmapped, world > 1 ? &store_host_fd : nullptr));
    EC_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&store_base), store_host, 0));
  }
  remap.alloc(remap_off[T]);
  EC_CUDA(cudaMemset(remap.p, 0xFF, remap.bytes()));
  alloc_sets();
  const uint64_t N = max_n * T;
  const uint64_t max_tiles = T * ((max_n + kTile - 1) / kTile) + T;
  for (BatchBufs& b : bb) {
    b.slot_of.alloc(N);
    b.inv.alloc(N);
    b.uniq.alloc(N);
    b.uslot.alloc(N);
    b.usrc.alloc(N);
    b.missq.alloc(N);
    b.utab.alloc(N);
    b.urows.alloc(N * D);
    b.ugrad.alloc(N * D);
    b.g64.alloc(N * D);
    EC_CUDA(cudaMemset(b.g64.p, 0, b.g64.bytes()));
    b.ucount.alloc(N);
    EC_CUDA(cudaMemset(b.ucount.p, 0, b.ucount.bytes()));
    b.status.alloc(max_tiles + 1);
    b.ctr.alloc(counters_size(T));
    b.cnt.alloc(N);
    b.off.alloc(N + 1);
    b.list.alloc(N);
    b.part.alloc((N + kScanTile) / kScanTile + 1);
    EC_CUDA(cudaMemset(b.ctr.p, 0, b.ctr.bytes()));
  }
  for (BatchBufs& b : bb) {
    b.tstat.alloc(T);
    EC_CUDA(cudaEventCreateWithFlags(&b.ev_free, cudaEventDisableTiming));
    EC_CUDA(cudaEventCreateWithFlags(&b.ev_ded, cudaEventDisableTiming));
    EC_CUDA(cudaEventCreateWithFlags(&b.ev_pf, cudaEventDisableTiming));
  }
  select(0);
  EC_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&ctr_host), counters_size(T) * sizeof(int), cudaHostAllocDefault));
  EC_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&ring_host), EC_STATS_SLOTS * counters_size(T) * sizeof(int),
                        cudaHostAllocDefault));
  for (cudaEvent_t& ev : ring_ev) EC_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  tiles.alloc(max_tiles);
  tdev_buf.alloc(kSets * T);
  td_host.resize(T);
  for (uint32_t t = 0; t < T; ++t) {
    TableDev& d = td_host[t];
    d.pad_ = 0;
    d.remap = remap.p + remap_off[t];
    d.store = store_base + store_off[t] * D;
    d.rows = rows[t];
    d.base = 0;
    d.n = 0;
  }
  set_views();
  upload_tdev();
  select(cur);
  EC_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
  EC_CUDA(cudaStreamCreateWithFlags(&pstream, cudaStreamNonBlocking));
  EC_CUDA(cudaStreamCreateWithFlags(&side2, cudaStreamNonBlocking));
  EC_CUDA(cudaEventCreateWithFlags(&ev_side2, cudaEventDisableTiming));
  EC_CUDA(cudaEventCreateWithFlags(&ev_grad, cudaEventDisableTiming));
  EC_CUDA(cudaEventCreateWithFlags(&ev_patch, cudaEventDisableTiming));
  EC_CUDA(cudaEventCreateWithFlags(&ev_pfcall, cudaEventDisableTiming));
  EC_CUDA(cudaEventCreateWithFlags(&ev_gate, cudaEventDisableTiming));
  EC_CUDA(cudaEventCreateWithFlags(&ev_b1, cudaEventDisableTiming));
  EC_CUDA(cudaEventCreateWithFlags(&ev_part, cudaEventDisableTiming));
  EC_CUDA(cudaEventCreateWithFlags(&ev_side, cudaEventDisableTiming));
  EC_CUDA(cudaDeviceSynchronize());
}

// Per table: hashed (open addressing, pow2 >= 2 * min(max lookups, rows)
// slots) or direct-mapped (slot = id) dedup set.  Tables that fit the hash
// capacity are always direct (no probing, one atomic per insert); larger ones
// up to direct_rows_limit() rows when `direct_big`, within kDirectBudget.
void Engine::plan_sets(bool direct_big) {
  hash_off.assign(T + 1, 0);
  hash_lg.resize(T);
  hash_direct.resize(T);
  uint64_t direct_bytes = 0;
  for (uint32_t t = 0; t < T; ++t) {
    hash_lg[t] = std::max<uint32_t>(5, log2_ceil(2 * std::min<uint64_t>(max_n, rows[t])));
    const uint64_t lim = std::max<uint64_t>(1ull << hash_lg[t], direct_big ? direct_rows_limit() : 0);
    hash_direct[t] = rows[t] <= lim && direct_bytes + rows[t] * 24 * kSets <= kDirectBudget ? 1 : 0;
    if (hash_direct[t]) direct_bytes += rows[t] * 24 * kSets;  // hash (+ remap copy) + idcnt, every buffer set
    // (64-bit words: a direct set interleaves each id's set word with a copy
    // of its remap entry, lookup_kernels.cuh:set_word)
    hash_off[t + 1] = hash_off[t] + (hash_direct[t] ? 2 * rows[t] : (1ull << hash_lg[t]));
  }
}

// One dedup set per batch-buffer set: a prefetched batch's dedup never waits
// for the current batch's gather to clean the shared slots.
void Engine::alloc_sets() {
  hash.alloc(kSets * hash_off[T]);
  EC_CUDA(cudaMemset(hash.p, 0xFF, hash.bytes()));
  idcnt.alloc(kSets * hash_off[T]);
  EC_CUDA(cudaMemset(idcnt.p, 0, idcnt.bytes()));
}

void Engine::set_views() {
  for (uint32_t t = 0; t < T; ++t) {
    TableDev& d = td_host[t];
    d.hash = hash.p + hash_off[t];
    d.shift = 32 - hash_lg[t];
    d.mask = static_cast<uint32_t>((1ull << hash_lg[t]) - 1);
    d.direct = hash_direct[t];
    d.idcnt = idcnt.p + hash_off[t];
  }
}

// Dedup modes 2 / 3 run kernels that need every set direct-mapped: re-lay the
// sets out (between batches; pending prefetches dropped) when some are hashed.
void Engine::require_direct_sets() {
  bool all = true;
  for (uint32_t t = 0; t < T; ++t) all = all && hash_direct[t];
  if (all) return;
  use_device(device);
  EC_CUDA(cudaDeviceSynchronize());
  drop_prefetch(nullptr);
  EC_CUDA(cudaDeviceSynchronize());
  plan_sets(true);
  alloc_sets();
  sync_set_remap();
  EC_CUDA(cudaDeviceSynchronize());  // (legacy-stream copies; the engine's streams do not wait for them)
  set_views();
  upload_tdev();
  select(cur);
  have_geom = false;  // per-batch descriptors are re-uploaded with the next geometry
  clear_graphs();
}

void Engine::upload_tdev() {
  std::vector<TableDev> all;
  for (int k = 0; k < kSets; ++k)
    for (uint32_t t = 0; t < T; ++t) {
      TableDev d = td_host[t];
      d.hash += k * hash_off[T];  // each set has its own dedup set and counters
      d.idcnt += k * hash_off[T];
      all.push_back(d);
    }
  EC_CUDA(cudaMemcpy(tdev_buf.p, all.data(), all.size() * sizeof(TableDev), cudaMemcpyHostToDevice));
}

void Engine::select(int i) {
  cur = i;
  tdev = View<TableDev>{tdev_buf.p + static_cast<size_t>(i) * T, T};
  BatchBufs& b = bb[i];
  slot_of = view(b.slot_of);
  inv = view(b.inv);
  uniq = view(b.uniq);
  uslot = view(b.uslot);
  missq = view(b.missq);
  usrc = view(b.usrc);
  utab = view(b.utab);
  urows = view(b.urows);
  ugrad = view(b.ugrad);
  g64 = view(b.g64);
  ucount = view(b.ucount);
  status = view(b.status);
  tstat = view(b.tstat);
  ctr = view(b.ctr);
  cnt = view(b.cnt);
  off = view(b.off);
  part = view(b.part);
  list = view(b.list);
}

uint64_t Engine::device_bytes() const {
  uint64_t sets = 0;
  for (const BatchBufs& b : bb) sets += b.bytes();
  return store_dev.bytes() + remap.bytes() + hash.bytes() + idcnt.bytes() + cache.bytes() + sets + tiles.bytes() + stiles.bytes() + cache_ids.bytes() + cache_tab.bytes() +
         exch_bytes();
}

void Engine::init_synthetic(uint64_t seed, float scale, cudaStream_t st) {
  use_device(device);
  join_host_writes(st);
  drop_prefetch(st);  // prefetched batches hold copies of the old rows
  ++geom_version;
  for (uint32_t t = 0; t < T; ++t) {
    if (!local_rows[t]) continue;
    const uint64_t n = local_rows[t] * D;
    const int grid = static_cast<int>(std::min<uint64_t>((n + 255) / 256, persistent_grid(device) * 4ull));
    k_init_shard<<<grid, 256, 0, st>>>(store_base + store_off[t] * D, local_rows[t], t, D, rank, world, seed, scale);
    EC_LAUNCH();
  }
  synth_seed = seed;
  synth_scale = scale;
  synth_valid = true;
  rows_trained = false;
  if (cache_k_total) fill_cache(st, /*from_store=*/world == 1);
}

void Engine::fill_cache(cudaStream_t st, bool from_store) {
  if (!cache_k_total) return;
  if (!from_store && !synth_valid)
    invalid("multi-rank cache placement needs ec_tables_init_synthetic first (rows of other shards are not local)");
  const uint64_t n = cache_k_total * D;
  const int grid = static_cast<int>(std::min<uint64_t>((n + 255) / 256, persistent_grid(device) * 4ull));
  // (re)initialised tables: every row is its synthetic value, shards included
  k_fill_cache<<<grid, 256, 0, st>>>(cache.p, cache_ids.p, cache_tab.p, cache_k_total, tdev.p, D, nullptr, nullptr,
                                     nullptr, nullptr, nullptr, T, 1, synth_seed, synth_scale,
                                     from_store ? rank : -1, world, nullptr);
  EC_LAUNCH();
}

void Engine::place_cache(const uint32_t* const* ids, const uint64_t* k) {
  use_device(device);
  EC_CUDA(cudaDeviceSynchronize());  // deferred host-tier write-backs land first
  // host-side validation + first-occurrence dedup of each table's list
  std::vector<uint32_t> all_ids;
  std::vector<uint16_t> all_tab;
  std::vector<uint64_t> koff(T + 1, 0);
  for (uint32_t t = 0; t < T; ++t) {
    std::vector<uint8_t> seen;
    const uint64_t kt = k ? k[t] : 0;
    if (kt && (!ids || !ids[t])) invalid("null cache id list for table " + std::to_string(t));
    if (kt > rows[t]) invalid("table " + std::to_string(t) + ": cache larger than the table");
    if (kt) seen.assign(rows[t], 0);
    for (uint64_t j = 0; j < kt; ++j) {
      const uint32_t id = ids[t][j];
      if (id >= rows[t])
        invalid("cache id " + std::to_string(id) + " out of range [0, " + std::to_string(rows[t]) + ")");
      if (seen[id]) continue;  // duplicates count once (cost_model.hpp:59-61)
      seen[id] = 1;
      all_ids.push_back(id);
      all_tab.push_back(static_cast<uint16_t>(t));
    }
    koff[t + 1] = all_ids.size();
  }
  if (all_ids.size() > 0x7FFFFFFFull) invalid("cache larger than 2^31 rows");
  // pending prefetches hold cache-slot numbers and row copies of the old
  // placement: drop them (and their graphs) before anything changes
  drop_prefetch(nullptr);
  ++geom_version;
  clear_graphs();
  EC_CUDA(cudaDeviceSynchronize());
  const uint64_t K = all_ids.size();
  DevBuf<float> ncache(K * D);
  DevBuf<uint32_t> nids(K);
  DevBuf<uint16_t> ntab(K);
  DevBuf<int> derr(1);
  EC_CUDA(cudaMemset(derr.p, 0, sizeof(int)));
  if (K) {
    EC_CUDA(cudaMemcpy(nids.p, all_ids.data(), K * sizeof(uint32_t), cudaMemcpyHostToDevice));
    EC_CUDA(cudaMemcpy(ntab.p, all_tab.data(), K * sizeof(uint16_t), cudaMemcpyHostToDevice));
    // new rows from the old replica, the own shard, a peer's shard, or the
    // synthetic init while nothing has been trained (remap is still the old one)
    DevBuf<int64_t> roff(T);
    EC_CUDA(cudaMemcpy(roff.p, remap_off.data(), T * sizeof(int64_t), cudaMemcpyHostToDevice));
    const int grid = static_cast<int>(std::min<uint64_t>((K * D + 255) / 256, persistent_grid(device) * 4ull));
    k_fill_cache<<<grid, 256>>>(ncache.p, nids.p, ntab.p, K, tdev.p, D, cache.p, cache_k_total ? remap.p : nullptr,
                                roff.p, p2p_peers(), p2p_shard_off(), T, synth_valid && !rows_trained ? 1 : 0,
                                synth_seed, synth_scale, rank, world, derr.p);
    EC_LAUNCH();
    EC_CUDA(cudaDeviceSynchronize());
    int e = 0;
    EC_CUDA(cudaMemcpy(&e, derr.p, sizeof(int), cudaMemcpyDeviceToHost));
    if (e)
      invalid(synth_valid ? "cache placement after training needs the peer-memory exchange: rows of other shards "
                            "are not readable from this rank"
                          : "multi-rank cache placement needs ec_tables_init_synthetic first (rows of other "
                            "shards are not local)");
  }
  // write the old cache's owned rows back to the shard before dropping it
  if (cache_k_total) {
    const uint64_t n = cache_k_total * D;
    const int grid = static_cast<int>(std::min<uint64_t>((n + 255) / 256, persistent_grid(device) * 4ull));
    k_flush_cache<<<grid, 256>>>(cache.p, cache_ids.p, cache_tab.p, cache_k_total, tdev.p, D, rank, world);
    EC_LAUNCH();
  }
  EC_CUDA(cudaMemset(remap.p, 0xFF, remap.bytes()));
  cache_k_total = K;
  cache_k.resize(T);
  for (uint32_t t = 0; t < T; ++t) cache_k[t] = koff[t + 1] - koff[t];
  std::swap(cache.p, ncache.p);
  std::swap(cache.n, ncache.n);
  std::swap(cache_ids.p, nids.p);
  std::swap(cache_ids.n, nids.n);
  std::swap(cache_tab.p, ntab.p);
  std::swap(cache_tab.n, ntab.n);
  for (uint32_t t = 0; t < T; ++t) {
    const uint64_t kt = koff[t + 1] - koff[t];
    if (!kt) continue;
    k_set_remap<<<static_cast<int>(std::min<uint64_t>((kt + 255) / 256, 4096)), 256>>>(
        remap.p + remap_off[t], cache_ids.p + koff[t], kt, static_cast<int64_t>(koff[t]));
    EC_LAUNCH();
  }
  sync_set_remap();
  EC_CUDA(cudaDeviceSynchronize());
}

// Direct-mapped dedup sets carry a copy of `remap` beside every id's set word
// (odd words), in every buffer set: refreshed whenever remap or the sets change.
void Engine::sync_set_remap() {
  for (int k = 0; k < kSets; ++k)
    for (uint32_t t = 0; t < T; ++t) {
      if (!hash_direct[t] || !rows[t]) continue;
      const int grid = static_cast<int>(std::min<uint64_t>((rows[t] + 255) / 256, persistent_grid(device) * 4ull));
      k_copy_remap<<<grid, 256>>>(hash.p + k * hash_off[T] + hash_off[t], remap.p + remap_off[t], rows[t]);
      EC_LAUNCH();
    }
}

void Engine::rw_rows(uint32_t t, const uint32_t* ids, uint64_t n, float* buf_host, bool write) {
  if (t >= T) invalid("table index out of range");
  use_device(device);
  if (!n) return;
  DevBuf<uint32_t> dids(n);
  DevBuf<float> dbuf(n * D);
  DevBuf<int> derr(1);
  EC_CUDA(cudaMemset(derr.p, 0, sizeof(int)));
  EC_CUDA(cudaMemcpy(dids.p, ids, n * sizeof(uint32_t), cudaMemcpyHostToDevice));
  if (write) EC_CUDA(cudaMemcpy(dbuf.p, buf_host, n * D * sizeof(float), cudaMemcpyHostToDevice));
  const int grid = static_cast<int>(std::min<uint64_t>((n * D + 255) / 256, 4096));
  if (write) {
    drop_prefetch(nullptr);  // prefetched batches may hold copies of these rows
    ++geom_version;
    rows_trained = true;
  }
  EC_CUDA(cudaDeviceSynchronize());
  k_rw_rows<<<grid, 256>>>(tdev.p, t, dids.p, n, D, cache.p, dbuf.p, write ? 1 : 0, rank, world, derr.p);
  EC_LAUNCH();
  EC_CUDA(cudaDeviceSynchronize());
  int e = 0;
  EC_CUDA(cudaMemcpy(&e, derr.p, sizeof(int), cudaMemcpyDeviceToHost));
  if (e == 1) invalid("row id out of range for table " + std::to_string(t));
  if (e == 2) invalid("row not held by this rank (neither cached nor owned)");
  if (!write) EC_CUDA(cudaMemcpy(buf_host, dbuf.p, n * D * sizeof(float), cudaMemcpyDeviceToHost));
}

// Per-batch geometry (uploaded only on change): dedup tiles never straddle
// tables; each tile knows which tables' ubase it publishes; scatter tiles are
// runs of bags of one table.
void Engine::set_geometry(const ec_batch& b, cudaStream_t st) {
  bool same = have_geom && b.batch_size == geom_b && b.pooling == geom_p && (b.bag_offsets_dev == nullptr) == geom_fixed;
  for (uint32_t t = 0; same && t <= T; ++t) same = geom_off[t] == b.table_offsets_host[t];
  if (same) return;
  drop_prefetch(st);
  clear_graphs();
  ++geom_version;
  geom_off.assign(b.table_offsets_host, b.table_offsets_host + T + 1);
  std::vector<Tile> tl;
  std::vector<int> ft(T + 1);
  for (uint32_t t = 0; t < T; ++t) {
    const int64_t lo = geom_off[t], n = geom_off[t + 1] - geom_off[t];
    ft[t] = static_cast<int>(tl.size());
    for (int64_t s = 0; s < n; s += kTile)
      tl.push_back(Tile{t, static_cast<uint32_t>(std::min<int64_t>(kTile, n - s)), lo + s, 0, 0});
    td_host[t].base = lo;
    td_host[t].n = n;
  }
  ntiles = static_cast<int>(tl.size());
  int64_t nmax = 0;
  for (uint32_t t = 0; t < T; ++t) nmax = std::max<int64_t>(nmax, geom_off[t + 1] - geom_off[t]);
  max_n_batch = nmax;
  // The cluster kernel wins when the tables alone fill the GPU (one cluster
  // of 8 CTAs per table); larger per-table batches need more items per thread.
  cluster_fits = nmax <= static_cast<int64_t>(kClusterCtas) * kClusterThreads * kClusterMaxItems;
  for (uint32_t t = 0; t < T; ++t) cluster_fits = cluster_fits && td_host[t].direct;
  table_fits = cluster_fits && nmax <= static_cast<int64_t>(kTableThreads) * kTableMaxItems;
  cluster_ok = cluster_fits && static_cast<int64_t>(T) * kClusterCtas >= sm_count(device) &&
               nmax <= static_cast<int64_t>(kClusterCtas) * kClusterThreads * 8;
  cluster_items = 1;
  while (static_cast<int64_t>(kClusterCtas) * kClusterThreads * cluster_items < nmax) cluster_items *= 2;
  tail_lo = static_cast<int>(T);
  for (int t = static_cast<int>(T) - 1; t >= 0 && ft[t] == ntiles; --t) tail_lo = t;  // trailing empty tables
  for (uint32_t t = 0; t < static_cast<uint32_t>(tail_lo); ++t) {
    Tile& x = tl[ft[t]];
    if (x.ub_hi == 0) x.ub_lo = t;
    x.ub_hi = t + 1;
  }
  // scatter tiles: ~kTile lookups of one table each (bag count for fixed
  // pooling; 256 bags for CSR)
  std::vector<int4> sc;
  const int per = b.bag_offsets_dev ? 256 : static_cast<int>(std::max<int64_t>(1, kTile / std::max<uint32_t>(1, b.pooling)));
  for (uint32_t t = 0; t < T; ++t) {
    if (geom_off[t + 1] == geom_off[t]) continue;
    for (int s0 = 0; s0 < static_cast<int>(b.batch_size); s0 += per)
      sc.push_back(make_int4(static_cast<int>(t), s0, std::min<int>(b.batch_size, s0 + per), 0));
  }
  nstiles = static_cast<int>(sc.size());
  EC_CUDA(cudaStreamSynchronize(st));
  if (ntiles) EC_CUDA(cudaMemcpy(tiles.p, tl.data(), tl.size() * sizeof(Tile), cudaMemcpyHostToDevice));
  for (BatchBufs& bs : bb)
    if (bs.status.n < static_cast<size_t>(ntiles) + 1) bs.status.alloc(ntiles + 1);
  select(cur);
  if (stiles.n < sc.size()) stiles.alloc(sc.size());
  if (nstiles) EC_CUDA(cudaMemcpy(stiles.p, sc.data(), sc.size() * sizeof(int4), cudaMemcpyHostToDevice));
  upload_tdev();
  geom_b = b.batch_size;
  geom_p = b.pooling;
  geom_fixed = b.bag_offsets_dev == nullptr;
  have_geom = true;
}


// K3 for rows this rank holds: pinned-host misses on the side stream, cache
// hits and local-HBM misses on the main stream.
template <int VEC>
void Engine::fwd_gather_local(cudaStream_t st) {
  const int grid = row_grid();
  if (storage == EC_STORAGE_HOST && !consuming_prefetch) {
    // host misses on the side stream, overlapping the HBM hit gather
    EC_CUDA(cudaEventRecord(ev_part, st));
    EC_CUDA(cudaStreamWaitEvent(side, ev_part, 0));
    // few CTAs: the host link, not the SMs, bounds this kernel, and a full
    // persistent grid would hold every SM slot while it waits on PCIe reads
    launch_gather_host<VEC>(side);
    EC_CUDA(cudaEventRecord(ev_side, side));
  }
  if (fused()) return;  // the pool reads cached / HBM rows where they are
  PhaseScope ph(prof, kPhaseGather, st);
  // rows in flight per lane group: 2 for single-rank pooling-1 batches (TB
  // shape 0.395 -> 0.3855 ms), else 4 (cfg1, P=20: 0.191 at 4, 0.208 at 2)
  if (world == 1 && geom_p == 1 && !bag_off)
    k_gather<VEC, 2><<<grid, kThreads, 0, st>>>(tdev.p, T, ctr.p, uniq.p, utab.p, uslot.p, usrc.p, cache.p, urows.p,
                                                ugrad.p, cnt.p, storage == EC_STORAGE_HBM ? 1 : 0, rank, world);
  else
    k_gather<VEC, 4><<<grid, kThreads, 0, st>>>(tdev.p, T, ctr.p, uniq.p, utab.p, uslot.p, usrc.p, cache.p, urows.p,
                                                ugrad.p, cnt.p, storage == EC_STORAGE_HBM ? 1 : 0, rank, world,
                                                p2p_peers(), p2p_shard_off());
  launched();
}

// K5 once every unique row is present (side stream joined).
template <int VEC>
void Engine::fwd_pool(cudaStream_t st) {
  if (storage == EC_STORAGE_HOST && !consuming_prefetch) EC_CUDA(cudaStreamWaitEvent(st, ev_side, 0));
  PhaseScope ph(prof, kPhasePool, st);
  if (fused()) {
    // rows read at their source; trailing blocks empty this batch's dedup set
    const RowSrc rs{usrc.p, uniq.p, cache.p, urows.p, storage == EC_STORAGE_HBM ? 1 : 0,
                    bb[cur].row_sources ? reinterpret_cast<const int32_t*>(slot_of.p) : nullptr};
    const ResetOut ro{ctr.p, utab.p, uslot.p, usrc.p, ugrad.p, cnt.p,
                      !bb[cur].counted ? kResetAll : storage == EC_STORAGE_HOST ? kResetMisses : kResetNone};
    const int pb = row_grid(), rb = sm_count(device);
    // 4 bags in flight per thread (measured, Kaggle: HBM tier 0.0647 -> 0.0615
    // ms vs 8; host tier, with 4 row CTAs per SM, 0.1007-0.1014 -> 0.0984-0.0995)
    const bool rsrc = bb[cur].row_sources;
    if (!bag_off && geom_p == 1)
      (rsrc ? k_pool1<VEC, kFusedPoolR, true, true> : k_pool1<VEC, kFusedPoolR, true, false>)<<<pb + rb, kThreads, 0, st>>>(
          tdev.p, T, static_cast<int>(geom_b), inv.p, urows.p, out_ptr, rs, pb, ro);
    else
      (rsrc ? k_pool<VEC, 4, true, true> : k_pool<VEC, 4, true, false>)<<<pb + rb, kThreads, 0, st>>>(
          tdev.p, T, static_cast<int>(geom_b), static_cast<int>(geom_p), bag_off, inv.p, urows.p, out_ptr, rs, pb, ro);
    launched();
    return;
  }
  if (!bag_off && geom_p == 1) {
    k_pool1<VEC, 8><<<row_grid(), kThreads, 0, st>>>(tdev.p, T, static_cast<int>(geom_b), inv.p, urows.p, out_ptr);
  } else {
    // 2 bags of P lookups in flight per thread (cfg1, P=20: 0.1924-0.1937 ms at 4, 0.1910-0.1913 at 2, 0.232 at 8)
    k_pool<VEC, 2><<<row_grid(), kThreads, 0, st>>>(tdev.p, T, static_cast<int>(geom_b), static_cast<int>(geom_p),
                                                    bag_off, inv.p, urows.p, out_ptr);
  }
  launched();
}

template <int VEC>
void Engine::bwd_scatter(const float* grad, cudaStream_t st) {
  PhaseScope ph(prof, kPhaseScatter, st);
  fold_g64 = false;
  direct_apply = false;
  if (fused()) {
    // -lr * grad scattered straight into the cache / HBM rows (SGD in the
    // scatter) for a row's first kLightAdds partials, the rest summed in fp64
    // (g64) for k_apply_g64; pinned-host misses accumulate in ugrad
    const RowSrc rs{usrc.p, uniq.p, cache.p, urows.p, storage == EC_STORAGE_HBM ? 1 : 0};
    k_scatter<VEC, kFusedScatterR, true><<<row_grid(), kThreads, 0, st>>>(tdev.p, T, static_cast<int>(geom_b), static_cast<int>(geom_p),
                                                             bag_off, inv.p, grad, ugrad.p, g64.p,
                                                             bb[cur].counted ? ucount.p : nullptr, ctr.p, rs, bwd_lr);
    launched();
    return;
  }
  // ugrad rows and occurrence counts were zeroed by k_gather
  // auto: the transpose pays off when tables see many lookups per batch (hot
  // rows repeat thousands of times); measured: 26 x 65536 lookups 418 -> 175 us,
  // 8 x 81920 91 -> 84 us, but 26 x 16384 30 -> 53 us
  const bool atomic = scatter_mode == 1 || (scatter_mode == 0 && max_n_batch < 32768);
  if (atomic) {
    k_scatter<VEC, 4><<<row_grid(), kThreads, 0, st>>>(tdev.p, T, static_cast<int>(geom_b), static_cast<int>(geom_p),
                                                       bag_off, inv.p, grad, ugrad.p, g64.p,
                                                       bb[cur].counted ? ucount.p : nullptr, ctr.p);
    launched();
    k_g64_finalize<VEC><<<row_grid(), kThreads, 0, st>>>(nullptr, bb[cur].counted ? ucount.p : nullptr, ctr.p,
                                                         static_cast<int>(T), ugrad.p, g64.p);
    launched();
    return;
  }
  if (!ntiles) return;
  // single rank, HBM rows: k_apply is ugrad's only consumer, so runs inside one
  // chunk are applied by k_bwd_reduce itself (TB shape: k_apply 76 -> see DESIGN)
  const DirectApply ap = world == 1 && !in_group && storage == EC_STORAGE_HBM
                             ? DirectApply{urows.p, usrc.p, uniq.p, utab.p, tdev.p, cache.p, bwd_lr}
                             : DirectApply{};
  direct_apply = ap.urows != nullptr;
  if (bb[cur].lists) {  // the forward grouped the lookups already (tile path)
    k_bwd_reduce<VEC><<<row_grid(), kThreads, 0, st>>>(off.p, ctr.p, static_cast<int>(T), list.p, grad, ugrad.p, g64.p,
                                                       ap);
    launched();
    finalize_transpose<VEC>(st);
    return;
  }
  const int tgrid = std::min(ntiles, sm_count(device) * 8);
  k_bwd_count<<<tgrid, kThreads, 0, st>>>(tiles.p, ntiles, inv.p, cnt.p);
  launched();
  const int nparts = static_cast<int>((max_n * T + kScanTile) / kScanTile);
  k_uscan_reduce<<<nparts, kScanThreads, 0, st>>>(cnt.p, ctr.p, static_cast<int>(T), part.p);
  launched();
  k_scan_partials<<<1, 1024, 0, st>>>(part.p, nparts, nullptr);
  launched();
  k_uscan_apply<<<nparts, kScanThreads, 0, st>>>(cnt.p, ctr.p, static_cast<int>(T), part.p, off.p);
  launched();
  k_bwd_fill<<<tgrid, kThreads, 0, st>>>(tiles.p, ntiles, tdev.p, bag_off, static_cast<int>(T), static_cast<int>(geom_b),
                                         static_cast<int>(geom_p), inv.p, off.p, cnt.p, list.p);
  launched();
  k_bwd_reduce<VEC><<<row_grid(), kThreads, 0, st>>>(off.p, ctr.p, static_cast<int>(T), list.p, grad, ugrad.p, g64.p,
                                                     ap);
  launched();
  finalize_transpose<VEC>(st);
}

// Rows spanning many k_bwd_reduce chunks have their gradient in g64: rounded
// into ugrad for the exchange / host write-back, or -- single rank, HBM rows,
// where k_apply is the only consumer -- read by k_apply itself.
template <int VEC>
void Engine::finalize_transpose(cudaStream_t st) {
  fold_g64 = world == 1 && !in_group && storage == EC_STORAGE_HBM;
  if (fold_g64) return;
  k_g64_finalize<VEC><<<row_grid(), kThreads, 0, st>>>(off.p, nullptr, ctr.p, static_cast<int>(T), ugrad.p, g64.p);
  launched();
}

// K6b for rows this rank applies itself: misses it owns (HBM, or pinned host
// on the side stream) and — single rank only — cache hits.  With world > 1
// the replicated hot rows are updated by the rank-ordered exchange instead.
// Cold rows written back over the host link on side2 (full duplex with the
// host reads of a prefetched batch), and the prefetched batch's copies of rows
// updated here refreshed on the side stream (after its host gather, FIFO on
// `side`).  Both start at ev_grad (gradients complete).  Never captured.
template <int VEC>
void Engine::enqueue_host_writeback(float lr) {
  EC_CUDA(cudaStreamWaitEvent(side2, ev_grad, 0));
  // the next batch's copies of host rows, if its gather already ran
  const int h = head_pending();
  const bool patch = h >= 0 && bb[h].gathered;
  const BatchBufs& nx = bb[patch ? h : cur];
  const TableDev* nxt_td = tdev_buf.p + static_cast<size_t>(patch ? h : cur) * T;
  // fused path: heavy misses' gradients are read from the fp64 sums (miss_sgd)
  const double* sums = fused() && bb[cur].counted ? g64.p : nullptr;
  const int* cnts = sums ? ucount.p : nullptr;
  if (patch && host_tma()) {
    // one kernel writes the rows back and refreshes the prefetched batch's
    // copies: it starts once that batch's host gather is done (host reads and
    // writes share the link's request rate, so the wait costs no link time)
    EC_CUDA(cudaStreamWaitEvent(side2, nx.ev_pf, 0));
    PhaseScope ph(prof, kPhaseApplyHost, side2);
    k_apply_host_tma<VEC><<<host_write_grid(), kThreads, 0, side2>>>(tdev.p, T, ctr.p, missq.p, uniq.p, utab.p, urows.p,
                                                                      ugrad.p, lr, rank, world, nxt_td, nx.usrc.p,
                                                                      nx.urows.p, sums, cnts);
    launched();
    EC_CUDA(cudaEventRecord(ev_side2, side2));
    EC_CUDA(cudaEventRecord(ev_patch, side2));
    return;
  }
  {
    PhaseScope ph(prof, kPhaseApplyHost, side2);
    if (host_tma())
      k_apply_host_tma<VEC><<<host_write_grid(), kThreads, 0, side2>>>(tdev.p, T, ctr.p, missq.p, uniq.p, utab.p,
                                                                        urows.p, ugrad.p, lr, rank, world, nullptr,
                                                                        nullptr, nullptr, sums, cnts);
    else
      k_apply_host<VEC, kHostR><<<host_write_grid(), kThreads, 0, side2>>>(tdev.p, T, ctr.p, missq.p, uniq.p, utab.p,
                                                                       urows.p, ugrad.p, lr, rank, world, sums, cnts);
    launched();
  }
  EC_CUDA(cudaEventRecord(ev_side2, side2));
  if (patch) {
    EC_CUDA(cudaStreamWaitEvent(side, ev_grad, 0));
    EC_CUDA(cudaStreamWaitEvent(side, nx.ev_pf, 0));
    // (the prefetched ids are found in the pending set's hash)
    k_patch_prefetch<VEC, 4><<<sm_count(device), kThreads, 0, side>>>(nxt_td, T, ctr.p, missq.p, uniq.p, utab.p, urows.p,
                                                                      ugrad.p, lr, rank, world, nx.usrc.p, nx.urows.p,
                                                                      sums, cnts);
    launched();
    EC_CUDA(cudaEventRecord(ev_patch, side));
  }
}

// Work a caller's stream must see before reusing the current set or the host
// tier: the deferred write-back and prefetch patch (single rank, host tier).
void Engine::join_host_writes(cudaStream_t st) {
  if (storage != EC_STORAGE_HOST) return;
  EC_CUDA(cudaStreamWaitEvent(st, ev_side2, 0));
  EC_CUDA(cudaStreamWaitEvent(st, ev_patch, 0));
}

// K6b for rows this rank applies itself: misses it owns (HBM, or pinned host
// via enqueue_host_writeback) and — single rank only — cache hits.  With
// world > 1 the replicated hot rows are updated by the rank-ordered exchange
// instead, and the host write-back is joined before it.
template <int VEC>
void Engine::bwd_apply_local(float lr, cudaStream_t st) {
  const bool host = storage == EC_STORAGE_HOST;
  // fused host tier: with counts the write-back reads heavy misses' fp64 sums
  // itself (miss_sgd), so it starts at ev_grad right after the scatter and
  // overlaps k_apply_g64 (k_clear_miss_sums clears the sums before the set's
  // next dedup); without counts every miss's sum is folded into ugrad first
  if (fused() && host && !bb[cur].counted) {
    PhaseScope ph(prof, kPhaseApply, st);
    k_g64_misses<VEC><<<sm_count(device), kThreads, 0, st>>>(static_cast<int>(T), ctr.p, missq.p, nullptr, ugrad.p,
                                                             g64.p);
    launched();
  }
  if (host) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    EC_CUDA(cudaStreamIsCapturing(st, &cs));
    // inside a captured backward the record becomes an external event node,
    // so the uncaptured write-back launched after the replay starts right here
    if (cs == cudaStreamCaptureStatusActive)
      EC_CUDA(cudaEventRecordWithFlags(ev_grad, st, cudaEventRecordExternal));
    else
      EC_CUDA(cudaEventRecord(ev_grad, st));
    if (world > 1) enqueue_host_writeback<VEC>(lr);
  }
  if (fused()) {
    // w - lr * sum(g) per cache / HBM row (one rounding for heavy rows)
    PhaseScope ph(prof, kPhaseApply, st);
    k_apply_g64<VEC><<<row_grid(), kThreads, 0, st>>>(tdev.p, T, ctr.p, uniq.p, utab.p, usrc.p,
                                                      bb[cur].counted ? ucount.p : nullptr, cache.p, ugrad.p, g64.p, lr,
                                                      host ? 0 : 1);
    launched();
  }
  if (!fused()) {
    PhaseScope ph(prof, kPhaseApply, st);
    k_apply<VEC, 4><<<row_grid(), kThreads, 0, st>>>(tdev.p, T, ctr.p, uniq.p, utab.p, usrc.p, urows.p, ugrad.p, lr,
                                                     cache.p, world == 1 ? 1 : 0, host ? 0 : 1, rank, world,
                                                     fold_g64 ? off.p : nullptr, g64.p, direct_apply ? 1 : 0);
    launched();
  }
  if (host && world > 1) join_host_writes(st);
}


void Engine::forward_prologue(const ec_batch& b, float* out, cudaStream_t st) {
  if (!b.table_offsets_host || !b.indices_dev) invalid("batch needs indices and table offsets");
  if (!out) invalid("null output");
  if (b.batch_size < 1 || b.batch_size > max_b) invalid("batch_size out of [1, max_batch_size]");
  if (b.table_offsets_host[0] != 0) invalid("table_offsets[0] must be 0");
  for (uint32_t t = 0; t < T; ++t) {
    const int64_t n = b.table_offsets_host[t + 1] - b.table_offsets_host[t];
    if (n < 0 || static_cast<uint64_t>(n) > max_n)
      invalid("table " + std::to_string(t) + ": lookups " + std::to_string(n) + " out of [0, max_lookups_per_table]");
    if (!b.bag_offsets_dev && n != static_cast<int64_t>(b.batch_size) * b.pooling)
      invalid("table " + std::to_string(t) + ": fixed pooling needs batch_size*pooling lookups");
  }
  if (b.table_offsets_host[T] >= (int64_t{1} << 31)) invalid("a batch holds at most 2^31-1 lookups");
  if (world > 1 && !comm_ready()) invalid("world > 1 needs ec_tables_attach_comm (or a loopback group)");
  use_device(device);
  set_geometry(b, st);
  bag_off = b.bag_offsets_dev;
  out_ptr = out;
}

int Engine::head_pending() const {
  int h = -1;
  for (int k = 0; k < kSets; ++k)
    if (bb[k].pending && (h < 0 || bb[k].seq < bb[h].seq)) h = k;
  return h;
}

int Engine::free_set() const {
  for (int k = 1; k < kSets; ++k) {
    const int s = (cur + k) % kSets;
    if (!bb[s].pending) return s;
  }
  return -1;
}

// Host-miss gather of a prefetched set whose dedup ran earlier (prefetch
// depth >= 2): on `side` once its dedup is done, every host write-back
// enqueued so far has landed -- so it reads current rows; only the backward
// still to come before its forward is patched in (enqueue_host_writeback) --
// and the caller's stream has reached this call (`gate`: the gather belongs to
// the step that starts here, not to the gap before it).
void Engine::launch_pending_gather(int s) {
  BatchBufs& b = bb[s];
  if (b.gathered) return;
  EC_CUDA(cudaStreamWaitEvent(side, ev_gate, 0));  // recorded by the forward at its start
  EC_CUDA(cudaStreamWaitEvent(side, b.ev_ded, 0));
  EC_CUDA(cudaStreamWaitEvent(side, ev_side2, 0));
  const int saved = cur;
  select(s);
  try {
    EC_DISPATCH_VEC(launch_gather_host, side);
  } catch (...) {
    select(saved);
    throw;
  }
  select(saved);
  EC_CUDA(cudaEventRecord(b.ev_pf, side));
  b.gathered = true;
}

void Engine::forward(const ec_batch& b, float* out, cudaStream_t st) {
  if (in_group) invalid("this rank belongs to a loopback group: use ec_group_lookup_fwd");
  forward_prologue(b, out, st);
  const int h = head_pending();
  if (h >= 0) {
    BatchBufs& nx = bb[h];
    if (nx.indices == b.indices_dev && nx.geom_version == geom_version && world > 1) {
      // peer exchange: only the dedup / hit-miss ran ahead; rows are read
      // once every rank applied the previous step
      nx.pending = false;
      EC_CUDA(cudaEventRecord(bb[cur].ev_free, st));
      select(h);
      EC_CUDA(cudaStreamWaitEvent(st, nx.rows_early ? nx.ev_pf : nx.ev_ded, 0));
      p2p_fwd_begin(st);
      if (nx.rows_early) p2p_patch_prefetched(st);  // rows the last step updated after the early read
      consuming_prefetch = nx.rows_early;
      try {
        gather_local(st);
        pool(st);
      } catch (...) {
        consuming_prefetch = false;
        throw;
      }
      consuming_prefetch = false;
      have_fwd = true;
      return;
    }
    if (nx.indices == b.indices_dev && nx.geom_version == geom_version) {
      // dedup, hit/miss and host-miss gather already ran (ec_lookup_prefetch)
      nx.pending = false;
      EC_CUDA(cudaEventRecord(ev_gate, st));  // this step starts here
      if (!nx.gathered) launch_pending_gather(h);  // (host tier, gather not started yet)
      // everything enqueued so far (the outgoing batch's backward and host-tier
      // joins) used the outgoing set: a prefetch may reuse it after this
      EC_CUDA(cudaEventRecord(bb[cur].ev_free, st));
      select(h);
      EC_CUDA(cudaStreamWaitEvent(st, nx.ev_pf, 0));
      if (storage == EC_STORAGE_HOST) EC_CUDA(cudaStreamWaitEvent(st, ev_patch, 0));
      consuming_prefetch = true;
      try {
        const GraphKey key{2, b.indices_dev, b.bag_offsets_dev, out, 0};
        run_maybe_graphed(key, st, [&] {
          gather_local(st);
          pool(st);
        });
      } catch (...) {
        consuming_prefetch = false;
        throw;
      }
      consuming_prefetch = false;
      // the next prefetched batch's host gather starts now: first on the host
      // link in this step, reading rows every earlier write-back has updated
      const int h2 = head_pending();
      if (h2 >= 0 && storage == EC_STORAGE_HOST) launch_pending_gather(h2);
      have_fwd = true;
      return;
    }
    drop_prefetch(st);
  }
  join_host_writes(st);  // this set's last write-back still reads its buffers
  if (world == 1) {
    const GraphKey key{0, b.indices_dev, b.bag_offsets_dev, out, 0};
    run_maybe_graphed(key, st, [&] { enqueue_forward(b.indices_dev, st); });
  } else if (p2p_on()) {
    p2p_fwd_begin(st);  // every rank applied the previous step
    enqueue_dedup_partition(b.indices_dev, st);
    gather_local(st);  // K4 fused: remote misses are loads from their owners' shards
    pool(st);          // (joins the host-row gather of the side stream)
  } else {
    enqueue_dedup_partition(b.indices_dev, st);
    gather_local(st);
    exchange_fwd(st);  // K4: remote misses fetched from their owners
    pool(st);
  }
  have_fwd = true;
}

// Start a later batch early (single rank; the current batch geometry): its
// dedup and hit/miss partition run on the prefetch stream into a free buffer
// set.  Pinned-host tier: the next batch in line also gathers its host misses
// right away; a batch further ahead (prefetch depth 2) gathers them when the
// forward before it starts, so the host link carries that gather first in the
// step.  Rows a backward writes to the host tier after a gather are patched
// into the gathered copy.  Up to kSets-1 batches may be pending; forwards
// consume them in prefetch order.
void Engine::prefetch(const ec_batch& b, cudaStream_t st) {
  if (in_group || (world > 1 && !p2p_on()))
    invalid("prefetch needs a single rank or the peer-memory exchange");
  if (!have_geom || !b.indices_dev || !b.table_offsets_host) invalid("prefetch needs a batch with the current geometry");
  bool same = b.batch_size == geom_b && b.pooling == geom_p && (b.bag_offsets_dev == nullptr) == geom_fixed &&
              b.bag_offsets_dev == bag_off;
  for (uint32_t t = 0; same && t <= T; ++t) same = geom_off[t] == b.table_offsets_host[t];
  if (!same) invalid("prefetch needs the geometry (offsets, batch size, pooling, bag offsets) of the last forward");
  use_device(device);
  const int s = free_set();
  if (s < 0) invalid("prefetch: " + std::to_string(kSets - 1) + " batches already pending (consume one first)");
  const bool next_in_line = head_pending() < 0;
  // the set (own hash, emptied by its last pool/gather) is free once its last
  // batch's main-stream work and host-tier write-back have run
  EC_CUDA(cudaStreamWaitEvent(pstream, bb[s].ev_free, 0));
  join_host_writes(pstream);
  // stream-ordered like every call: work the caller enqueued on `st` before
  // this prefetch (e.g. the copy that produced these indices) comes first
  EC_CUDA(cudaEventRecord(ev_pfcall, st));
  EC_CUDA(cudaStreamWaitEvent(pstream, ev_pfcall, 0));
  // A prefetched dedup launched together with the forward's pool competes with
  // it for SM slots (the cluster kernel needs 8 co-resident CTAs per table);
  // started ~10 us later it runs beside the pool's tail and the scatter.
  // Measured (interleaved A/B on three boxes): HBM tier 0.053 ->
  // 0.049 ms, configs[3] uniform 0.066 -> 0.055, host tier / TB / cfg1 within
  // noise; 20 us about the same, 30 us worse (HBM 0.060); waiting for the
  // pool's end worse still (HBM 0.074: the dedup then sits on the next
  // forward's path).  EC_PF_DELAY_NS overrides (0: off).
  // Default 10 us for the pinned-host tier, 20 us with HBM rows (re-measured
  // after k_clear_miss_sums, which runs just before the dedup, became 12 -> 8
  // us: HBM tier 0.0529 at 10 vs 0.0490 at 20; configs[3] uniform 0.0622 vs
  // 0.0540; host tier 0.0979 at 10 vs 0.0995 at 20).
  static const int env_delay = [] {
    const char* v = std::getenv("EC_PF_DELAY_NS");
    return v && *v ? std::atoi(v) : -1;
  }();
  // The tile path (TB, cfg1) gains a little more at 40 us (TB 0.368 / 0.360 /
  // 0.354 / 0.353 ms at 0 / 20 / 40 / 80 us, cfg1 0.178 / 0.180 / 0.173 /
  // 0.183), but the later dedup chain then overlaps K3: k_gather falls from
  // 0.56 to 0.36 of the HBM roofline (north star: >= 0.5), so it stays at 20.
  const int delay_ns = env_delay >= 0 ? env_delay : storage == EC_STORAGE_HBM ? 20000 : 10000;
  if (delay_ns > 0 && have_fwd) {
    k_spin_ns<<<1, 32, 0, pstream>>>(static_cast<unsigned>(delay_ns));
    launched();
  }
  // peer exchange: rows are read once the forward in flight passed its step
  // barrier (every update of the step before is in), and the ones this step
  // updates are patched after the next barrier (p2p_patch_prefetched)
  const bool gather_now = storage == EC_STORAGE_HOST && next_in_line;
  if (gather_now && world > 1) EC_CUDA(cudaStreamWaitEvent(pstream, ev_b1, 0));
  const int saved = cur;
  select(s);
  try {
    // dedup + hit/miss (+ the host-miss gather when next in line), in stream
    // order on pstream: one graph launch per prefetch
    const GraphKey key{gather_now ? 4 : 5, b.indices_dev, b.bag_offsets_dev, nullptr, 0};
    run_maybe_graphed(key, pstream, [&] {
      enqueue_dedup_partition(b.indices_dev, pstream);
      if (gather_now) EC_DISPATCH_VEC(launch_gather_host, pstream);
    });
    EC_CUDA(cudaEventRecord(bb[s].ev_ded, pstream));
    EC_CUDA(cudaEventRecord(bb[s].ev_pf, pstream));
  } catch (...) {
    select(saved);
    throw;
  }
  BatchBufs& nb = bb[s];
  nb.pending = true;
  nb.gathered = storage != EC_STORAGE_HOST || gather_now || world > 1;
  nb.rows_early = world > 1 && gather_now;
  nb.seq = ++pf_seq;
  nb.indices = b.indices_dev;
  nb.geom_version = geom_version;
  select(saved);
}

// Drop every pending prefetch (a forward of another batch, a new geometry).
void Engine::drop_prefetch(cudaStream_t st) {
  for (int k = 0; k < kSets; ++k) {
    BatchBufs& nx = bb[k];
    if (!nx.pending) continue;
    EC_CUDA(cudaStreamWaitEvent(st, nx.gathered ? nx.ev_pf : nx.ev_ded, 0));
    join_host_writes(st);
    k_clear_hash<<<sm_count(device) * 2, 256, 0, st>>>(tdev_buf.p + static_cast<size_t>(k) * T, T, nx.ctr.p, nx.utab.p,
                                                        nx.uslot.p);
    launched();
    EC_CUDA(cudaEventRecord(nx.ev_free, st));  // the set is free again
    nx.pending = false;
    nx.gathered = false;
  }
}

template <int VEC>
void Engine::launch_gather_host(cudaStream_t s) {
  PhaseScope ph(prof, kPhaseGatherHost, s);
  const bool tma = host_tma();
  if (tma && !p2p_on())
    k_gather_host_tma<VEC><<<host_grid(), kThreads, 0, s>>>(tdev.p, T, ctr.p, missq.p, uniq.p, utab.p, urows.p, rank,
                                                             world);
  else  // (peer exchange: remote owners' rows from their shared host shards, over this GPU's link)
    k_gather_host<VEC, kHostR><<<host_grid(), kThreads, 0, s>>>(tdev.p, T, ctr.p, missq.p, uniq.p, utab.p, urows.p, rank,
                                                            world, p2p_peers(), p2p_shard_off());
  launched();
}

void Engine::gather_local(cudaStream_t st) { EC_DISPATCH_VEC(fwd_gather_local, st); }
void Engine::scatter_grads(const float* grad, cudaStream_t st) {
  use_device(device);
  EC_DISPATCH_VEC(bwd_scatter, grad, st);
}

// Debug/parity export on the fused path: copy the current batch's cached and
// HBM rows into the compact buffer as K3 would (pinned-host misses are there
// already).  Harmless for the backward: ugrad rows and counters it zeroes are
// zero at this point, and the dedup set was already emptied by the pool.
template <int VEC>
void Engine::export_gather() {
  EC_CUDA(cudaDeviceSynchronize());
  k_gather<VEC, 4><<<row_grid(), kThreads>>>(tdev.p, T, ctr.p, uniq.p, utab.p, uslot.p, usrc.p, cache.p, urows.p,
                                             ugrad.p, cnt.p, storage == EC_STORAGE_HBM ? 1 : 0, rank, world);
  EC_LAUNCH();
  EC_CUDA(cudaDeviceSynchronize());
}
void Engine::gather_for_export() { EC_DISPATCH_VEC(export_gather); }
void Engine::pool(cudaStream_t st) { EC_DISPATCH_VEC(fwd_pool, st); }
void Engine::scatter_and_apply_local(const float* grad, float lr, cudaStream_t st) {
  if (!grad) invalid("null gradient");
  use_device(device);
  bwd_lr = lr;
  EC_DISPATCH_VEC(bwd_scatter, grad, st);
  EC_DISPATCH_VEC(bwd_apply_local, lr, st);
}

// Replay a captured CUDA graph of the per-batch kernel sequence when the
// stream allows it (launch gaps dominate these short kernels); capture on
// first use of a (kind, pointers) key.  Profiling, the legacy stream, an
// outer capture and the multi-rank exchange (host syncs) launch directly.
template <class F>
void Engine::run_maybe_graphed(const GraphKey& key, cudaStream_t st, F&& enqueue) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  bool direct = !use_graphs || prof.on || world > 1 || st == nullptr || st == cudaStreamLegacy ||
                st == cudaStreamPerThread;
  if (!direct) {
    EC_CUDA(cudaStreamIsCapturing(st, &cs));
    direct = cs != cudaStreamCaptureStatusNone;
  }
  if (direct) {
    enqueue();
    return;
  }
  GraphKey k = key;
  k.set = cur;
  auto it = graphs.find(k);
  if (it == graphs.end()) {
    if (graphs.size() >= 64) clear_graphs();
    const uint64_t before = launches;
    cudaGraph_t g = nullptr;
    EC_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    try {
      enqueue();
    } catch (...) {
      cudaStreamEndCapture(st, &g);
      if (g) cudaGraphDestroy(g);
      launches = before;
      throw;
    }
    EC_CUDA(cudaStreamEndCapture(st, &g));
    cudaGraphExec_t ex = nullptr;
    const cudaError_t e = cudaGraphInstantiate(&ex, g, 0);
    cudaGraphDestroy(g);
    EC_CUDA(e);
    it = graphs.emplace(k, GraphEntry{ex, launches - before}).first;
    launches = before;
  }
  EC_CUDA(cudaGraphLaunch(it->second.exec, st));
  launches += it->second.kernels;
}

void Engine::clear_graphs() {
  for (auto& kv : graphs) cudaGraphExecDestroy(kv.second.exec);
  graphs.clear();
}

void Engine::enqueue_forward(const uint32_t* indices, cudaStream_t st) {
  enqueue_dedup_partition(indices, st);
  gather_local(st);
  pool(st);
}

template <int ITEMS, bool RSRC>
void Engine::launch_dedup_cluster_k(const uint32_t* indices, cudaStream_t st) {
  constexpr size_t smem = cluster_smem_bytes(ITEMS);
  static bool attr_set[64] = {};  // per device
  if (!attr_set[device & 63]) {
    if (kClusterCtas > 8)  // (a build with 16-CTA clusters: non-portable size)
      EC_CUDA(cudaFuncSetAttribute(k_dedup_cluster<ITEMS, RSRC>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    EC_CUDA(cudaFuncSetAttribute(k_dedup_cluster<ITEMS, RSRC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
    attr_set[device & 63] = true;
  }
  k_dedup_cluster<ITEMS, RSRC><<<kClusterCtas * T, kClusterThreads, smem, st>>>(
      tdev.p, static_cast<int>(T), indices, tstat.p, ctr.p, uniq.p, uslot.p, utab.p, inv.p, usrc.p, missq.p, ucount.p,
      storage == EC_STORAGE_HOST ? 1 : 0, RSRC ? reinterpret_cast<int32_t*>(slot_of.p) : nullptr);
}
template <int ITEMS>
void Engine::launch_dedup_cluster(const uint32_t* indices, cudaStream_t st) {
  // (row sources only on the fused path: per-table batches < 32768, ITEMS <= 8)
  if constexpr (ITEMS <= 8)
    if (bb[cur].row_sources) return launch_dedup_cluster_k<ITEMS, true>(indices, st);
  launch_dedup_cluster_k<ITEMS, false>(indices, st);
}

// The per-unique counts (and the fp64 sums of the rows they made heavy) the
// set's last batch left behind -- the fused host tier's misses, read by their
// write-back, or a batch whose backward never ran -- cleared before the next
// dedup that counts, from the last batch's counters (before their reset).
// Launched whenever the cluster kernel counts, so captured graphs hold it.
template <int VEC>
void Engine::clear_sums(cudaStream_t st) {
  PhaseScope ph(prof, kPhaseClearSums, st);
  k_clear_miss_sums<VEC><<<sm_count(device) * 4, kThreads, 0, st>>>(static_cast<int>(T), ctr.p, ucount.p, g64.p);
  launched();
}


void Engine::enqueue_dedup_partition(const uint32_t* indices, cudaStream_t st) {
  bb[cur].counted = !use_table_kernel() && use_cluster();
  // the fused pool's per-lookup row sources (slot_of is the tile path's
  // buffer), pinned-host tier only.  Interleaved A/B (profiles/r02/
  // row_sources_ab.txt): the host-tier step 0.096-0.099 -> 0.089-0.093 ms
  // (the pool reads one word per lookup, no inverse -> usrc hop; the
  // prefetched dedup has slack there), but with HBM rows the dedup's extra
  // work lands on the step (Kaggle HBM 0.049 -> 0.050, uniform skew 0.054 ->
  // 0.062 ms); EC_ROW_SOURCES=all turns them on there too
  bb[cur].row_sources = bb[cur].counted && fused() && (storage == EC_STORAGE_HOST || row_sources_all());
  // also after a counting batch when this one does not count (a mode or
  // geometry change): its heavy rows' fp64 sums would otherwise meet the next
  // scatter that sums into g64.  (Graphs are re-captured on such changes, and a
  // clear with nothing left is a no-op.)
  if (bb[cur].counted || bb[cur].left_counts) EC_DISPATCH_VEC(clear_sums, st);
  bb[cur].left_counts = bb[cur].counted;
  if (use_table_kernel()) {
    EC_CUDA(cudaMemsetAsync(ctr.p, 0, (counters_size(T) - 1) * sizeof(int), st));  // keeps err
    EC_CUDA(cudaMemsetAsync(tstat.p, 0, T * sizeof(unsigned long long), st));
    PhaseScope ph(prof, kPhaseDedupCluster, st);
    static bool attr_set[64] = {};
    if (!attr_set[device & 63]) {
      EC_CUDA(cudaFuncSetAttribute(k_dedup_table, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(table_smem_bytes())));
      attr_set[device & 63] = true;
    }
    k_dedup_table<<<T, kTableThreads, table_smem_bytes(), st>>>(tdev.p, static_cast<int>(T), indices, tstat.p, ctr.p,
                                                                uniq.p, uslot.p, utab.p, inv.p, usrc.p, missq.p);
    launched();
    return;
  }
  if (use_cluster()) {
    // one thread-block cluster per table: K1 + K2 in a single kernel
    EC_CUDA(cudaMemsetAsync(ctr.p, 0, (counters_size(T) - 1) * sizeof(int), st));  // keeps err
    EC_CUDA(cudaMemsetAsync(tstat.p, 0, T * sizeof(unsigned long long), st));
    PhaseScope ph(prof, kPhaseDedupCluster, st);
    switch (cluster_items) {
      case 1: launch_dedup_cluster<1>(indices, st); break;
      case 2: launch_dedup_cluster<2>(indices, st); break;
      case 4: launch_dedup_cluster<4>(indices, st); break;
      case 8: launch_dedup_cluster<8>(indices, st); break;
      default: launch_dedup_cluster<16>(indices, st); break;
    }
    launched();
    return;
  }
  const bool lists = lists_in_forward();
  bb[cur].lists = lists;
  {
    if (ntiles) {
      {
        PhaseScope ph(prof, kPhaseInsert, st);
        k_insert<<<ntiles, kThreads, 0, st>>>(tiles.p, tdev.p, indices, slot_of.p, status.p, ctr.p, static_cast<int>(T),
                                              lists ? 1 : 0);
        launched();
      }
      PhaseScope ph(prof, kPhaseCompact, st);
      k_compact<<<ntiles, kThreads, 0, st>>>(tiles.p, tdev.p, indices, slot_of.p, status.p, ctr.p, static_cast<int>(T),
                                             ntiles, tail_lo, uniq.p, uslot.p, utab.p, lists ? cnt.p : nullptr);
      launched();
      if (lists) {  // group offsets: exclusive scan of the per-unique counts (cnt becomes the fill cursor)
        const int nparts = static_cast<int>((max_n * T + kScanTile) / kScanTile);
        k_uscan_reduce<<<nparts, kScanThreads, 0, st>>>(cnt.p, ctr.p, static_cast<int>(T), part.p);
        launched();
        k_scan_partials<<<1, 1024, 0, st>>>(part.p, nparts, nullptr);
        launched();
        k_uscan_apply<<<nparts, kScanThreads, 0, st>>>(cnt.p, ctr.p, static_cast<int>(T), part.p, off.p);
        launched();
      }
    } else {
      EC_CUDA(cudaMemsetAsync(ctr.p, 0, (counters_size(T) - 1) * sizeof(int), st));  // keeps err
    }
  }
  {
    PhaseScope ph(prof, kPhaseInversePartition, st);
    GroupFill gf{};
    if (lists) gf = GroupFill{list.p, off.p, cnt.p, bag_off, static_cast<int>(geom_b), static_cast<int>(geom_p)};
    k_inverse_partition<<<ntiles + sm_count(device) * 2, kThreads, 0, st>>>(tiles.p, tdev.p, slot_of.p, inv.p, ntiles,
                                                                          static_cast<int>(T), ctr.p, uniq.p, utab.p,
                                                                          usrc.p, missq.p, gf);
    launched();
  }
}

void Engine::backward(const float* grad, float lr, cudaStream_t st) {
  if (!have_fwd) invalid("ec_lookup_bwd needs a preceding ec_lookup_fwd");
  if (in_group) invalid("this rank belongs to a loopback group: use ec_group_lookup_bwd");
  if (!grad) invalid("null gradient");
  use_device(device);
  rows_trained = true;
  if (world == 1) {
    uint32_t lr_bits;
    std::memcpy(&lr_bits, &lr, sizeof(lr_bits));
    const int h = head_pending();
    const GraphKey key{h >= 0 && bb[h].gathered ? 3 : 1, grad, bag_off, out_ptr, lr_bits};
    run_maybe_graphed(key, st, [&] { scatter_and_apply_local(grad, lr, st); });
    // host-tier write-back left running: it overlaps the next forward and is
    // joined by whatever next reuses this set or the host tier
    if (storage == EC_STORAGE_HOST) EC_DISPATCH_VEC(enqueue_host_writeback, lr);
  } else if (p2p_on()) {
    if (!p2p_step_open()) invalid("the peer-memory exchange takes one backward per forward");
    EC_DISPATCH_VEC(bwd_scatter, grad, st);
    p2p_bwd_publish(lr, st);  // hits -> own list (host tier: misses -> owners' inboxes); signals barrier 0
    p2p_bwd_finish(lr, st);   // owners' rows, then every rank's list in rank order into the cache replica
  } else {
    scatter_and_apply_local(grad, lr, st);
    exchange_bwd(lr, st);  // remote misses -> owners, replicated hot rows in rank order
  }
}

void Engine::read_counters(cudaStream_t st, std::vector<int>& h) {
  use_device(device);
  h.resize(counters_size(T));
  // the counters are final once this batch's dedup/partition ran on `st`
  // (a consumed prefetch was joined into `st`); one small pinned copy
  EC_CUDA(cudaMemcpyAsync(ctr_host, ctr.p, h.size() * sizeof(int), cudaMemcpyDeviceToHost, st));
  EC_CUDA(cudaStreamSynchronize(st));
  std::memcpy(h.data(), ctr_host, h.size() * sizeof(int));
  Counters c = counters(h.data(), T);
  if (*c.err) {
    *c.err = 0;
    EC_CUDA(cudaMemset(counters(ctr.p, T).err, 0, sizeof(int)));
    invalid("lookup id out of range of its table in the last batch");
  }
}


// ------------------------------------------------------------ profiling
NvtxRange::NvtxRange(const char* name) { nvtxRangePushA(name); }
NvtxRange::~NvtxRange() { nvtxRangePop(); }
const char* phase_name(int phase) {
  static const char* const names[kNumPhases] = {"ec:insert",  "ec:compact", "ec:inverse_partition", "ec:gather",
                                                "ec:gather_host", "ec:exchange", "ec:pool", "ec:scatter",
                                                "ec:apply", "ec:apply_host", "ec:dedup_cluster", "ec:clear_miss_sums"};
  return phase >= 0 && phase < kNumPhases ? names[phase] : "ec:?";
}

PhaseScope::PhaseScope(Profiler& p, int phase, cudaStream_t st)
    : nvtx_(phase_name(phase)), p_(p), phase_(phase), st_(st) {
  if (!p_.on) return;
  a_ = p_.take();
  EC_CUDA(cudaEventRecord(a_, st_));
}
PhaseScope::~PhaseScope() {
  if (!p_.on || !a_) return;
  cudaEvent_t b = p_.take();
  cudaEventRecord(b, st_);
  p_.recs.push_back({phase_, a_, b});
}
cudaEvent_t Profiler::take() {
  if (free_.empty()) {
    cudaEvent_t e;
    EC_CUDA(cudaEventCreate(&e));
    return e;
  }
  cudaEvent_t e = free_.back();
  free_.pop_back();
  return e;
}
void Profiler::collect() {
  for (const Rec& r : recs) {
    EC_CUDA(cudaEventSynchronize(r.b));
    float ms = 0.f;
    EC_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
    ms_[r.phase] += ms;
    calls_[r.phase] += 1;
    if (timeline.size() < kTimelineCap) {
      if (!t0) t0 = r.a;  // first event since the last timeline read
      float s = 0.f;
      EC_CUDA(cudaEventElapsedTime(&s, t0, r.a));
      timeline.push_back({static_cast<double>(r.phase), static_cast<double>(s), static_cast<double>(s + ms)});
    }
    if (r.a != t0) free_.push_back(r.a);
    free_.push_back(r.b);
  }
  recs.clear();
}
Profiler::~Profiler() {
  for (auto& r : recs) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  if (t0) cudaEventDestroy(t0);
  for (auto e : free_) cudaEventDestroy(e);
}

}  // namespace ec

// ===================================================================== ABI
using namespace ec;

static Engine& E(ec_tables t) {
  if (!t) invalid("null tables handle");
  return t->e;
}

extern "C" {

int ec_tables_create(const ec_tables_config* cfg, ec_tables* out) {
  return guard([&] {
    if (!cfg || !out) invalid("null argument");
    auto* t = new ec_tables_s;
    try {
      t->e.create(*cfg);
    } catch (...) {
      delete t;
      throw;
    }
    *out = t;
  });
}

void ec_tables_destroy(ec_tables t) {
  if (!t) return;
  cudaSetDevice(t->e.device);
  cudaDeviceSynchronize();
  delete t;
}

int ec_tables_profile(ec_tables t, int enable) {
  return guard([&] {
    Engine& e = E(t);
    use_device(e.device);
    e.prof.collect();
    e.prof.on = enable != 0;
  });
}

int ec_tables_profile_timeline(ec_tables t, double* out, uint64_t cap, uint64_t* count) {
  return guard([&] {
    Engine& e = E(t);
    use_device(e.device);
    e.prof.collect();
    const uint64_t n = std::min<uint64_t>(cap, e.prof.timeline.size());
    for (uint64_t i = 0; i < n; ++i) {
      out[3 * i] = e.prof.timeline[i][0];
      out[3 * i + 1] = e.prof.timeline[i][1];
      out[3 * i + 2] = e.prof.timeline[i][2];
    }
    *count = e.prof.timeline.size();
    e.prof.timeline.clear();
    if (e.prof.t0) {
      e.prof.free_.push_back(e.prof.t0);
      e.prof.t0 = nullptr;
    }
  });
}

int ec_tables_profile_read(ec_tables t, double* ms, uint64_t* calls, uint64_t* launches, int reset) {
  return guard([&] {
    Engine& e = E(t);
    use_device(e.device);
    e.prof.collect();
    for (int i = 0; i < kNumPhases; ++i) {
      if (ms) ms[i] = e.prof.ms_[i];
      if (calls) calls[i] = e.prof.calls_[i];
    }
    if (launches) *launches = e.launches;
    if (reset) {
      for (int i = 0; i < kNumPhases; ++i) e.prof.ms_[i] = 0.0, e.prof.calls_[i] = 0;
      e.launches = 0;
    }
  });
}

int ec_tables_dedup_mode(ec_tables t, int mode) {
  return guard([&] {
    if (mode < 0 || mode > 3)
      invalid("dedup mode: 0 auto, 1 tiles, 2 cluster per table, 3 one CTA per table (when it fits)");
    Engine& e = E(t);
    if (mode == 2 || mode == 3) e.require_direct_sets();
    e.dedup_mode = mode;
    e.clear_graphs();
  });
}

int ec_tables_scatter_mode(ec_tables t, int mode) {
  return guard([&] {
    if (mode < 0 || mode > 2) invalid("scatter mode: 0 auto, 1 float4 atomics, 2 transpose");
    Engine& e = E(t);
    e.scatter_mode = mode;
    e.clear_graphs();
  });
}

int ec_tables_use_graphs(ec_tables t, int enable) {
  return guard([&] {
    Engine& e = E(t);
    e.use_graphs = enable != 0;
    if (!e.use_graphs) e.clear_graphs();
  });
}

int ec_tables_memory(ec_tables t, uint64_t* dev, uint64_t* host) {
  return guard([&] {
    Engine& e = E(t);
    if (dev) *dev = e.device_bytes();
    if (host) *host = e.store_host ? e.store_off[e.T] * e.D * sizeof(float) : 0;
  });
}

int ec_tables_init_synthetic(ec_tables t, uint64_t seed, float scale, void* stream) {
  return guard([&] { E(t).init_synthetic(seed, scale, as_stream(stream)); });
}

int ec_tables_place_cache(ec_tables t, const uint32_t* const* ids, const uint64_t* k) {
  return guard([&] { E(t).place_cache(ids, k); });
}

int ec_tables_read_rows(ec_tables t, uint32_t table, const uint32_t* ids, uint64_t n, float* out) {
  return guard([&] { E(t).rw_rows(table, ids, n, out, false); });
}

int ec_tables_write_rows(ec_tables t, uint32_t table, const uint32_t* ids, uint64_t n, const float* rows) {
  return guard([&] { E(t).rw_rows(table, ids, n, const_cast<float*>(rows), true); });
}

int ec_lookup_fwd(ec_tables t, const ec_batch* b, float* out, void* stream) {
  return guard([&] {
    NvtxRange r("ec_lookup_fwd");
    if (!b || !out) invalid("null argument");
    E(t).forward(*b, out, as_stream(stream));
  });
}

int ec_lookup_prefetch(ec_tables t, const ec_batch* b, void* stream) {
  return guard([&] {
    NvtxRange r("ec_lookup_prefetch");
    if (!b) invalid("null batch");
    E(t).prefetch(*b, as_stream(stream));
  });
}

int ec_tables_schedule(ec_tables t, const uint32_t* ids_dev, uint64_t q, uint32_t* order_dev, uint64_t* num_hot,
                       void* stream) {
  return guard([&] {
    Engine& e = E(t);
    if (!ids_dev || !order_dev || !num_hot) invalid("null argument");
    if (q == 0) invalid("empty dataset");
    if (q >= (1ull << 31)) invalid("at most 2^31-1 samples");
    use_device(e.device);
    cudaStream_t st = as_stream(stream);
    DevBuf<int> hot(q), excl(q), part(scan_parts(q)), scal(2);
    EC_CUDA(cudaMemsetAsync(scal.p, 0, 2 * sizeof(int), st));
    const int grid = sm_count(e.device) * 4;
    k_classify_tables<<<grid, 256, 0, st>>>(e.tdev.p, static_cast<int>(e.T), ids_dev, q, hot.p, scal.p + 1);
    EC_LAUNCH();
    exclusive_scan(hot.p, static_cast<int64_t>(q), excl.p, part.p, scal.p, st);
    k_stable_order<<<grid, 256, 0, st>>>(hot.p, excl.p, scal.p, q, order_dev);
    EC_LAUNCH();
    int h[2];
    EC_CUDA(cudaMemcpyAsync(h, scal.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    EC_CUDA(cudaStreamSynchronize(st));
    if (h[1]) invalid("dataset id out of range of its table");
    *num_hot = static_cast<uint64_t>(h[0]);
  });
}

int ec_tables_gather_batch(ec_tables t, const uint32_t* ids_dev, const uint32_t* order_dev, uint64_t first,
                           uint32_t count, uint32_t* indices_dev, void* stream) {
  return guard([&] {
    Engine& e = E(t);
    if (!ids_dev || !order_dev || !indices_dev) invalid("null argument");
    use_device(e.device);
    if (!count) return;
    const uint64_t n = static_cast<uint64_t>(count) * e.T;
    const int grid = static_cast<int>(std::min<uint64_t>((n + 255) / 256, sm_count(e.device) * 8ull));
    k_gather_batch<<<grid, 256, 0, as_stream(stream)>>>(ids_dev, order_dev, first, count, static_cast<int>(e.T),
                                                         indices_dev);
    EC_LAUNCH();
  });
}

int ec_lookup_prefetch_drop(ec_tables t, void* stream) {
  return guard([&] {
    Engine& e = E(t);
    use_device(e.device);
    e.drop_prefetch(as_stream(stream));
  });
}

int ec_lookup_prefetch_wait(ec_tables t, void* stream) {
  return guard([&] {
    Engine& e = E(t);
    use_device(e.device);
    for (BatchBufs& b : e.bb)
      if (b.pending) EC_CUDA(cudaStreamWaitEvent(as_stream(stream), b.gathered ? b.ev_pf : b.ev_ded, 0));
    e.join_host_writes(as_stream(stream));
  });
}

int ec_lookup_bwd(ec_tables t, const float* grad, float lr, void* stream) {
  return guard([&] {
    NvtxRange r("ec_lookup_bwd");
    E(t).backward(grad, lr, as_stream(stream));
  });
}

static void decode_stats(Engine& e, int* h, uint64_t lookups, uint64_t wire_rows, uint64_t wire_bytes,
                         ec_batch_stats* out, int64_t* u_per, int64_t* m_per) {
  Counters c = counters(h, e.T);
  ec_batch_stats s{};
  s.lookups = lookups;
  s.index_units = s.lookups;
  for (uint32_t i = 0; i < e.T; ++i) {
    const int Ui = c.ubase[i + 1] - c.ubase[i];
    s.unique_rows += Ui;
    s.miss_rows += c.M[i];
    s.hot_tables += c.M[i] == 0;
    if (u_per) u_per[i] = Ui;
    if (m_per) m_per[i] = c.M[i];
  }
  s.hit_rows = s.unique_rows - s.miss_rows;
  s.model_bytes = s.miss_rows * e.D * sizeof(float) + s.index_units * sizeof(uint32_t);
  s.wire_rows = wire_rows;
  s.wire_bytes = wire_bytes;
  if (e.p2p_on()) {
    // peer-memory exchange: rows this rank pulled (device count) and their
    // gradient atomics back (the reference-priced miss rows), plus the hot-row
    // sync (not in the reference's model): gradients to other owners, updated
    // rows from them (counted on the device, complete once the backward ran)
    const uint64_t rowb = static_cast<uint64_t>(e.D) * sizeof(float);
    s.wire_rows = static_cast<uint64_t>(*c.wire);
    s.hot_sync_rows = static_cast<uint64_t>(*c.hot_out) + static_cast<uint64_t>(*c.hot_in);
    s.hot_sync_bytes = s.hot_sync_rows * (4 + rowb);
    s.wire_bytes = 2 * s.wire_rows * rowb + s.hot_sync_bytes;
  }
  *out = s;
}

int ec_lookup_stats_enqueue(ec_tables t, void* stream, int slot) {
  return guard([&] {
    Engine& e = E(t);
    if (!e.have_fwd) invalid("no forward batch yet");
    if (slot < 0 || slot >= EC_STATS_SLOTS) invalid("stats slot out of [0, EC_STATS_SLOTS)");
    use_device(e.device);
    const size_t n = counters_size(e.T);
    cudaStream_t st = as_stream(stream);
    // a slot is reused only after its previous copy landed
    if (e.ring_full[slot]) EC_CUDA(cudaEventSynchronize(e.ring_ev[slot]));
    EC_CUDA(cudaMemcpyAsync(e.ring_host + slot * n, e.ctr.p, n * sizeof(int), cudaMemcpyDeviceToHost, st));
    EC_CUDA(cudaEventRecord(e.ring_ev[slot], st));
    e.ring_lookups[slot] = static_cast<uint64_t>(e.geom_off[e.T]);
    e.ring_wire_rows[slot] = e.last_wire_rows;
    e.ring_wire_bytes[slot] = e.last_wire_bytes;
    e.ring_full[slot] = true;
  });
}

int ec_lookup_stats_collect(ec_tables t, int slot, ec_batch_stats* out, int64_t* u_per, int64_t* m_per) {
  return guard([&] {
    Engine& e = E(t);
    if (slot < 0 || slot >= EC_STATS_SLOTS) invalid("stats slot out of [0, EC_STATS_SLOTS)");
    if (!e.ring_full[slot]) invalid("stats slot was not enqueued");
    use_device(e.device);
    EC_CUDA(cudaEventSynchronize(e.ring_ev[slot]));
    e.ring_full[slot] = false;
    int* h = e.ring_host + slot * counters_size(e.T);
    Counters c = counters(h, e.T);
    if (*c.err) {
      EC_CUDA(cudaMemset(counters(e.ctr.p, e.T).err, 0, sizeof(int)));
      invalid("lookup id out of range of its table in the enqueued batch");
    }
    decode_stats(e, h, e.ring_lookups[slot], e.ring_wire_rows[slot], e.ring_wire_bytes[slot], out, u_per, m_per);
  });
}

int ec_lookup_stats(ec_tables t, void* stream, ec_batch_stats* out, int64_t* u_per, int64_t* m_per) {
  return guard([&] {
    Engine& e = E(t);
    if (!e.have_fwd) invalid("no forward batch yet");
    std::vector<int> h;
    e.read_counters(as_stream(stream), h);
    decode_stats(e, h.data(), static_cast<uint64_t>(e.geom_off[e.T]), e.last_wire_rows, e.last_wire_bytes, out, u_per,
                 m_per);
  });
}

static void table_span(Engine& e, uint32_t table, std::vector<int>& h, int* lo, int* n) {
  if (table >= e.T) invalid("table index out of range");
  if (!e.have_fwd) invalid("no forward batch yet");
  e.read_counters(nullptr, h);
  Counters c = counters(h.data(), e.T);
  *lo = c.ubase[table];
  *n = c.ubase[table + 1] - c.ubase[table];
}

int ec_export_unique(ec_tables t, uint32_t table, uint32_t* out, uint64_t cap, uint64_t* count) {
  return guard([&] {
    Engine& e = E(t);
    std::vector<int> h;
    int lo, n;
    table_span(e, table, h, &lo, &n);
    *count = static_cast<uint64_t>(n);
    if (out) EC_CUDA(cudaMemcpy(out, e.uniq.p + lo, std::min<uint64_t>(cap, n) * sizeof(uint32_t), cudaMemcpyDeviceToHost));
  });
}

int ec_export_inverse(ec_tables t, uint32_t table, uint32_t* out) {
  return guard([&] {
    Engine& e = E(t);
    std::vector<int> h;
    int lo, n;
    table_span(e, table, h, &lo, &n);
    const int64_t a = e.geom_off[table], m = e.geom_off[table + 1] - a;
    EC_CUDA(cudaMemcpy(out, e.inv.p + a, m * sizeof(uint32_t), cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < m; ++i) out[i] -= static_cast<uint32_t>(lo);
  });
}

int ec_export_hit(ec_tables t, uint32_t table, uint8_t* out) {
  return guard([&] {
    Engine& e = E(t);
    std::vector<int> h;
    int lo, n;
    table_span(e, table, h, &lo, &n);
    std::vector<int32_t> s(n);
    if (n) EC_CUDA(cudaMemcpy(s.data(), e.usrc.p + lo, n * sizeof(int32_t), cudaMemcpyDeviceToHost));
    for (int i = 0; i < n; ++i) out[i] = s[i] >= 0;
  });
}

int ec_export_rows(ec_tables t, uint32_t table, float* out) {
  return guard([&] {
    Engine& e = E(t);
    std::vector<int> h;
    int lo, n;
    table_span(e, table, h, &lo, &n);
    if (n && e.fused()) e.gather_for_export();  // the fused forward pooled from the source rows
    if (n) EC_CUDA(cudaMemcpy(out, e.urows.p + static_cast<int64_t>(lo) * e.D, static_cast<int64_t>(n) * e.D * sizeof(float),
                              cudaMemcpyDeviceToHost));
  });
}

}  // extern "C"
