// sm_100a kernels of the lookup engine (K1 dedup, K2 hit/miss, K3 gather,
// K5 pool, K6 backward).  Included by engine.cu; see the pipeline and HBM
// layout described there.
//
// Per batch (fixed kernel sequence, no host synchronisation, CUDA-graph
// capturable):
//   k_insert           lookup -> hash slot (warp match-any collapse, packed
//                      atomicMin keeps each id's first position); resets the
//                      look-back status words and per-batch counters
//   k_compact          first-occurrence flags, single-pass decoupled
//                      look-back scan over tiles (table-major) -> global unique
//                      index, unique ids emitted, slot tagged with the index
//   k_inverse_partition  lookup -> unique index (inverse) | unique -> cache slot
//                      or miss (per-table miss counts, miss queue)
//   k_gather           cache/HBM rows -> compact unique rows; also clears the
//                      hash slot and zeroes the unique's gradient row
//   k_gather_host      pinned-host misses (side stream)
//   k_pool             EmbeddingBag sum through inverse indices
//   k_scatter          bag gradients -> unique rows: fp64 RED sums per distinct row (g64)
//                      of a warp (equal rows pre-summed with shuffles)
//   k_apply(_host)     SGD into cache rows / owning shard
#pragma once

#include <cooperative_groups.h>

#include "device_util.cuh"
#include "engine.hpp"
#include "scan.cuh"

namespace ec {

constexpr int kThreads = 256;
constexpr int kItems = 4;
constexpr int kTile = kThreads * kItems;  // lookups per dedup tile
constexpr int kRunChunk = 32;             // grouped-gradient list entries per lane group (K6a)
// k_bwd_reduce chunks a unique's list entries [a, b) fall in
__host__ __device__ inline int chunk_span(int a, int b) { return (b - 1) / kRunChunk - a / kRunChunk + 1; }

// ------------------------------------------------------------------ K1
// Insert (id, lpos) starting at slot h whose current content `cur` was
// already loaded; returns the slot holding id.  Packed words (id << 32 | pos)
// make "keep the first position" a 64-bit atomicMin on an existing key.
__device__ __forceinline__ uint32_t hash_insert_from(unsigned long long* tab, uint32_t mask, uint32_t h,
                                                     unsigned long long cur, uint32_t id, uint32_t lpos) {
  const unsigned long long mine = (static_cast<unsigned long long>(id) << 32) | lpos;
  for (;;) {
    if (cur == kEmptySlot) {
      cur = atomicCAS(tab + h, kEmptySlot, mine);
      if (cur == kEmptySlot) return h;
    }
    if (static_cast<uint32_t>(cur >> 32) == id) {
      if (static_cast<uint32_t>(cur) > lpos) atomicMin(tab + h, mine);
      return h;
    }
    h = (h + 1) & mask;
    cur = __ldcg(tab + h);
  }
}

// The 64-bit set word of `slot`.  A direct-mapped set interleaves (set word,
// copy of the id's remap entry) per id, so the DRAM sector a unique's first
// insert pulls into L2 also holds its cache row: one random sector per unique
// instead of two (the cluster dedup reads the copy; Engine::sync_set_remap
// keeps it equal to `remap`).  Hashed sets: one word per slot.
__device__ __forceinline__ unsigned long long* set_word(const TableDev& t, uint32_t slot) {
  return t.hash + (t.direct ? 2 * static_cast<uint64_t>(slot) : static_cast<uint64_t>(slot));
}
// id's cache row from a direct-mapped set's interleaved remap copy
__device__ __forceinline__ int32_t set_remap(const TableDev& t, uint32_t id) {
  return __ldg(reinterpret_cast<const int32_t*>(t.hash + 2 * static_cast<uint64_t>(id) + 1));
}

// Slot of `id` in a table's dedup set: the id itself when direct-mapped.
__device__ __forceinline__ uint32_t table_slot(const TableDev& t, uint32_t id) {
  return t.direct ? id : hash_slot(id, t.shift);
}

// Insert (id, first position lpos) into a table's dedup set; returns its slot.
// Direct-mapped: one 64-bit atomicMin on the id's own slot (empty = ~0).
__device__ __forceinline__ uint32_t set_insert(const TableDev& t, uint32_t id, uint32_t lpos) {
  const unsigned long long mine = (static_cast<unsigned long long>(id) << 32) | lpos;
  if (t.direct) {
    atomicMin(set_word(t, id), mine);
    return id;
  }
  const uint32_t h = hash_slot(id, t.shift);
  const unsigned long long cur = atomicCAS(t.hash + h, kEmptySlot, mine);
  return cur == kEmptySlot ? h : hash_insert_from(t.hash, t.mask, h, cur, id, lpos);
}

// grad-row index (bag) of lookup p in table t
__device__ __forceinline__ int bag_of(const TableDev& tb, const int64_t* bag_off, int B, int P, int t, int64_t p) {
  if (!bag_off) return static_cast<int>((p - tb.base) / P);
  const int64_t* b = bag_off + static_cast<int64_t>(t) * B;  // last s with b[s] <= p
  int lo = 0, hi = B;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (b[mid] <= p) lo = mid; else hi = mid;
  }
  return lo;
}

// Unique-grouped gradient list built by the forward's k_inverse_partition
// (tile dedup path, transpose backward): lookups of unique u occupy
// list[off[u] .. off[u+1]), as (u, grad row); `cursor` starts at zero.
struct GroupFill {
  uint2* list;  // null: not built here
  const int* off;
  int* cursor;
  const int64_t* bag_off;
  int B, P;
};

// With `count` set, also counts each id's lookups on its slot (idcnt, one
// atomic per warp group) for the unique-grouped gradient lists.
__global__ void __launch_bounds__(kThreads) k_insert(const Tile* __restrict__ tiles, const TableDev* __restrict__ td,
                                                     const uint32_t* __restrict__ indices,
                                                     uint32_t* __restrict__ slot_of,
                                                     unsigned long long* __restrict__ status, int* __restrict__ ctr,
                                                     int T, int count) {
  const Tile tile = tiles[blockIdx.x];
  const TableDev t = td[tile.table];
  Counters c = counters(ctr, T);
  if (threadIdx.x == 0) status[blockIdx.x] = 0;  // look-back word of this tile, read by k_compact
  if (blockIdx.x == 0) {
    for (int i = threadIdx.x; i < T; i += blockDim.x) c.M[i] = 0;
    if (threadIdx.x == 0) {
      *c.miss_total = 0;
      *c.tile_counter = 0;
      *c.wire = 0;
    }
  }
  uint32_t id[kItems];
  bool live[kItems];
#pragma unroll
  for (int j = 0; j < kItems; ++j) {  // all loads first: kItems independent requests in flight
    const uint32_t off = j * kThreads + threadIdx.x;
    live[j] = off < tile.count;
    id[j] = live[j] ? __ldcs(indices + tile.start + off) : kEmptyKey;
  }
  unsigned peers[kItems];
  uint32_t h[kItems];
  unsigned long long cur[kItems];
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    if (live[j] && id[j] >= t.rows) {
      atomicExch(c.err, 1);
      live[j] = false;
      id[j] = kEmptyKey;
    }
    // lanes holding the same id collapse to their lowest lane (= smallest position)
    peers[j] = __match_any_sync(kFull, id[j]);
    h[j] = table_slot(t, id[j]);
  }
#pragma unroll
  for (int j = 0; j < kItems; ++j)  // home-slot probes of all items in flight together
    cur[j] = (live[j] && __ffs(peers[j]) - 1 == lane_id()) ? __ldcg(set_word(t, h[j])) : 0;
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const uint32_t off = j * kThreads + threadIdx.x;
    const int64_t p = tile.start + off;
    const int leader = __ffs(peers[j]) - 1;
    uint32_t slot = 0;
    if (live[j] && leader == lane_id()) {
      if (t.direct) {
        if (static_cast<uint32_t>(cur[j]) > static_cast<uint32_t>(p - t.base))
          atomicMin(set_word(t, h[j]), (static_cast<unsigned long long>(id[j]) << 32) | static_cast<uint32_t>(p - t.base));
        slot = h[j];
      } else {
        slot = hash_insert_from(t.hash, t.mask, h[j], cur[j], id[j], static_cast<uint32_t>(p - t.base));
      }
      if (count) atomicAdd(t.idcnt + slot, static_cast<uint32_t>(__popc(peers[j])));
    }
    slot = __shfl_sync(kFull, slot, leader);
    if (live[j]) slot_of[p] = slot;
    else if (off < tile.count) slot_of[p] = kInvalidSlot;  // out-of-range id: skipped downstream
  }
}

// Lookup p is its id's first occurrence iff the slot's packed minimum is p.
__device__ __forceinline__ bool is_first(const TableDev& t, const uint32_t* slot_of, int64_t p, uint32_t* h) {
  *h = slot_of[p];
  return *h != kInvalidSlot && static_cast<uint32_t>(__ldcg(set_word(t, *h))) == static_cast<uint32_t>(p - t.base);
}

constexpr unsigned long long kStatAgg = 1ull << 32;  // status word: (flag << 32) | value
constexpr unsigned long long kStatInc = 2ull << 32;

__device__ __forceinline__ void publish(unsigned long long* p, unsigned long long v) {
  __threadfence();
  *reinterpret_cast<volatile unsigned long long*>(p) = v;
}

// Flags + single-pass scan (decoupled look-back over tiles claimed in order
// through an atomic counter) + emission.  Tiles are table-major, so the
// global exclusive prefix is the unique index in (table, first occurrence)
// order and the prefix at a table's first tile is that table's ubase.
__global__ void __launch_bounds__(kThreads) k_compact(const Tile* __restrict__ tiles, const TableDev* __restrict__ td,
                                                      const uint32_t* __restrict__ indices,
                                                      const uint32_t* __restrict__ slot_of,
                                                      unsigned long long* __restrict__ status, int* __restrict__ ctr,
                                                      int T, int ntiles, int tail_lo, uint32_t* __restrict__ uniq,
                                                      uint32_t* __restrict__ uslot, uint16_t* __restrict__ utab,
                                                      int* __restrict__ ucnt) {
  __shared__ int s_tile, s_excl;
  __shared__ int sw[kThreads / 32];
  Counters c = counters(ctr, T);
  if (threadIdx.x == 0) s_tile = atomicAdd(c.tile_counter, 1);
  __syncthreads();
  const int ti = s_tile;
  const Tile tile = tiles[ti];
  const TableDev t = td[tile.table];
  bool first[kItems];
  uint32_t h[kItems];
  int ex[kItems], count = 0;
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const uint32_t off = j * kThreads + threadIdx.x;
    h[j] = off < tile.count ? slot_of[tile.start + off] : kInvalidSlot;
  }
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const uint32_t off = j * kThreads + threadIdx.x;
    first[j] = h[j] != kInvalidSlot &&
               static_cast<uint32_t>(__ldcg(set_word(t, h[j]))) == static_cast<uint32_t>(tile.start + off - t.base);
  }
#pragma unroll
  for (int j = 0; j < kItems; ++j) {  // position order within the tile: j-major, then thread
    int tot;
    ex[j] = count + block_exclusive_scan<kThreads>(first[j] ? 1 : 0, sw, &tot);
    count += tot;
  }
  // Block-wide decoupled look-back: each thread watches one predecessor per
  // round; the walk stops at the nearest tile with an inclusive prefix.
  if (threadIdx.x == 0) publish(status + ti, (ti == 0 ? kStatInc : kStatAgg) | static_cast<uint32_t>(count));
  __shared__ int s_stop, s_sum;
  int excl = 0;
  for (int k = ti - 1; k >= 0; k -= kThreads) {
    const int idx = k - static_cast<int>(threadIdx.x);
    unsigned long long v = kStatInc;  // before tile 0: an inclusive zero ends the walk
    if (idx >= 0) {
      do {
        v = *reinterpret_cast<volatile unsigned long long*>(status + idx);
      } while ((v >> 32) == 0);
    }
    if (threadIdx.x == 0) { s_stop = kThreads; s_sum = 0; }
    __syncthreads();
    if ((v >> 32) == 2) atomicMin(&s_stop, static_cast<int>(threadIdx.x));
    __syncthreads();
    const int stop = s_stop;
    const int part = __reduce_add_sync(kFull, static_cast<int>(threadIdx.x) <= stop ? static_cast<int>(static_cast<uint32_t>(v)) : 0);
    if (lane_id() == 0 && part) atomicAdd(&s_sum, part);
    __syncthreads();
    excl += s_sum;
    __syncthreads();
    if (stop < kThreads) break;
  }
  if (threadIdx.x == 0) {
    if (ti > 0) publish(status + ti, kStatInc | static_cast<uint32_t>(excl + count));
    s_excl = excl;
    for (uint32_t tb = tile.ub_lo; tb < tile.ub_hi; ++tb) c.ubase[tb] = excl;  // tables starting here
    if (ti == ntiles - 1)
      for (int tb = tail_lo; tb <= T; ++tb) c.ubase[tb] = excl + count;  // trailing empty tables + total
  }
  __syncthreads();
  const int base = s_excl;
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    if (!first[j]) continue;
    const uint32_t off = j * kThreads + threadIdx.x;
    const uint32_t g = static_cast<uint32_t>(base + ex[j]);
    const uint32_t id = indices[tile.start + off];
    uniq[g] = id;
    uslot[g] = h[j];
    utab[g] = static_cast<uint16_t>(tile.table);
    if (ucnt) ucnt[g] = static_cast<int>(t.idcnt[h[j]]);  // lookups of this unique (k_insert counted them)
    // only this thread writes this slot; concurrent flag tests never match a tagged value
    *set_word(t, h[j]) = (static_cast<unsigned long long>(id) << 32) | kRankTag | g;
  }
}

// Blocks [0, ntiles): inverse of each lookup (the slot now holds its tagged
// unique index).  Blocks [ntiles, ...): hit/miss partition of the uniques.
__global__ void __launch_bounds__(kThreads) k_inverse_partition(const Tile* __restrict__ tiles,
                                                                const TableDev* __restrict__ td,
                                                                const uint32_t* __restrict__ slot_of,
                                                                uint32_t* __restrict__ inv, int ntiles, int T,
                                                                int* __restrict__ ctr, const uint32_t* __restrict__ uniq,
                                                                const uint16_t* __restrict__ utab,
                                                                int32_t* __restrict__ usrc,
                                                                uint32_t* __restrict__ missq, GroupFill gf) {
  if (static_cast<int>(blockIdx.x) < ntiles) {
    const Tile tile = tiles[blockIdx.x];
    const TableDev t = td[tile.table];
    uint32_t hs[kItems];
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
      const uint32_t off = j * kThreads + threadIdx.x;
      hs[j] = off < tile.count ? slot_of[tile.start + off] : kInvalidSlot;
    }
    uint32_t u[kItems];
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
      const uint32_t off = j * kThreads + threadIdx.x;
      u[j] = hs[j] == kInvalidSlot ? kInvalidSlot : static_cast<uint32_t>(__ldcg(set_word(t, hs[j]))) & ~kRankTag;
      if (off < tile.count) inv[tile.start + off] = u[j];
    }
    if (gf.list) {  // K6 grouping: lookup -> its unique's group (offsets from the scan of the counts)
#pragma unroll
      for (int j = 0; j < kItems; ++j) {
        const int64_t p = tile.start + j * kThreads + threadIdx.x;
        const unsigned peers = __match_any_sync(kFull, u[j]);
        const int leader = __ffs(peers) - 1;
        int b0 = 0;
        if (u[j] != kInvalidSlot && leader == lane_id()) b0 = atomicAdd(gf.cursor + u[j], __popc(peers));
        b0 = __shfl_sync(kFull, b0, leader);
        if (u[j] != kInvalidSlot) {
          const int pos = gf.off[u[j]] + b0 + __popc(peers & ((1u << lane_id()) - 1));
          gf.list[pos] = make_uint2(u[j], static_cast<uint32_t>(bag_of(t, gf.bag_off, gf.B, gf.P, static_cast<int>(tile.table), p)) *
                                               static_cast<uint32_t>(T) + tile.table);
        }
      }
    }
    return;
  }
  // K2: cache slot (>= 0) or miss (-1) per unique; a lookup misses iff its id
  // is not cached (core/src/simulator.cpp:99)
  Counters c = counters(ctr, T);
  const int U = c.ubase[T];
  const int nb = gridDim.x - ntiles, b = blockIdx.x - ntiles;
  for (int base = b * blockDim.x; base < U; base += nb * blockDim.x) {
    const int g = base + threadIdx.x;
    const bool live = g < U;
    int tab = -1;
    bool miss = false;
    if (live) {
      tab = utab[g];
      const int32_t s = __ldg(td[tab].remap + uniq[g]);
      usrc[g] = s;
      miss = s < 0;
    }
    const unsigned peers = __match_any_sync(kFull, tab);
    const int nm = group_count(peers, miss);
    if (live && nm && (__ffs(peers) - 1) == lane_id()) atomicAdd(c.M + tab, nm);
    const unsigned mb = __ballot_sync(kFull, miss);
    int qbase = 0;
    if (mb && lane_id() == __ffs(mb) - 1) qbase = atomicAdd(c.miss_total, __popc(mb));
    qbase = __shfl_sync(kFull, qbase, __ffs(mb ? mb : 1u) - 1);
    if (miss) missq[qbase + __popc(mb & ((1u << lane_id()) - 1))] = static_cast<uint32_t>(g);
  }
}

// ------------------------------------------------------------------ K3
// VEC = D/4 lanes per row, 128-bit accesses; R rows in flight per thread.
template <int VEC>
struct RowMap {
  static constexpr int kRowsPerWarp = 32 / VEC;
  int sub, c;
  __device__ RowMap() : sub(lane_id() / VEC), c(lane_id() % VEC) {}
};

// With `peers` (the P2P exchange, HBM shards), misses owned by another rank
// are read straight from that rank's shard over NVLink: the forward exchange
// is this kernel's remote loads -- no request/response round, no host sync.
template <int VEC, int R>
__global__ void __launch_bounds__(kThreads) k_gather(const TableDev* __restrict__ td, int T, int* __restrict__ ctr,
                                                     const uint32_t* __restrict__ uniq, const uint16_t* __restrict__ utab,
                                                     const uint32_t* __restrict__ uslot,
                                                     const int32_t* __restrict__ usrc, const float* __restrict__ cache,
                                                     float* __restrict__ urows, float* __restrict__ ugrad,
                                                     int* __restrict__ cnt, int local_hbm, int rank, int world,
                                                     const PeerView* __restrict__ peers = nullptr,
                                                     const int64_t* __restrict__ shard_off = nullptr) {
  constexpr int D = VEC * 4;
  constexpr int RPW = RowMap<VEC>::kRowsPerWarp;
  const RowMap<VEC> m;
  const Counters cs = counters(ctr, T);
  const int U = cs.ubase[T];
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
  int remote = 0;
  for (int g0 = warp * RPW * R; g0 < U; g0 += nwarps * RPW * R) {
    float4 v[R];
    int dst[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int g = g0 + r * RPW + m.sub;
      dst[r] = -1;
      if (g < U) {
        const int32_t s = usrc[g];
        const float* src = nullptr;
        const uint32_t tab = utab[g];
        if (s >= 0) {
          src = cache + static_cast<int64_t>(s) * D;
        } else if (local_hbm) {
          const uint32_t id = uniq[g];
          const int o = static_cast<int>(id % world);
          if (o == rank) {
            src = td[tab].store + static_cast<int64_t>(id / world) * D;
          } else if (peers) {
            src = peers[o].store + (shard_off[static_cast<int64_t>(o) * (T + 1) + tab] + id / world) * D;
            remote += m.c == 0;
          }
        }
        if (src) {
          v[r] = ldg4(src + m.c * 4);
          dst[r] = g;
        }
        if (m.c == 0) {
          const TableDev& tb = td[tab];
          *set_word(tb, uslot[g]) = kEmptySlot;  // leave the set empty for the next batch
          tb.idcnt[uslot[g]] = 0;
          cnt[g] = 0;  // backward occurrence count
        }
        st4(ugrad + static_cast<int64_t>(g) * D + m.c * 4, zero);
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (dst[r] >= 0) st4(urows + static_cast<int64_t>(dst[r]) * D + m.c * 4, v[r]);
  }
  if (peers) {
    remote = __reduce_add_sync(kFull, remote);
    if (remote && lane_id() == 0) atomicAdd(cs.wire, remote);
  }
}

// Misses served from pinned host memory (UVA-mapped shard), side stream.
template <int VEC, int R>
__global__ void __launch_bounds__(kThreads) k_gather_host(const TableDev* __restrict__ td, int T, const int* __restrict__ ctr,
                                                          const uint32_t* __restrict__ missq,
                                                          const uint32_t* __restrict__ uniq,
                                                          const uint16_t* __restrict__ utab, float* __restrict__ urows,
                                                          int rank, int world,
                                                          const PeerView* __restrict__ peers = nullptr,
                                                          const int64_t* __restrict__ shard_off = nullptr) {
  constexpr int D = VEC * 4;
  constexpr int RPW = RowMap<VEC>::kRowsPerWarp;
  const RowMap<VEC> m;
  const Counters cs = counters(const_cast<int*>(ctr), T);
  const int nm = *cs.miss_total;
  int remote = 0;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int q0 = warp * RPW * R; q0 < nm; q0 += nwarps * RPW * R) {
    float4 v[R];
    int dst[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int q = q0 + r * RPW + m.sub;
      dst[r] = -1;
      if (q < nm) {
        const uint32_t g = missq[q];
        const uint32_t id = uniq[g];
        const int o = static_cast<int>(id % world);
        const float* src = nullptr;
        if (o == rank) {
          src = td[utab[g]].store + static_cast<int64_t>(id / world) * D;
        } else if (peers) {
          src = peers[o].store + (shard_off[static_cast<int64_t>(o) * (T + 1) + utab[g]] + id / world) * D;
          remote += m.c == 0;
        }
        if (src) {
          v[r] = *reinterpret_cast<const float4*>(src + m.c * 4);
          dst[r] = static_cast<int>(g);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (dst[r] >= 0) st4(urows + static_cast<int64_t>(dst[r]) * D + m.c * 4, v[r]);
  }
  if (peers) {
    remote = __reduce_add_sync(kFull, remote);
    if (remote && lane_id() == 0) atomicAdd(cs.wire, remote);
  }
}

// ------------------------------------------------------------------ K5
__device__ __forceinline__ void bag_range(const TableDev* td, const int64_t* bag_off, int B, int P, int s, int t,
                                          int64_t* lo, int64_t* hi) {
  if (bag_off) {
    *lo = bag_off[static_cast<int64_t>(t) * B + s];
    *hi = bag_off[static_cast<int64_t>(t) * B + s + 1];
  } else {  // fixed pooling: table t's lookups start at t*B*P (ec_lookup_fwd checks n_t == B*P)
    *lo = (static_cast<int64_t>(t) * B + s) * P;
    *hi = *lo + P;
  }
}

// Row u's float4 #c of the compact unique-row buffer; invalid lookups read 0.
__device__ __forceinline__ float4 load_row(const float* urows, uint32_t u, int D, int c) {
  if (u == kInvalidSlot) return make_float4(0.f, 0.f, 0.f, 0.f);
  return ldg4(urows + static_cast<int64_t>(u) * D + c * 4);
}

// Where unique u's current row lives (single rank, no K3 gather): its cache
// row, its local HBM shard row, or — pinned-host misses, gathered by
// k_gather_host — its row of the compact buffer.
struct RowSrc {
  const int32_t* usrc;
  const uint32_t* uniq;
  const float* cache;
  const float* urows;
  int local_hbm;
  const int32_t* isrc = nullptr;  // per lookup: row_source() words (cluster dedup; pools with RSRC)
};
__device__ __forceinline__ const float* src_row(const RowSrc& rs, const TableDev& tb, uint32_t u, int D) {
  const int32_t s = rs.usrc[u];
  if (s >= 0) return rs.cache + static_cast<int64_t>(s) * D;
  if (rs.local_hbm) return tb.store + static_cast<int64_t>(rs.uniq[u]) * D;
  return rs.urows + static_cast<int64_t>(u) * D;
}

// Per-lookup row source word written by the cluster dedup (k_dedup_cluster,
// phase I): the cache row (>= 0), ~unique index for a miss (its row is the
// local HBM shard's uniq[g], or the compact buffer's row g), kNoSource for an
// invalid lookup (pools a zero row).  Unique indices < 2^31 - 1.
constexpr int32_t kNoSource = INT32_MIN;
__device__ __forceinline__ int32_t row_source(uint32_t g, int32_t cache_row) {
  return g == kInvalidSlot ? kNoSource : cache_row >= 0 ? cache_row : ~static_cast<int32_t>(g);
}
__device__ __forceinline__ const float* src_of_word(const RowSrc& rs, const TableDev& tb, int32_t w, int D) {
  if (w >= 0) return rs.cache + static_cast<int64_t>(w) * D;
  if (w == kNoSource) return nullptr;
  const uint32_t g = static_cast<uint32_t>(~w);
  if (rs.local_hbm) return tb.store + static_cast<int64_t>(rs.uniq[g]) * D;
  return rs.urows + static_cast<int64_t>(g) * D;
}

// Reset tail of a direct-source pool (what k_gather does on the gathering
// path): the batch's dedup-set slots go back to empty, and the gradient rows
// of its misses (the only ones k_scatter<SGD> accumulates) start at zero.
struct ResetOut {
  const int* ctr;
  const uint16_t* utab;
  const uint32_t* uslot;
  const int32_t* usrc;
  float* ugrad;
  int* cnt;  // per-unique add counters of the fused SGD scatter
  // set slots the batch's dedup left behind: kResetAll (tile / per-table
  // kernels: every unique's slot and idcnt), kResetMisses (cluster kernel
  // with `tag`: the tagged misses), kResetNone (cluster kernel, no tags)
  int hash_reset;
};
constexpr int kResetNone = 0, kResetMisses = 1, kResetAll = 2;
template <int VEC>
__device__ __forceinline__ void reset_sets(const TableDev* td, int T, const ResetOut& ro, int b, int nb) {
  constexpr int D = VEC * 4;
  constexpr int RPW = 32 / VEC;
  const int U = counters(const_cast<int*>(ro.ctr), T).ubase[T];
  const int sub = lane_id() / VEC, c = lane_id() % VEC;
  const int warp = (b * blockDim.x + threadIdx.x) >> 5, nwarps = (nb * blockDim.x) >> 5;
  for (int g = warp * RPW + sub; g < U; g += nwarps * RPW) {
    const bool miss = ro.usrc[g] < 0;
    if (c == 0) {
      if (ro.hash_reset == kResetAll || (ro.hash_reset == kResetMisses && miss)) {
        const TableDev& tb = td[ro.utab[g]];
        *set_word(tb, ro.uslot[g]) = kEmptySlot;
        if (ro.hash_reset == kResetAll) tb.idcnt[ro.uslot[g]] = 0;
      }
      ro.cnt[g] = 0;
    }
    if (miss) st4(ro.ugrad + static_cast<int64_t>(g) * D + c * 4, make_float4(0.f, 0.f, 0.f, 0.f));
  }
}

// Bags visited sample-major (q = s*T + t) so a warp writes a contiguous
// stretch of the [B, T*D] output; R bags in flight per thread; each bag is
// summed in lookup order.
template <int VEC, int R, bool DIRECT = false, bool RSRC = false>
__global__ void __launch_bounds__(kThreads, 4) k_pool(const TableDev* __restrict__ td, int T, int B, int P,
                                                   const int64_t* __restrict__ bag_off, const uint32_t* __restrict__ inv,
                                                   const float* __restrict__ urows, float* __restrict__ out,
                                                   RowSrc rs = {}, int pool_blocks = 0, ResetOut ro = {}) {
  constexpr int D = VEC * 4;
  constexpr int RPW = RowMap<VEC>::kRowsPerWarp;
  const RowMap<VEC> m;
  const int nbags = T * B;
  if (DIRECT && static_cast<int>(blockIdx.x) >= pool_blocks) {
    reset_sets<VEC>(td, T, ro, blockIdx.x - pool_blocks, gridDim.x - pool_blocks);
    return;
  }
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = ((DIRECT ? pool_blocks : gridDim.x) * blockDim.x) >> 5;
  for (int q0 = warp * RPW * R; q0 < nbags; q0 += nwarps * RPW * R) {
    int lo[R], len[R];  // batch positions < 2^31 (checked by Engine::forward)
    int maxlen = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int q = q0 + r * RPW + m.sub;
      lo[r] = 0;
      len[r] = 0;
      if (q < nbags) {
        const int s = q / T, t = q - s * T;
        int64_t l64, h64;
        bag_range(td, bag_off, B, P, s, t, &l64, &h64);
        lo[r] = static_cast<int>(l64);
        len[r] = static_cast<int>(h64 - l64);
        maxlen = max(maxlen, len[r]);
      }
    }
    float4 acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int i = 0; i < maxlen; ++i) {
      uint32_t u[R];
      if constexpr (RSRC) {
#pragma unroll
        for (int r = 0; r < R; ++r) u[r] = i < len[r] ? static_cast<uint32_t>(rs.isrc[lo[r] + i]) : kNoSource;
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) u[r] = i < len[r] ? inv[lo[r] + i] : kInvalidSlot;
      }
      if constexpr (DIRECT) {
        const float* src[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int q = q0 + r * RPW + m.sub;
          const TableDev& tb = td[q - (q / T) * T];
          if constexpr (RSRC) src[r] = src_of_word(rs, tb, static_cast<int32_t>(u[r]), D);
          else src[r] = u[r] == kInvalidSlot ? nullptr : src_row(rs, tb, u[r], D);
        }
#pragma unroll
        for (int r = 0; r < R; ++r)
          if (src[r]) acc[r] = add4(acc[r], ldg4(src[r] + m.c * 4));
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = add4(acc[r], load_row(urows, u[r], D, m.c));
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int q = q0 + r * RPW + m.sub;
      if (q < nbags) st4(out + static_cast<int64_t>(q) * D + m.c * 4, acc[r]);  // q = s*T + t
    }
  }
}

// Pooling 1 (the Criteo configs): every bag is one lookup, so the pool is an
// indexed row copy; R bags in flight per thread, evict-first stores for the
// [B, T*D] output (written once, not re-read by this step).
template <int VEC, int R, bool DIRECT = false, bool RSRC = false>
__global__ void __launch_bounds__(kThreads) k_pool1(const TableDev* __restrict__ td, int T, int B,
                                                    const uint32_t* __restrict__ inv, const float* __restrict__ urows,
                                                    float* __restrict__ out, RowSrc rs = {}, int pool_blocks = 0,
                                                    ResetOut ro = {}) {
  constexpr int D = VEC * 4;
  constexpr int RPW = RowMap<VEC>::kRowsPerWarp;
  const RowMap<VEC> m;
  const int nbags = T * B;
  if (DIRECT && static_cast<int>(blockIdx.x) >= pool_blocks) {
    reset_sets<VEC>(td, T, ro, blockIdx.x - pool_blocks, gridDim.x - pool_blocks);
    return;
  }
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = ((DIRECT ? pool_blocks : gridDim.x) * blockDim.x) >> 5;
  for (int q0 = warp * RPW * R; q0 < nbags; q0 += nwarps * RPW * R) {
    uint32_t u[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int q = q0 + r * RPW + m.sub;
      u[r] = RSRC ? static_cast<uint32_t>(kNoSource) : kInvalidSlot;
      if (q < nbags) {
        const int s = q / T, t = q - s * T;
        // pooling 1: table t's lookups start at t*B
        u[r] = __ldcs((RSRC ? reinterpret_cast<const uint32_t*>(rs.isrc) : inv) + static_cast<int64_t>(t) * B + s);
      }
    }
    float4 v[R];
    if constexpr (DIRECT) {
      const float* src[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int q = q0 + r * RPW + m.sub;
        const TableDev& tb = td[q - (q / T) * T];
        if constexpr (RSRC) src[r] = src_of_word(rs, tb, static_cast<int32_t>(u[r]), D);
        else src[r] = u[r] == kInvalidSlot ? nullptr : src_row(rs, tb, u[r], D);
      }
#pragma unroll
      for (int r = 0; r < R; ++r) v[r] = src[r] ? ldg4(src[r] + m.c * 4) : make_float4(0.f, 0.f, 0.f, 0.f);
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) v[r] = load_row(urows, u[r], D, m.c);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int q = q0 + r * RPW + m.sub;
      if (q < nbags) __stcs(reinterpret_cast<float4*>(out + static_cast<int64_t>(q) * D + m.c * 4), v[r]);
    }
  }
}

// ------------------------------------------------- fp64 gradient sums
// Unique-row gradient sums that many lookups feed are kept in fp64 so the
// SGD update is one rounding of w - lr * sum(g) (north_star: updated rows
// within 1e-5 relative of the fp64 restatement; fp32 adds of thousands of
// gradients into one row drift past that).  Layout interleaved per row so the
// VEC lanes of a row touch one contiguous stretch per component: element
// (unique g, lane c, component k) lives at g*D + k*VEC + c.
template <int VEC>
__device__ __forceinline__ void red_g64(double* g64, int64_t g, int c, double x, double y, double z, double w) {
  double* p = g64 + g * (VEC * 4) + c;
  atomicAdd(p, x);
  atomicAdd(p + VEC, y);
  atomicAdd(p + 2 * VEC, z);
  atomicAdd(p + 3 * VEC, w);
}
// read a row's sums and leave zeros behind (the buffer is self-cleaning)
template <int VEC>
__device__ __forceinline__ void take_g64(double* g64, int64_t g, int c, double* out) {
  double* p = g64 + g * (VEC * 4) + c;
#pragma unroll
  for (int k = 0; k < 4; ++k) out[k] = __ldcg(p + k * VEC);
#pragma unroll
  for (int k = 0; k < 4; ++k) p[k * VEC] = 0.0;
}
__device__ __forceinline__ float4 sgd4(float4 w, const double* gs, float lr) {
  const double l = lr;
  return make_float4(static_cast<float>(w.x - l * gs[0]), static_cast<float>(w.y - l * gs[1]),
                     static_cast<float>(w.z - l * gs[2]), static_cast<float>(w.w - l * gs[3]));
}

// ------------------------------------------------------------------ K6
// Each warp owns a contiguous range of one table's bags (whole R-slot windows
// of RPW bags), so hot rows repeat inside the warp many times over.  Per
// window, lanes holding the same row (same component c) are summed with
// shuffles.  Then, by the row's lookup count in the batch (the dedup's
// `ucount`):
//   * light rows (<= kLightAdds lookups) leave as one fp32 RED per window (SGD:
//     -lr * v straight into the cache / HBM row; else into ugrad): at most
//     kLightAdds roundings, <= 3.8e-6 of the magnitudes summed;
//   * heavy rows go to the row's fp64 sum in g64, rounded once by
//     k_apply_g64 / k_g64_finalize -- through the warp's private shared-memory
//     accumulator when the row is among the table's first kAcc uniques (first-
//     occurrence order puts a table's heaviest ids there; plain read-modify-
//     write, a window's leaders hold distinct rows), flushed once per range.
// Without counts (ucount null) every row takes the fp64 path.  Measured
// (profiles/r02/parity.md): the all-fp32 scatter left the 3-row Kaggle tables'
// rows 1.1e-5 off (~2K adds each, north_star bar 1e-5); fp64 REDs per window
// for heavy rows cost +30 us (same-address atomics on a 3-row table's rows),
// which the per-warp accumulators remove: 26 us standalone (r01 fp32: 28 us).
constexpr int kLightAdds = 64;

template <int VEC>
struct ScatterAcc {
  static constexpr int D = VEC * 4;
  static constexpr int kRows = 1024 / D < 8 ? 8 : (1024 / D > 64 ? 64 : 1024 / D);  // rows per warp accumulator
};

template <int VEC, int R, bool SGD = false>
__global__ void __launch_bounds__(kThreads, 4) k_scatter(const TableDev* __restrict__ td, int T, int B, int P,
                                                         const int64_t* __restrict__ bag_off,
                                                         const uint32_t* __restrict__ inv, const float* __restrict__ grad,
                                                         float* __restrict__ ugrad, double* __restrict__ g64,
                                                         const int* __restrict__ ucount, const int* __restrict__ ctr,
                                                         RowSrc rs = {}, float lr = 0.f) {
  constexpr int D = VEC * 4;
  constexpr int RPW = RowMap<VEC>::kRowsPerWarp;
  constexpr int kAcc = ScatterAcc<VEC>::kRows;
  __shared__ __align__(16) float sacc[kThreads / 32][kAcc * D];
  const RowMap<VEC> m;
  const int wib = threadIdx.x >> 5;
  float* acc = sacc[wib];
  const Counters cn = counters(const_cast<int*>(ctr), T);
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int i = lane_id(); i < kAcc * VEC; i += 32) st4(acc + i * 4, make_float4(0.f, 0.f, 0.f, 0.f));
  __syncwarp();
  // ranges of whole R-slot windows (RPW * R bags), about one per warp
  const int win = RPW * R;
  const int per = max(1, (B + max(1, nwarps / T) - 1) / max(1, nwarps / T) + win - 1) / win * win;
  const int wt = (B + per - 1) / per;  // ranges per table

  // a light row's partial leaves as an fp32 RED (SGD: -lr * v into its cache /
  // HBM row; else into ugrad)
  auto emit_light = [&](uint32_t u, int t, int32_t sr, float4 v) {
    float* dst = ugrad + static_cast<int64_t>(u) * D;
    if constexpr (SGD) {
      if (sr >= 0 || rs.local_hbm) {
        dst = sr >= 0 ? const_cast<float*>(rs.cache) + static_cast<int64_t>(sr) * D
                      : td[t].store + static_cast<int64_t>(rs.uniq[u]) * D;
        v = make_float4(-lr * v.x, -lr * v.y, -lr * v.z, -lr * v.w);
      }
    }
    atomicAdd(reinterpret_cast<float4*>(dst + m.c * 4), v);
  };

  for (int item = warp; item < T * wt; item += nwarps) {
    const int t = item / wt;
    const int b0 = (item - t * wt) * per, b1 = min(B, b0 + per);
    if (b0 >= b1) continue;
    const uint32_t ub = static_cast<uint32_t>(cn.ubase[t]);
    const int nacc = min(kAcc, cn.ubase[t + 1] - cn.ubase[t]);
    uint64_t touched = 0;  // accumulator rows this lane wrote (the rows are zero between ranges)
    for (int s0 = b0; s0 < b1; s0 += RPW * R) {
      int lo[R], len[R], maxlen = 0;
      float4 gv[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int sb = s0 + r * RPW + m.sub;
        lo[r] = 0;
        len[r] = 0;
        gv[r] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (sb < b1) {
          int64_t l64, h64;
          bag_range(td, bag_off, B, P, sb, t, &l64, &h64);
          lo[r] = static_cast<int>(l64);
          len[r] = static_cast<int>(h64 - l64);
          maxlen = max(maxlen, len[r]);
          gv[r] = ld_stream4(grad + (static_cast<int64_t>(sb) * T + t) * D + m.c * 4);
        }
      }
      maxlen = __reduce_max_sync(kFull, maxlen);
      for (int i = 0; i < maxlen; ++i) {
        uint32_t u[R];
#pragma unroll
        for (int r = 0; r < R; ++r) u[r] = i < len[r] ? inv[lo[r] + i] : kInvalidSlot;
        // every slot's count (and SGD source) in flight before the pre-sums
        int cnt[R];
        int32_t srr[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          cnt[r] = u[r] != kInvalidSlot ? (ucount ? __ldcg(ucount + u[r]) : kLightAdds + 1) : 0;
          srr[r] = SGD && u[r] != kInvalidSlot ? rs.usrc[u[r]] : 0;
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
          float4 v = gv[r];
          bool lead = u[r] != kInvalidSlot;
          if (RPW > 1 && __any_sync(kFull, __popc(__match_any_sync(kFull, u[r])) > VEC)) {
            // some row repeats in this window: rotate by whole bags (same component c)
#pragma unroll
            for (int k = 1; k < RPW; ++k) {
              const int src = (lane_id() + k * VEC) & 31;
              const uint32_t uo = __shfl_sync(kFull, u[r], src);
              const float4 o = make_float4(__shfl_sync(kFull, gv[r].x, src), __shfl_sync(kFull, gv[r].y, src),
                                           __shfl_sync(kFull, gv[r].z, src), __shfl_sync(kFull, gv[r].w, src));
              if (uo == u[r]) {
                if (src < lane_id()) lead = false;  // a lower bag owns this row
                else v = add4(v, o);
              }
            }
          }
          // heavy rows (more than kLightAdds lookups): the warp accumulator if
          // among the table's first kAcc uniques, else the fp64 sum
          const int n = cnt[r];
          const int32_t sr = srr[r];
          const uint32_t local = u[r] - ub;
          if (lead && n > kLightAdds) {
            if (local < static_cast<uint32_t>(nacc)) {
              float* a = acc + local * D + m.c * 4;
              st4(a, add4(*reinterpret_cast<const float4*>(a), v));
              touched |= 1ull << local;
            } else {
              red_g64<VEC>(g64, u[r], m.c, v.x, v.y, v.z, v.w);
            }
          } else if (lead) {
            emit_light(u[r], t, sr, v);
          }
          __syncwarp();  // the next slot's leaders read what this one wrote
        }
      }
    }
    // flush the accumulator rows this warp touched (union over lanes) into
    // their fp64 sums and zero them: lane group `sub` takes every RPW-th row
    uint64_t tall = touched;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tall |= __shfl_xor_sync(kFull, tall, o);
    __syncwarp();
    for (int k = 0; k < m.sub && tall; ++k) tall &= tall - 1;
    while (tall) {
      const int row = __ffsll(static_cast<long long>(tall)) - 1;
      float* a = acc + row * D + m.c * 4;
      const float4 x = *reinterpret_cast<const float4*>(a);
      st4(a, make_float4(0.f, 0.f, 0.f, 0.f));
      red_g64<VEC>(g64, ub + static_cast<uint32_t>(row), m.c, x.x, x.y, x.z, x.w);
      for (int k = 0; k < RPW && tall; ++k) tall &= tall - 1;
    }
    __syncwarp();
  }
}

// Fused single-rank SGD, pinned-host tier: a miss's new row.  A miss heavier
// than kLightAdds lookups (every miss without counts) has its whole gradient
// in g64 -- w - lr * sum rounded once, read without clearing, so the host
// write-back and the prefetch patch (two streams) compute the same row; a
// light one sums in ugrad.  `g64` null: the gradient is in ugrad (other paths).
template <int VEC>
__device__ __forceinline__ float4 miss_sgd(float4 w, const float* __restrict__ ugrad, const double* __restrict__ g64,
                                           const int* __restrict__ ucount, uint32_t g, int c, float lr) {
  constexpr int D = VEC * 4;
  if (g64 && (!ucount || __ldcg(ucount + g) > kLightAdds)) {
    const double* p = g64 + static_cast<int64_t>(g) * D + c;
    double gs[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) gs[k] = __ldcg(p + k * VEC);
    return sgd4(w, gs, lr);
  }
  const float4 gr = ldg4(ugrad + static_cast<int64_t>(g) * D + c * 4);
  return make_float4(w.x - lr * gr.x, w.y - lr * gr.y, w.z - lr * gr.z, w.w - lr * gr.w);
}

// Fused single-rank SGD, pinned-host tier without per-unique counts (dedup by
// the tile path: every row took the fp64 path): each miss's fp64 sum rounded
// into ugrad for the host write-back, sums and counts left zeroed.  Walks the
// miss queue.  (With counts the write-back reads the heavy misses' sums itself
// -- miss_sgd -- and k_clear_miss_sums clears them before the set's next dedup.)
template <int VEC>
__global__ void __launch_bounds__(kThreads) k_g64_misses(int T, const int* __restrict__ ctr,
                                                         const uint32_t* __restrict__ missq, int* __restrict__ ucount,
                                                         float* __restrict__ ugrad, double* __restrict__ g64) {
  constexpr int D = VEC * 4;
  constexpr int RPW = RowMap<VEC>::kRowsPerWarp;
  constexpr int R = 4;
  const RowMap<VEC> m;
  const int nm = *counters(const_cast<int*>(ctr), T).miss_total;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int q0 = warp * RPW * R; q0 < nm; q0 += nwarps * RPW * R) {
    uint32_t g[R];
    int n[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int q = q0 + r * RPW + m.sub;
      g[r] = q < nm ? missq[q] : kInvalidSlot;
    }
#pragma unroll
    for (int r = 0; r < R; ++r) n[r] = g[r] == kInvalidSlot ? 0 : ucount ? __ldcg(ucount + g[r]) : kLightAdds + 1;
    __syncwarp();  // every lane of a row read its count before lane 0 clears it
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (g[r] == kInvalidSlot) continue;
      if (ucount && m.c == 0) ucount[g[r]] = 0;
      if (n[r] <= kLightAdds) continue;
      double gs[4];
      take_g64<VEC>(g64, g[r], m.c, gs);
      float* dst = ugrad + static_cast<int64_t>(g[r]) * D + m.c * 4;
      const float4 w = *reinterpret_cast<const float4*>(dst);
      st4(dst, make_float4(static_cast<float>(w.x + gs[0]), static_cast<float>(w.y + gs[1]),
                           static_cast<float>(w.z + gs[2]), static_cast<float>(w.w + gs[3])));
    }
  }
}

// Before a buffer set's next dedup, on that dedup's stream (off the host
// link's path): every per-unique count its last batch left (the fused host
// tier's misses, read by their write-back; any batch whose backward never ran,
// e.g. a dropped prefetch), and the fp64 sums of the rows those counts made
// heavy.  Reads the last batch's counters, so it runs before their reset.
template <int VEC>
__global__ void __launch_bounds__(kThreads) k_clear_miss_sums(int T, const int* __restrict__ ctr,
                                                              int* __restrict__ ucount, double* __restrict__ g64) {
  constexpr int D = VEC * 4;
  const int n = counters(const_cast<int*>(ctr), T).ubase[T];
  // one count per thread (coalesced, all in flight); a heavy row's D sums by
  // its own thread (rare).  (One row per lane group, as the row kernels do,
  // left 16 lanes per count at D = 64: 117 us for the TB shape's 266K uniques.)
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < n; g += gridDim.x * blockDim.x) {
    const int cnt = __ldcg(ucount + g);
    if (!cnt) continue;
    ucount[g] = 0;
    if (cnt > kLightAdds) {
      double2* p = reinterpret_cast<double2*>(g64 + static_cast<int64_t>(g) * D);
#pragma unroll 4
      for (int k = 0; k < D / 2; ++k) p[k] = make_double2(0.0, 0.0);
    }
  }
}

// Fused single-rank SGD, second half: rows heavier than kLightAdds (their
// partials went to g64) get w - lr * sum(g64) with one rounding (cache row,
// or the HBM shard row of a miss).  Pinned-host misses are the host
// write-back's (miss_sgd; skipped here, their sums cleared by
// k_clear_miss_sums).  Leaves the other rows' g64 and ucount zeroed.
template <int VEC>
__global__ void __launch_bounds__(kThreads) k_apply_g64(const TableDev* __restrict__ td, int T, const int* __restrict__ ctr,
                                                        const uint32_t* __restrict__ uniq, const uint16_t* __restrict__ utab,
                                                        const int32_t* __restrict__ usrc, int* __restrict__ ucount,
                                                        float* __restrict__ cache, float* __restrict__ ugrad,
                                                        double* __restrict__ g64, float lr, int local_hbm) {
  constexpr int D = VEC * 4;
  constexpr int RPW = RowMap<VEC>::kRowsPerWarp;
  constexpr int R = 4;  // rows per lane group in flight
  const RowMap<VEC> m;
  const int U = counters(const_cast<int*>(ctr), T).ubase[T];
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int g0 = warp * RPW * R; g0 < U; g0 += nwarps * RPW * R) {
    int n[R];
    bool own[R];  // not a pinned-host miss (those are the host write-back's)
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int g = g0 + r * RPW + m.sub;
      own[r] = g < U && (local_hbm || usrc[g] >= 0);
      n[r] = own[r] ? (ucount ? __ldcg(ucount + g) : kLightAdds + 1) : 0;
    }
    __syncwarp();
    if (ucount && m.c == 0) {
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (own[r]) ucount[g0 + r * RPW + m.sub] = 0;
    }
    double gs[R][4];
    float* dst[R];
    float4 w[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int g = g0 + r * RPW + m.sub;
      dst[r] = nullptr;
      if (n[r] <= kLightAdds) continue;
      take_g64<VEC>(g64, g, m.c, gs[r]);
      const int32_t s = usrc[g];
      dst[r] = s >= 0 ? cache + static_cast<int64_t>(s) * D : td[utab[g]].store + static_cast<int64_t>(uniq[g]) * D;
    }
#pragma unroll
    for (int r = 0; r < R; ++r) w[r] = dst[r] ? *reinterpret_cast<const float4*>(dst[r] + m.c * 4) : float4{};
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (dst[r]) st4(dst[r] + m.c * 4, sgd4(w[r], gs[r], lr));
  }
}

// SGD on every unique row: w = w_gathered - lr * g, written to the cache copy
// (hits) or, for misses whose shard is in HBM, to the owning local shard.
template <int VEC, int R>
__global__ void __launch_bounds__(kThreads) k_apply(const TableDev* __restrict__ td, int T, const int* __restrict__ ctr,
                                                    const uint32_t* __restrict__ uniq, const uint16_t* __restrict__ utab,
                                                    const int32_t* __restrict__ usrc, const float* __restrict__ urows,
                                                    const float* __restrict__ ugrad, float lr, float* __restrict__ cache,
                                                    int hits, int misses_local, int rank, int world,
                                                    const int* __restrict__ off = nullptr, double* __restrict__ g64 = nullptr,
                                                    int skip_sole = 0) {
  constexpr int D = VEC * 4;
  constexpr int RPW = RowMap<VEC>::kRowsPerWarp;
  const RowMap<VEC> m;
  const int U = counters(const_cast<int*>(ctr), T).ubase[T];
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int g0 = warp * RPW * R; g0 < U; g0 += nwarps * RPW * R) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int g = g0 + r * RPW + m.sub;
      if (g >= U) continue;
      if (skip_sole && chunk_span(off[g], off[g + 1]) == 1) continue;  // k_bwd_reduce applied it
      const int32_t s = usrc[g];
      float* dst = nullptr;
      if (s >= 0) {
        if (hits) dst = cache + static_cast<int64_t>(s) * D;
      } else if (misses_local) {
        const uint32_t id = uniq[g];
        if (static_cast<int>(id % world) == rank) dst = td[utab[g]].store + static_cast<int64_t>(id / world) * D;
      }
      if (!dst) continue;
      const float4 w = ldg4(urows + static_cast<int64_t>(g) * D + m.c * 4);
      if (off && chunk_span(off[g], off[g + 1]) > kLightAdds) {
        // (k_g64_finalize folded in) a row spread over many k_bwd_reduce chunks:
        // its fp64 sum, one rounding
        double gs[4];
        take_g64<VEC>(g64, g, m.c, gs);
        st4(dst + m.c * 4, sgd4(w, gs, lr));
        continue;
      }
      const float4 gr = ldg4(ugrad + static_cast<int64_t>(g) * D + m.c * 4);
      st4(dst + m.c * 4, make_float4(w.x - lr * gr.x, w.y - lr * gr.y, w.z - lr * gr.z, w.w - lr * gr.w));
    }
  }
}

// SGD for cold rows held in pinned host memory (miss queue, side stream).
template <int VEC, int R>
__global__ void __launch_bounds__(kThreads) k_apply_host(const TableDev* __restrict__ td, int T, const int* __restrict__ ctr,
                                                         const uint32_t* __restrict__ missq,
                                                         const uint32_t* __restrict__ uniq,
                                                         const uint16_t* __restrict__ utab, const float* __restrict__ urows,
                                                         const float* __restrict__ ugrad, float lr, int rank, int world,
                                                         const double* __restrict__ g64 = nullptr,
                                                         const int* __restrict__ ucount = nullptr) {
  constexpr int D = VEC * 4;
  constexpr int RPW = RowMap<VEC>::kRowsPerWarp;
  const RowMap<VEC> m;
  const int nm = *counters(const_cast<int*>(ctr), T).miss_total;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int q0 = warp * RPW * R; q0 < nm; q0 += nwarps * RPW * R) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int q = q0 + r * RPW + m.sub;
      if (q >= nm) continue;
      const uint32_t g = missq[q];
      const uint32_t id = uniq[g];
      if (static_cast<int>(id % world) != rank) continue;
      const float4 w = ldg4(urows + static_cast<int64_t>(g) * D + m.c * 4);
      const float4 nw = miss_sgd<VEC>(w, ugrad, g64, ucount, g, m.c, lr);
      st4(td[utab[g]].store + static_cast<int64_t>(id / world) * D + m.c * 4, nw);
    }
  }
}

// A prefetched next batch gathered its host rows before this batch's SGD
// reached the host tier: for every row this batch updates, find it in the next
// batch's hash (id -> tagged unique index, left by its dedup) and refresh the
// copy with the new value.  On-device only; the host write-back runs apart.
template <int VEC, int R>
__global__ void __launch_bounds__(kThreads) k_patch_prefetch(const TableDev* __restrict__ td, int T,
                                                             const int* __restrict__ ctr,
                                                             const uint32_t* __restrict__ missq,
                                                             const uint32_t* __restrict__ uniq,
                                                             const uint16_t* __restrict__ utab,
                                                             const float* __restrict__ urows,
                                                             const float* __restrict__ ugrad, float lr, int rank,
                                                             int world, const int32_t* __restrict__ nxt_usrc,
                                                             float* __restrict__ nxt_urows,
                                                             const double* __restrict__ g64 = nullptr,
                                                             const int* __restrict__ ucount = nullptr) {
  constexpr int D = VEC * 4;
  constexpr int RPW = RowMap<VEC>::kRowsPerWarp;
  const RowMap<VEC> m;
  const int nm = *counters(const_cast<int*>(ctr), T).miss_total;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int q0 = warp * RPW * R; q0 < nm; q0 += nwarps * RPW * R) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int q = q0 + r * RPW + m.sub;
      if (q >= nm) continue;
      const uint32_t g = missq[q];
      const uint32_t id = uniq[g];
      if (static_cast<int>(id % world) != rank) continue;
      const TableDev tb = td[utab[g]];
      uint32_t h = table_slot(tb, id);
      for (;;) {
        const unsigned long long v = __ldcg(set_word(tb, h));
        if (v == kEmptySlot) break;
        if (static_cast<uint32_t>(v >> 32) == id) {
          const uint32_t g2 = static_cast<uint32_t>(v) & ~kRankTag;
          if (nxt_usrc[g2] < 0) {
            const float4 w = ldg4(urows + static_cast<int64_t>(g) * D + m.c * 4);
            st4(nxt_urows + static_cast<int64_t>(g2) * D + m.c * 4, miss_sgd<VEC>(w, ugrad, g64, ucount, g, m.c, lr));
          }
          break;
        }
        h = (h + 1) & tb.mask;
      }
    }
  }
}

// Drop the hash entries of a prefetched batch that will not be consumed.
__global__ void k_clear_hash(const TableDev* __restrict__ td, int T, const int* __restrict__ ctr,
                             const uint16_t* __restrict__ utab, const uint32_t* __restrict__ uslot) {
  const int U = counters(const_cast<int*>(ctr), T).ubase[T];
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < U; g += gridDim.x * blockDim.x) {
    const TableDev& tb = td[utab[g]];
    *set_word(tb, uslot[g]) = kEmptySlot;
    tb.idcnt[uslot[g]] = 0;
  }
}

}  // namespace ec


// ===================================================================
// K1 + K2 in one kernel: one thread-block cluster per table.
//
// Needs every table's dedup set direct-mapped (slot = id; engine.cu sizes
// those sets at creation).  The batch of a table is split into kClusterCtas
// contiguous chunks, one per CTA; inside a CTA each thread owns up to ITEMS
// consecutive positions (thread-major), so the rank of a first occurrence is
// an exclusive scan of per-thread counts plus a popcount inside the thread.
// Ids and per-item state stay in registers for the whole kernel.
//
//   L  hot ids (id < kClusterLocal: the top ranks of a parametric table, or
//      all of a small table) are deduplicated per CTA in shared memory
//      (direct-mapped atomicMin after a warp match-any collapse): the L2 set
//      then sees one insert per (CTA, hot id) instead of thousands of
//      same-address atomics.  Colder ids go straight to L2.
//   G  representatives: one 64-bit atomicMin (id << 32 | position) on the
//      id's slot keeps its first position                  -- cluster barrier
//   F  each representative reads its id's first position p_f; firsts are the
//      representatives with p_f == own position; CTA scan; per-thread words
//      (exclusive count << 16 | first mask) to shared memory -- cluster barrier
//   B  unique base: CTA totals over DSMEM; table totals by a warp-parallel
//      look-back over the lower tables (clusters are dispatched in order)
//   E  unique index of every representative: its own rank if first, else
//      computed from p_f and the owning thread's word (DSMEM) -- no third
//      barrier and no re-read of the L2 set; emit the firsts with the K2
//      hit/miss partition (usrc, miss queue, per-table miss counts); empty
//      their L2 slots, or with `tag` tag the misses' (read by k_patch_prefetch)
//   I  inverse: representatives hold their index, hot duplicates read it from
//      shared memory; with RSRC, each lookup's row source into `isrc` (the fused
//      pool then reads one word per lookup and the row: no inverse -> usrc hop)
// ===================================================================
#ifdef EC_TRACE  // phase timestamps for tools/dedup_bench.cu only
__device__ unsigned long long* g_trace;
#define EC_TRACE_AT(ph)                                                       \
  do {                                                                       \
    if (g_trace && threadIdx.x == 0) {                                       \
      unsigned long long ns;                                                 \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));                 \
      g_trace[blockIdx.x * 8 + (ph)] = ns;                                   \
    }                                                                        \
  } while (0)
#else
#define EC_TRACE_AT(ph) \
  do {                  \
  } while (0)
#endif

namespace ec {

namespace cg = cooperative_groups;
#ifndef EC_CLUSTER_CTAS
#define EC_CLUSTER_CTAS 8
#endif
constexpr int kClusterCtas = EC_CLUSTER_CTAS;
#ifndef EC_CLUSTER_THREADS
#define EC_CLUSTER_THREADS 512
#endif
constexpr int kClusterThreads = EC_CLUSTER_THREADS;
constexpr int kClusterMaxItems = 16;     // per thread -> n_t <= 8 * 512 * 16 = 65536
constexpr uint32_t kClusterLocal = 16384;  // hot ids deduplicated in shared memory
// per-table look-back word: count [0,32), CTA arrivals [32,40), inclusive flag
constexpr unsigned long long kTabInc = 1ull << 40;
__host__ __device__ constexpr size_t cluster_smem_bytes(int) { return kClusterLocal * sizeof(uint32_t); }


template <int ITEMS, bool RSRC = false>
__global__ void __cluster_dims__(kClusterCtas, 1, 1)
__launch_bounds__(kClusterThreads, kClusterThreads >= 512 ? (ITEMS <= 4 ? 2 : 1) : (ITEMS <= 8 ? 3 : 2))
    k_dedup_cluster(const TableDev* __restrict__ td, int T, const uint32_t* __restrict__ indices,
                    unsigned long long* __restrict__ tstatus, int* __restrict__ ctr, uint32_t* __restrict__ uniq,
                    uint32_t* __restrict__ uslot, uint16_t* __restrict__ utab, uint32_t* __restrict__ inv,
                    int32_t* __restrict__ usrc, uint32_t* __restrict__ missq, int* __restrict__ ucount, int tag,
                    int32_t* __restrict__ isrc = nullptr) {
  static_assert(ITEMS <= 16, "per-thread first masks are 16 bits");
  extern __shared__ __align__(16) uint32_t sval[];  // hot id -> local min position, later its unique index
  __shared__ uint32_t sxm[kClusterThreads];          // per thread: (exclusive first count << 16) | first mask
  __shared__ int s_total, s_base, s_qbase, s_pref[kClusterCtas];
  __shared__ int sw[kClusterThreads / 32];
  cg::cluster_group cluster = cg::this_cluster();
  const unsigned crank = cluster.block_rank();
  // clusters are dispatched in blockIdx order, so every lower table is running
  // or done when this one looks back (the forward-progress rule of a
  // decoupled-look-back scan over blockIdx)
  const int t = static_cast<int>(blockIdx.x) / kClusterCtas;
  EC_TRACE_AT(0);
  Counters c = counters(ctr, T);
  const TableDev tb = td[t];
  const int64_t n = tb.n;
  const int64_t chunk = (n + kClusterCtas - 1) / kClusterCtas;
  const int64_t c0 = min(n, static_cast<int64_t>(crank) * chunk), c1 = min(n, c0 + chunk);
  const int items = static_cast<int>((c1 - c0 + kClusterThreads - 1) / kClusterThreads);
  const int64_t p0 = c0 + static_cast<int64_t>(threadIdx.x) * items;  // this thread's first position
  const int my = static_cast<int>(max(int64_t{0}, min(static_cast<int64_t>(items), c1 - p0)));
  const uint32_t nloc = tb.rows < kClusterLocal ? static_cast<uint32_t>(tb.rows) : kClusterLocal;
  uint32_t id[ITEMS];
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) id[j] = j < my ? __ldcs(indices + tb.base + p0 + j) : kEmptyKey;
  {  // clear the hot-id slots (while the ids are in flight)
    uint4* s4 = reinterpret_cast<uint4*>(sval);
    const uint4 e = make_uint4(kEmptyKey, kEmptyKey, kEmptyKey, kEmptyKey);
    for (uint32_t i = threadIdx.x; i < (nloc + 3) / 4; i += kClusterThreads) s4[i] = e;
  }
  __syncthreads();
  EC_TRACE_AT(1);

  // ---- L: local representatives of hot ids
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    if (j < my && id[j] >= tb.rows) {
      atomicExch(c.err, 1);
      id[j] = kEmptyKey;  // out of range: skipped, inverse = kInvalidSlot
    }
    const uint32_t key = id[j] < nloc ? id[j] : kEmptyKey;
    const unsigned peers = __match_any_sync(kFull, key);
    // lowest lane of a group = its smallest position
    if (key != kEmptyKey && __ffs(peers) - 1 == lane_id()) atomicMin(sval + key, static_cast<uint32_t>(p0 + j));
  }
  __syncthreads();
  EC_TRACE_AT(2);

  // ---- G: representatives insert into the direct-mapped L2 set.  With
  // RSRC every lookup needs its remap entry (phase I): loaded here, in
  // flight across both cluster barriers (duplicates share the first's sector)
  uint32_t rep = 0;
  int32_t rm[ITEMS];
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const bool r = id[j] < nloc ? sval[id[j]] == static_cast<uint32_t>(p0 + j) : id[j] != kEmptyKey;
    if (r) {
      rep |= 1u << j;
      atomicMin(set_word(tb, id[j]), (static_cast<unsigned long long>(id[j]) << 32) | static_cast<uint32_t>(p0 + j));
    }
    if constexpr (RSRC) rm[j] = id[j] != kEmptyKey ? set_remap(tb, id[j]) : 0;
  }
  EC_TRACE_AT(3);
  cluster.sync();  // every insert of this table is done

  // ---- F: first positions; firsts; CTA scan
  uint32_t pf[ITEMS], first = 0;
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) pf[j] = ((rep >> j) & 1) ? static_cast<uint32_t>(__ldcg(set_word(tb, id[j]))) : 0u;
#pragma unroll
  for (int j = 0; j < ITEMS; ++j)
    if (((rep >> j) & 1) && pf[j] == static_cast<uint32_t>(p0 + j)) first |= 1u << j;
  int total;
  const int ex = block_exclusive_scan<kClusterThreads>(__popc(first), sw, &total);
  sxm[threadIdx.x] = (static_cast<uint32_t>(ex) << 16) | first;
  if (threadIdx.x == 0) {
    s_total = total;
    // table aggregate: every CTA adds (1 << 32 | its count); complete at 8 arrivals
    atomicAdd(tstatus + t, (1ull << 32) | static_cast<uint32_t>(total));
  }
  EC_TRACE_AT(4);
  cluster.sync();

  // remap of the firsts, in flight during the look-back (RSRC: loaded in G)
  if constexpr (!RSRC) {
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) rm[j] = ((first >> j) & 1) ? set_remap(tb, id[j]) : 0;
  }

  // ---- B: unique base of the table and of every CTA of it
  if (threadIdx.x < 32) {
    // CTA totals over DSMEM, one lane each
    const int v = lane_id() < kClusterCtas ? *cluster.map_shared_rank(&s_total, lane_id()) : 0;
    int incl = v;
#pragma unroll
    for (int o = 1; o < kClusterCtas; o <<= 1) {
      const int y = __shfl_up_sync(kFull, incl, o);
      if (lane_id() >= o) incl += y;
    }
    if (lane_id() < kClusterCtas) s_pref[lane_id()] = incl - v;
    const int all = __shfl_sync(kFull, incl, kClusterCtas - 1);
    // look-back over the lower tables, 32 at a time: a word is usable once all
    // 8 CTAs of its table added their counts; an inclusive word ends the walk
    int excl = 0;
    for (int k0 = t - 1; k0 >= 0; k0 -= 32) {
      const int k = k0 - lane_id();
      unsigned long long w = kTabInc;  // before table 0: an inclusive zero
      if (k >= 0) {
        do {
          w = *reinterpret_cast<volatile unsigned long long*>(tstatus + k);
        } while (!(w & kTabInc) && ((w >> 32) & 0xFF) < kClusterCtas);
      }
      const unsigned inc = __ballot_sync(kFull, (w & kTabInc) != 0);
      const int stop = inc ? __ffs(inc) - 1 : 32;  // nearest inclusive predecessor
      excl += __reduce_add_sync(kFull, lane_id() <= stop ? static_cast<int>(static_cast<uint32_t>(w)) : 0);
      if (inc) break;
    }
    if (lane_id() == 0) {
      if (crank == 0) {
        publish(tstatus + t, kTabInc | (static_cast<unsigned long long>(kClusterCtas) << 32) |
                                 static_cast<uint32_t>(excl + all));
        c.ubase[t] = excl;
        if (t == T - 1) c.ubase[T] = excl + all;
      }
      s_base = excl;
    }
  }
  __syncthreads();
  EC_TRACE_AT(5);

  // ---- E: unique index of every representative (pf[j] becomes it)
  const int tbase = s_base;
  const int base = tbase + s_pref[crank] + ex;
  {
    uint32_t xw[ITEMS];
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {  // remote thread words, all in flight
      xw[j] = 0;
      if (((rep & ~first) >> j) & 1) {
        const int64_t q = pf[j];
        const int cf = static_cast<int>(q / chunk);
        const int64_t q0 = static_cast<int64_t>(cf) * chunk, q1 = min(n, q0 + chunk);
        const int itf = static_cast<int>((q1 - q0 + kClusterThreads - 1) / kClusterThreads);
        const int thf = static_cast<int>((q - q0) / itf);
        xw[j] = *cluster.map_shared_rank(sxm + thf, cf);
        pf[j] = (static_cast<uint32_t>(cf) << 8) | static_cast<uint32_t>(q - q0 - static_cast<int64_t>(thf) * itf);
      }
    }
    int r = 0;
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      if ((first >> j) & 1) {
        pf[j] = static_cast<uint32_t>(base + r++);
      } else if ((rep >> j) & 1) {
        const uint32_t cf = pf[j] >> 8, jf = pf[j] & 0xFF;
        pf[j] = static_cast<uint32_t>(tbase + s_pref[cf]) + (xw[j] >> 16) + __popc(xw[j] & 0xFFFFu & ((1u << jf) - 1));
      }
      // for this CTA's hot duplicates: table-local unique index (< 65536) in
      // the high half; the low half counts the CTA's lookups of the id (phase I)
      if (((rep >> j) & 1) && id[j] < nloc) sval[id[j]] = (pf[j] - static_cast<uint32_t>(tbase)) << 16;
    }
  }
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");  // remote reads done
  {
    uint32_t missm = 0;
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      if (!((first >> j) & 1)) continue;
      const uint32_t g = pf[j];
      uniq[g] = id[j];
      uslot[g] = id[j];
      utab[g] = static_cast<uint16_t>(t);
      usrc[g] = rm[j];  // cache row, or -1: a miss iff the id is not cached (core/src/simulator.cpp:99)
      if (rm[j] < 0) missm |= 1u << j;
      // the set is left holding only what a later kernel reads: with `tag`
      // (pinned-host tier) each miss's unique index for k_patch_prefetch; every
      // other slot goes back to empty here (every read of it was before the
      // second cluster barrier), so the pool's reset tail touches misses only
      *set_word(tb, id[j]) = tag && rm[j] < 0 ? (static_cast<unsigned long long>(id[j]) << 32) | kRankTag | g : kEmptySlot;
    }
    // miss queue: one atomic per CTA (the queue counter is shared by every
    // CTA of every table; per-warp atomics queued ~3.3K same-address returns)
    const int nm = __popc(missm);
    int mtot;
    const int mex = block_exclusive_scan<kClusterThreads>(nm, sw, &mtot);
    if (threadIdx.x == 0) {
      s_qbase = mtot ? atomicAdd(c.miss_total, mtot) : 0;
      if (mtot) atomicAdd(c.M + t, mtot);
    }
    __syncthreads();
    int qbase = s_qbase + mex;
#pragma unroll
    for (int j = 0; j < ITEMS; ++j)
      if ((missm >> j) & 1) missq[qbase++] = pf[j];
  }
  EC_TRACE_AT(6);

  // ---- I: inverse, and each unique's lookup count (the backward's fp32 /
  // fp64 split, k_scatter): hot ids counted per CTA in shared memory, then one
  // RED per (CTA, hot id); other ids one RED per distinct unique per warp item
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const bool hot = id[j] < nloc;
    const uint32_t g = id[j] == kEmptyKey ? kInvalidSlot
                       : ((rep >> j) & 1) ? pf[j]
                       : hot ? static_cast<uint32_t>(tbase) + (sval[id[j]] >> 16) : kInvalidSlot;
    if (j < my) inv[tb.base + p0 + j] = g;
    if (RSRC && j < my) {
      isrc[tb.base + p0 + j] = row_source(g, rm[j]);
    }
    const unsigned peers = __match_any_sync(kFull, g);
    if (g != kInvalidSlot && __ffs(peers) - 1 == lane_id()) {
      if (hot) atomicAdd(sval + id[j], __popc(peers));
      else atomicAdd(ucount + g, __popc(peers));
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < ITEMS; ++j)
    if (((rep >> j) & 1) && id[j] < nloc) atomicAdd(ucount + pf[j], static_cast<int>(sval[id[j]] & 0xFFFFu));
  EC_TRACE_AT(7);
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");  // keep this CTA's smem alive for remote readers
}

}  // namespace ec

// ===================================================================
// K1 + K2 with ONE CTA per table, for small per-table batches (<= 16K
// lookups: the Kaggle configs).  Same algorithm and output as the cluster
// kernel, but every phase boundary is a __syncthreads -- all inserts into a
// table's direct-mapped L2 set come from this CTA, so a CTA barrier orders
// them -- and the kernel occupies T SMs instead of 8*T/2, leaving the rest of
// the GPU to the pool/scatter/host kernels it overlaps in the pipelined step.
//
// Thread t owns positions [t*I, (t+1)*I) (I = ceil(n / threads) <= 32);
// ids are staged in shared memory item-major (conflict-free) and processed
// 8 per round.  Hot ids (< kTableLocal) are deduplicated in a direct-mapped
// shared table (first position by atomicMin, later the unique index); colder
// ids by one 64-bit atomicMin on their L2 slot.
// ===================================================================
namespace ec {

constexpr int kTableThreads = 512;
constexpr int kTableMaxItems = 32;       // n_t <= 16384
constexpr uint32_t kTableLocal = 16384;  // hot ids in shared memory
constexpr int kTableRound = 8;
__host__ __device__ constexpr size_t table_smem_bytes() {
  return (static_cast<size_t>(kTableThreads) * kTableMaxItems + kTableLocal) * sizeof(uint32_t);
}

__global__ void __launch_bounds__(kTableThreads, 1)
    k_dedup_table(const TableDev* __restrict__ td, int T, const uint32_t* __restrict__ indices,
                  unsigned long long* __restrict__ tstatus, int* __restrict__ ctr, uint32_t* __restrict__ uniq,
                  uint32_t* __restrict__ uslot, uint16_t* __restrict__ utab, uint32_t* __restrict__ inv,
                  int32_t* __restrict__ usrc, uint32_t* __restrict__ missq) {
  extern __shared__ __align__(16) uint32_t smem[];
  uint32_t* s_id = smem;                                       // [I][threads]: ids, item-major
  uint32_t* sval = smem + kTableThreads * kTableMaxItems;      // hot id -> first position, later unique index
  __shared__ int sw[kTableThreads / 32];
  __shared__ int s_base;
  const int t = blockIdx.x;  // blocks dispatch in order: lower tables are running or done
  Counters c = counters(ctr, T);
  const TableDev tb = td[t];
  const int n = static_cast<int>(tb.n);
  const int I = (n + kTableThreads - 1) / kTableThreads;
  const int tid = threadIdx.x;
  const int p0 = tid * I;
  const int my = max(0, min(I, n - p0));
  const uint32_t nloc = tb.rows < kTableLocal ? static_cast<uint32_t>(tb.rows) : kTableLocal;
  // ids -> shared (item-major), all of a thread's loads in flight at once;
  // hot slots cleared meanwhile
  if (my == I && I % 4 == 0 && ((tb.base + p0) & 3) == 0) {
    const uint4* src = reinterpret_cast<const uint4*>(indices + tb.base + p0);
#pragma unroll
    for (int q0 = 0; q0 < kTableMaxItems / 4; q0 += 4) {
      uint4 v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = (q0 + q) * 4 < I ? __ldg(src + q0 + q) : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int j = (q0 + q) * 4;
        if (j < I) {
          s_id[(j + 0) * kTableThreads + tid] = v[q].x;
          s_id[(j + 1) * kTableThreads + tid] = v[q].y;
          s_id[(j + 2) * kTableThreads + tid] = v[q].z;
          s_id[(j + 3) * kTableThreads + tid] = v[q].w;
        }
      }
    }
  } else {
    for (int r0 = 0; r0 < my; r0 += kTableRound) {
      uint32_t v[kTableRound];
#pragma unroll
      for (int k = 0; k < kTableRound; ++k) v[k] = r0 + k < my ? __ldg(indices + tb.base + p0 + r0 + k) : 0u;
#pragma unroll
      for (int k = 0; k < kTableRound; ++k)
        if (r0 + k < my) s_id[(r0 + k) * kTableThreads + tid] = v[k];
    }
  }
  for (uint32_t i = tid; i < nloc; i += kTableThreads) sval[i] = kEmptyKey;
  __syncthreads();

  // ---- inserts: hot ids into shared memory, cold ids into the L2 set
  for (int r0 = 0; r0 < I; r0 += kTableRound) {
#pragma unroll
    for (int k = 0; k < kTableRound; ++k) {
      const int j = r0 + k;
      uint32_t id = j < my ? s_id[j * kTableThreads + tid] : kEmptyKey;
      if (j < my && id >= tb.rows) {
        atomicExch(c.err, 1);
        id = kEmptyKey;
        s_id[j * kTableThreads + tid] = kEmptyKey;
      }
      const uint32_t key = id < nloc ? id : kEmptyKey;
      const unsigned peers = __match_any_sync(kFull, key);
      if (key != kEmptyKey) {
        if (__ffs(peers) - 1 == lane_id()) atomicMin(sval + key, static_cast<uint32_t>(p0 + j));
      } else if (id != kEmptyKey) {
        atomicMin(set_word(tb, id), (static_cast<unsigned long long>(id) << 32) | static_cast<uint32_t>(p0 + j));
      }
    }
  }
  __syncthreads();  // this CTA made every insert of the table

  // ---- first occurrences (per-thread masks, I <= 32), CTA scan
  uint32_t first = 0;
  for (int r0 = 0; r0 < I; r0 += kTableRound) {
    uint32_t w[kTableRound];
#pragma unroll
    for (int k = 0; k < kTableRound; ++k) {
      const int j = r0 + k;
      const uint32_t id = j < my ? s_id[j * kTableThreads + tid] : kEmptyKey;
      w[k] = id == kEmptyKey ? kEmptyKey : id < nloc ? sval[id] : static_cast<uint32_t>(__ldcg(set_word(tb, id)));
    }
#pragma unroll
    for (int k = 0; k < kTableRound; ++k)
      if (w[k] == static_cast<uint32_t>(p0 + r0 + k)) first |= 1u << (r0 + k);
  }
  int total;
  const int ex = block_exclusive_scan<kTableThreads>(__popc(first), sw, &total);

  // ---- table base: publish, warp-parallel look-back over lower tables
  if (tid < 32) {
    if (tid == 0) publish(tstatus + t, (t == 0 ? kStatInc : kStatAgg) | static_cast<uint32_t>(total));
    int excl = 0;
    for (int k0 = t - 1; k0 >= 0; k0 -= 32) {
      const int k = k0 - lane_id();
      unsigned long long v = kStatInc;  // before table 0: an inclusive zero
      if (k >= 0) {
        do {
          v = *reinterpret_cast<volatile unsigned long long*>(tstatus + k);
        } while ((v >> 32) == 0);
      }
      const unsigned inc = __ballot_sync(kFull, (v >> 32) == 2);
      const int stop = inc ? __ffs(inc) - 1 : 32;
      excl += __reduce_add_sync(kFull, lane_id() <= stop ? static_cast<int>(static_cast<uint32_t>(v)) : 0);
      if (inc) break;
    }
    if (tid == 0) {
      if (t > 0) publish(tstatus + t, kStatInc | static_cast<uint32_t>(excl + total));
      c.ubase[t] = excl;
      if (t == T - 1) c.ubase[T] = excl + total;
      s_base = excl;
    }
  }
  __syncthreads();

  // ---- emit the firsts (+ K2 partition), unique index into the hot slot / L2 tag
  {
    int g = s_base + ex;
    for (int r0 = 0; r0 < I; r0 += kTableRound) {
      uint32_t id[kTableRound];
      int32_t rm[kTableRound];
#pragma unroll
      for (int k = 0; k < kTableRound; ++k) {
        const int j = r0 + k;
        id[k] = ((first >> j) & 1) ? s_id[j * kTableThreads + tid] : kEmptyKey;
        rm[k] = id[k] != kEmptyKey ? __ldg(tb.remap + id[k]) : 0;
      }
      uint32_t missm = 0;
#pragma unroll
      for (int k = 0; k < kTableRound; ++k) {
        if (id[k] == kEmptyKey) continue;
        uniq[g] = id[k];
        uslot[g] = id[k];
        utab[g] = static_cast<uint16_t>(t);
        usrc[g] = rm[k];  // a miss iff the id is not cached (core/src/simulator.cpp:99)
        if (id[k] < nloc) sval[id[k]] = static_cast<uint32_t>(g);
        *set_word(tb, id[k]) = (static_cast<unsigned long long>(id[k]) << 32) | kRankTag | static_cast<uint32_t>(g);
        if (rm[k] < 0) missm |= 1u << k;
        id[k] = static_cast<uint32_t>(g++);  // now the unique index
      }
      // miss queue: one atomic per warp and round
      const int nm = __popc(missm);
      int incl = nm;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, incl, o);
        if (lane_id() >= o) incl += y;
      }
      const int wtot = __shfl_sync(kFull, incl, 31);
      int qbase = 0;
      if (lane_id() == 31 && wtot) {
        qbase = atomicAdd(c.miss_total, wtot);
        atomicAdd(c.M + t, wtot);
      }
      qbase = __shfl_sync(kFull, qbase, 31) + incl - nm;
#pragma unroll
      for (int k = 0; k < kTableRound; ++k)
        if ((missm >> k) & 1) missq[qbase++] = id[k];
    }
  }
  __syncthreads();  // hot slots and L2 tags hold unique indices

  // ---- inverse
  for (int r0 = 0; r0 < I; r0 += kTableRound) {
    uint32_t g[kTableRound];
#pragma unroll
    for (int k = 0; k < kTableRound; ++k) {
      const int j = r0 + k;
      const uint32_t id = j < my ? s_id[j * kTableThreads + tid] : kEmptyKey;
      g[k] = id == kEmptyKey ? kInvalidSlot
             : id < nloc     ? sval[id]
                             : static_cast<uint32_t>(__ldcg(set_word(tb, id))) & ~kRankTag;
    }
#pragma unroll
    for (int k = 0; k < kTableRound; ++k)
      if (r0 + k < my) inv[tb.base + p0 + r0 + k] = g[k];
  }
}

}  // namespace ec

// ===================================================================
// K6a as a transpose: gradients of a unique row are summed in registers.
//
//   k_bwd_count   per lookup: cnt[inverse] += 1 (match-any warp aggregation)
//   k_uscan_*     off = exclusive scan of cnt over the U uniques (device U)
//   k_bwd_fill    per lookup: slot = off[u] + cursor[u]++ ; lists hold (u, grad row)
//   k_bwd_reduce  fixed 32-entry chunks of the u-grouped list per lane group:
//                 runs of one u are summed in registers; runs wholly inside a
//                 chunk are stored, the two boundary runs add atomically
// Hot rows of tiny tables no longer serialise on L2 atomics: every grad row
// is read once and ~2 float4 REDs per chunk remain.
// ===================================================================
namespace ec {



__global__ void __launch_bounds__(kThreads) k_bwd_count(const Tile* __restrict__ tiles, int ntiles,
                                                        const uint32_t* __restrict__ inv, int* __restrict__ cnt) {
  for (int ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
    const Tile tile = tiles[ti];
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
      const uint32_t off = j * kThreads + threadIdx.x;
      const uint32_t u = off < tile.count ? inv[tile.start + off] : kInvalidSlot;
      const unsigned peers = __match_any_sync(kFull, u);
      if (u != kInvalidSlot && (__ffs(peers) - 1) == lane_id()) atomicAdd(cnt + u, __popc(peers));
    }
  }
}

// Exclusive scan of cnt[0, U) with U read on the device; cnt is reset to 0 so
// it can serve as the fill cursor.  part needs ceil(N / kScanTile) + 1 ints.
__global__ void k_uscan_reduce(const int* __restrict__ cnt, const int* __restrict__ ctr, int T, int* __restrict__ part) {
  const int U = counters(const_cast<int*>(ctr), T).ubase[T];
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile;
  int s = 0;
  if (base < U) {
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
      const int64_t i = base + j * kScanThreads + threadIdx.x;
      if (i < U) s += cnt[i];
    }
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

__global__ void k_uscan_apply(int* __restrict__ cnt, const int* __restrict__ ctr, int T, const int* __restrict__ part,
                              int* __restrict__ off) {
  const int U = counters(const_cast<int*>(ctr), T).ubase[T];
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile;
  if (base > U) return;  // whole block past the end (block-uniform)
  __shared__ int sw[kScanThreads / 32];
  int run = part[blockIdx.x];
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    const int64_t i = base + j * kScanThreads + threadIdx.x;
    const int v = i < U ? cnt[i] : 0;
    int tot;
    const int ex = block_exclusive_scan<kScanThreads>(v, sw, &tot);
    if (i < U) {
      off[i] = run + ex;
      cnt[i] = 0;
    } else if (i == U) {
      off[i] = run + ex;  // total
    }
    run += tot;
  }
}

__global__ void __launch_bounds__(kThreads) k_bwd_fill(const Tile* __restrict__ tiles, int ntiles,
                                                       const TableDev* __restrict__ td, const int64_t* __restrict__ bag_off,
                                                       int T, int B, int P, const uint32_t* __restrict__ inv,
                                                       const int* __restrict__ off, int* __restrict__ cursor,
                                                       uint2* __restrict__ list) {
  for (int ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
    const Tile tile = tiles[ti];
    const TableDev tb = td[tile.table];
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
      const uint32_t o = j * kThreads + threadIdx.x;
      const int64_t p = tile.start + o;
      const uint32_t u = o < tile.count ? inv[p] : kInvalidSlot;
      const unsigned peers = __match_any_sync(kFull, u);
      const int leader = __ffs(peers) - 1;
      int b0 = 0;
      if (u != kInvalidSlot && leader == lane_id()) b0 = atomicAdd(cursor + u, __popc(peers));
      b0 = __shfl_sync(kFull, b0, leader);
      if (u != kInvalidSlot) {
        const int pos = off[u] + b0 + __popc(peers & ((1u << lane_id()) - 1));
        // (unique, row of grad viewed as [B*T, D]) in one 8-byte store
        list[pos] = make_uint2(u, static_cast<uint32_t>(bag_of(tb, bag_off, B, P, static_cast<int>(tile.table), p)) * T +
                                      tile.table);
      }
    }
  }
}

// Single rank, HBM rows (`ap.urows` set): a run wholly inside one chunk is the
// row's whole gradient, so the SGD update w - lr * g is written straight to its
// cache / HBM row here (the arithmetic k_apply would do, bit for bit) and
// k_apply only handles rows whose runs cross a chunk edge.
struct DirectApply {
  const float* urows;  // null: store sums in ugrad
  const int32_t* usrc;
  const uint32_t* uniq;
  const uint16_t* utab;
  const TableDev* td;
  float* cache;
  float lr;
};

template <int VEC>
__global__ void __launch_bounds__(kThreads, 4) k_bwd_reduce(const int* __restrict__ off, const int* __restrict__ ctr, int T,
                                                         const uint2* __restrict__ list,
                                                         const float* __restrict__ grad, float* __restrict__ ugrad,
                                                         double* __restrict__ g64, DirectApply ap = {}) {
  constexpr int D = VEC * 4;
  const RowMap<VEC> m;
  const int U = counters(const_cast<int*>(ctr), T).ubase[T];
  const int n = off[U];
  const int groups = (gridDim.x * blockDim.x) / VEC;
  const int gid = (blockIdx.x * blockDim.x + threadIdx.x) / VEC;
  for (int c0 = gid * kRunChunk; c0 < n; c0 += groups * kRunChunk) {
    const int c1 = min(n, c0 + kRunChunk);
    uint32_t cu = list[c0].x;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};  // fp64: a run's sum rounds once
    bool first_run = true;  // the run containing c0 may start before the chunk
    int i = c0;
    // a run wholly inside the chunk is stored; one that crosses a chunk edge
    // adds its part to ugrad (zeroed) -- or, for rows spread over more than
    // kLightAdds chunks, to the row's fp64 sum, which k_g64_finalize rounds
    // into ugrad (at most kLightAdds fp32 roundings per row either way)
    // direct apply: the run's row operands are loaded when the run starts, so
    // they arrive while its gradients are summed (at the run's end they were a
    // dependent usrc -> row chain on every short run: 23% of stall samples).
    // Held to 64 registers (4 CTAs/SM): TB 0.378 -> 0.369 ms, cfg1 0.189 ->
    // 0.181; unbounded (79 registers, 3 CTAs/SM) it was slower than before.
    int32_t p_sr = 0;
    uint32_t p_id = 0;
    uint16_t p_t = 0;
    float4 p_w = make_float4(0.f, 0.f, 0.f, 0.f);
    auto prep = [&](uint32_t u) {
      if (!ap.urows) return;
      p_sr = ap.usrc[u];
      p_id = ap.uniq[u];
      p_t = ap.utab[u];
      p_w = ldg4(ap.urows + static_cast<int64_t>(u) * D + m.c * 4);
    };
    prep(cu);
    auto flush = [&](bool spans) {
      const float4 a = make_float4(static_cast<float>(acc[0]), static_cast<float>(acc[1]),
                                   static_cast<float>(acc[2]), static_cast<float>(acc[3]));
      float* dst = ugrad + static_cast<int64_t>(cu) * D + m.c * 4;
      if (!spans && ap.urows) {
        float* row = p_sr >= 0 ? ap.cache + static_cast<int64_t>(p_sr) * D
                               : ap.td[p_t].store + static_cast<int64_t>(p_id) * D;
        const float4 w = p_w;
        st4(row + m.c * 4, make_float4(w.x - ap.lr * a.x, w.y - ap.lr * a.y, w.z - ap.lr * a.z, w.w - ap.lr * a.w));
      } else if (!spans) st4(dst, a);
      else if (chunk_span(off[cu], off[cu + 1]) > kLightAdds) red_g64<VEC>(g64, cu, m.c, acc[0], acc[1], acc[2], acc[3]);
      else atomicAdd(reinterpret_cast<float4*>(dst), a);
    };
    while (i < c1) {
      // 4 grad rows in flight, then fold them in list order
      uint32_t u4[4], g4[4];
      float4 v4[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint2 e = i + k < c1 ? list[i + k] : make_uint2(kInvalidSlot, 0);
        u4[k] = e.x;
        g4[k] = e.y;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k)
        v4[k] = u4[k] != kInvalidSlot ? ld_stream4(grad + static_cast<int64_t>(g4[k]) * D + m.c * 4)
                                      : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (u4[k] == kInvalidSlot) continue;
        if (u4[k] != cu) {
          // run of cu ends inside this chunk: sole owner unless it began before c0
          flush(first_run && off[cu] < c0);
          first_run = false;
          cu = u4[k];
          prep(cu);
          acc[0] = acc[1] = acc[2] = acc[3] = 0.0;
        }
        acc[0] += v4[k].x;
        acc[1] += v4[k].y;
        acc[2] += v4[k].z;
        acc[3] += v4[k].w;
      }
      i += 4;
    }
    // last run: it may continue past the chunk, or began before it
    flush((first_run && off[cu] < c0) || off[cu + 1] > c1);
  }
}

// Unique-row gradients whose sums went to g64, rounded into ugrad (g64 left
// zeroed): after k_bwd_reduce (off != nullptr) the rows spanning more than
// kLightAdds chunks; after the atomic k_scatter (off == nullptr) the rows
// heavier than kLightAdds lookups (every row without counts).  Leaves ucount
// zeroed.
template <int VEC>
__global__ void __launch_bounds__(kThreads) k_g64_finalize(const int* __restrict__ off, int* __restrict__ ucount,
                                                           const int* __restrict__ ctr, int T, float* __restrict__ ugrad,
                                                           double* __restrict__ g64) {
  constexpr int D = VEC * 4;
  constexpr int RPW = RowMap<VEC>::kRowsPerWarp;
  const RowMap<VEC> m;
  const int U = counters(const_cast<int*>(ctr), T).ubase[T];
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int g = warp * RPW + m.sub; g < U; g += nwarps * RPW) {
    bool heavy;
    if (off) {
      heavy = chunk_span(off[g], off[g + 1]) > kLightAdds;
    } else {
      heavy = !ucount || ucount[g] > kLightAdds;
      if (ucount && m.c == 0) ucount[g] = 0;
    }
    if (!heavy) continue;
    double gs[4];
    take_g64<VEC>(g64, g, m.c, gs);
    float* p = ugrad + static_cast<int64_t>(g) * D + m.c * 4;
    const float4 a = *reinterpret_cast<const float4*>(p);
    st4(p, make_float4(static_cast<float>(a.x + gs[0]), static_cast<float>(a.y + gs[1]),
                       static_cast<float>(a.z + gs[2]), static_cast<float>(a.w + gs[3])));
  }
}

}  // namespace ec

// ===================================================================
// Hot/normal scheduling of a multi-table dataset (
// classify_samples / build_schedule, core/src/trace.cpp:185-240, extended to
// one id per table per sample): a sample is hot iff every id is cached.
// ===================================================================
namespace ec {

__global__ void k_classify_tables(const TableDev* __restrict__ td, int T, const uint32_t* __restrict__ ids, uint64_t q,
                                  int* __restrict__ hot, int* __restrict__ err) {
  for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < q; s += (uint64_t)gridDim.x * blockDim.x) {
    int h = 1;
    for (int t = 0; t < T; ++t) {
      const uint32_t id = ids[s * T + t];
      const TableDev tb = td[t];
      if (id >= tb.rows) {
        atomicExch(err, 1);
        h = 0;
        continue;
      }
      h &= __ldg(tb.remap + id) >= 0;
    }
    hot[s] = h;
  }
}

__global__ void k_stable_order(const int* __restrict__ hot, const int* __restrict__ excl, const int* __restrict__ n_hot,
                               uint64_t q, uint32_t* __restrict__ order) {
  const int H = *n_hot;
  for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < q; s += (uint64_t)gridDim.x * blockDim.x) {
    const int e = excl[s];
    order[hot[s] ? e : H + static_cast<int>(s) - e] = static_cast<uint32_t>(s);
  }
}

// indices[t*count + i] = ids[order[first + i]*T + t]: a batch in the
// table-major layout ec_lookup_fwd takes (pooling 1).
__global__ void k_gather_batch(const uint32_t* __restrict__ ids, const uint32_t* __restrict__ order, uint64_t first,
                               uint32_t count, int T, uint32_t* __restrict__ out) {
  const uint64_t n = static_cast<uint64_t>(count) * T;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t t = i / count, k = i - t * count;
    out[i] = ids[static_cast<uint64_t>(order[first + k]) * T + t];
  }
}

}  // namespace ec

// ===================================================================
// Experimental: pinned-host misses fetched by the TMA bulk-copy engine
// (cp.async.bulk global -> shared, completion counted on an mbarrier) rather
// than by SM loads; rows then go smem -> urows.  One elected thread per CTA
// issues a batch of row copies.
// ===================================================================
namespace ec {

constexpr int kTmaBytes = 16384;  // staged row bytes in flight per CTA

template <int VEC>
__global__ void __launch_bounds__(kThreads) k_gather_host_tma(const TableDev* __restrict__ td, int T,
                                                              const int* __restrict__ ctr,
                                                              const uint32_t* __restrict__ missq,
                                                              const uint32_t* __restrict__ uniq,
                                                              const uint16_t* __restrict__ utab,
                                                              float* __restrict__ urows, int rank, int world) {
  constexpr int D = VEC * 4;
  constexpr uint32_t kRowBytes = D * 4;
  constexpr int kTmaRows = kTmaBytes / (D * 4) < 256 ? kTmaBytes / (D * 4) : 256;
  __shared__ __align__(128) float buf[kTmaRows * D];
  __shared__ __align__(8) unsigned long long bar;
  __shared__ uint32_t dst_g[kTmaRows];
  const int nm = *counters(const_cast<int*>(ctr), T).miss_total;
  const uint32_t bar_addr = static_cast<uint32_t>(__cvta_generic_to_shared(&bar));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(bar_addr));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  uint32_t phase = 0;
  // spread the misses over every CTA (each SM's TMA unit issues its own rows)
  const int chunk = max(1, min(kTmaRows, (nm + static_cast<int>(gridDim.x) - 1) / static_cast<int>(gridDim.x)));
  for (int q0 = blockIdx.x * chunk; q0 < nm; q0 += gridDim.x * chunk) {
    const int cnt = min(chunk, nm - q0);
    // every thread issues the bulk copies of its rows; thread 0 arms the barrier
    // with the batch's byte count (tx may complete before the expect: the phase
    // still needs thread 0's arrival)
    int mine = 0;
    for (int r = threadIdx.x; r < cnt; r += blockDim.x) {
      const uint32_t g = missq[q0 + r];
      const uint32_t id = uniq[g];
      const bool own = static_cast<int>(id % world) == rank;
      dst_g[r] = own ? g : 0xFFFFFFFFu;
      if (!own) continue;
      ++mine;
      const float* src = td[utab[g]].store + static_cast<int64_t>(id / world) * D;
      const uint32_t dsts = static_cast<uint32_t>(__cvta_generic_to_shared(buf + r * D));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dsts),
                   "l"(src), "r"(kRowBytes), "r"(bar_addr)
                   : "memory");
    }
    const int rows = __syncthreads_count(mine);  // mine <= 1 when cnt <= blockDim
    if (threadIdx.x == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(bar_addr), "r"(rows * kRowBytes) : "memory");
    // wait for the bytes of this batch
    asm volatile(
        "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(bar_addr),
        "r"(phase)
        : "memory");
    phase ^= 1;
    for (int i = threadIdx.x; i < cnt * VEC; i += blockDim.x) {
      const int r = i / VEC, c = i - r * VEC;
      const uint32_t g = dst_g[r];
      if (g != 0xFFFFFFFFu)
        st4(urows + static_cast<int64_t>(g) * D + c * 4, *reinterpret_cast<const float4*>(buf + r * D + c * 4));
    }
    __syncthreads();
  }
}

}  // namespace ec

namespace ec {

// Host write-back through the TMA engine: new rows are built in shared memory
// and bulk-stored to the pinned host shard (cp.async.bulk global <- shared).
// With a pending prefetched batch (nxt_td != null; launched after its host
// gather) the same new rows also refresh that batch's gathered copies — the
// k_patch_prefetch work, without a separate launch on the critical path.
template <int VEC>
__global__ void __launch_bounds__(kThreads) k_apply_host_tma(const TableDev* __restrict__ td, int T,
                                                             const int* __restrict__ ctr,
                                                             const uint32_t* __restrict__ missq,
                                                             const uint32_t* __restrict__ uniq,
                                                             const uint16_t* __restrict__ utab,
                                                             const float* __restrict__ urows,
                                                             const float* __restrict__ ugrad, float lr, int rank,
                                                             int world, const TableDev* __restrict__ nxt_td = nullptr,
                                                             const int32_t* __restrict__ nxt_usrc = nullptr,
                                                             float* __restrict__ nxt_urows = nullptr,
                                                             const double* __restrict__ g64 = nullptr,
                                                             const int* __restrict__ ucount = nullptr) {
  constexpr int D = VEC * 4;
  constexpr uint32_t kRowBytes = D * 4;
  constexpr int kTmaRows = kTmaBytes / (D * 4) < 256 ? kTmaBytes / (D * 4) : 256;
  __shared__ __align__(128) float buf[kTmaRows * D];
  __shared__ uint32_t dst_g[kTmaRows], pat_g[kTmaRows];
  const int nm = *counters(const_cast<int*>(ctr), T).miss_total;
  // spread the misses over every CTA (each SM's TMA unit issues its own rows)
  const int chunk = max(1, min(kTmaRows, (nm + static_cast<int>(gridDim.x) - 1) / static_cast<int>(gridDim.x)));
  for (int q0 = blockIdx.x * chunk; q0 < nm; q0 += gridDim.x * chunk) {
    const int cnt = min(chunk, nm - q0);
    if (threadIdx.x < cnt) {
      const uint32_t g = missq[q0 + threadIdx.x];
      const uint32_t id = uniq[g];
      const bool own = static_cast<int>(id % world) == rank;
      dst_g[threadIdx.x] = own ? g : 0xFFFFFFFFu;
      uint32_t g2 = 0xFFFFFFFFu;
      if (own && nxt_td) {  // the id's entry in the pending batch's set: its (tagged) unique index
        const TableDev tb = nxt_td[utab[g]];
        uint32_t h = table_slot(tb, id);
        for (;;) {
          const unsigned long long v = __ldcg(set_word(tb, h));
          if (v == kEmptySlot) break;
          if (static_cast<uint32_t>(v >> 32) == id) {
            const uint32_t u2 = static_cast<uint32_t>(v) & ~kRankTag;
            if (nxt_usrc[u2] < 0) g2 = u2;  // gathered from the host tier: stale copy
            break;
          }
          h = (h + 1) & tb.mask;
        }
      }
      pat_g[threadIdx.x] = g2;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < cnt * VEC; i += blockDim.x) {
      const int r = i / VEC, c = i - r * VEC;
      const uint32_t g = dst_g[r];
      if (g == 0xFFFFFFFFu) continue;
      const float4 w = ldg4(urows + static_cast<int64_t>(g) * D + c * 4);
      const float4 nw = miss_sgd<VEC>(w, ugrad, g64, ucount, g, c, lr);
      *reinterpret_cast<float4*>(buf + r * D + c * 4) = nw;
      if (pat_g[r] != 0xFFFFFFFFu) st4(nxt_urows + static_cast<int64_t>(pat_g[r]) * D + c * 4, nw);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // smem writes -> async (TMA) proxy
    __syncthreads();
    for (int r = threadIdx.x; r < cnt; r += blockDim.x) {
      const uint32_t g = dst_g[r];
      if (g == 0xFFFFFFFFu) continue;
      float* dst = td[utab[g]].store + static_cast<int64_t>(uniq[g] / world) * D;
      const uint32_t srcs = static_cast<uint32_t>(__cvta_generic_to_shared(buf + r * D));
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(srcs), "r"(kRowBytes)
                   : "memory");
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // smem reusable
    __syncthreads();
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // writes done before exit
}

}  // namespace ec
