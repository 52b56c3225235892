// Lookup-engine state shared by engine.cu and exchange.cu.
#pragma once

#include <cstdint>
#include <array>
#include <map>
#include <tuple>
#include <vector>

#include "common.hpp"

namespace ec {

// Per-table constants + per-batch geometry, read by every engine kernel.
struct TableDev {
  unsigned long long* hash;  // open-addressing set for this table's batch
  uint32_t shift, mask;      // hash_slot shift, capacity - 1
  const int32_t* remap;      // id -> global cache row, -1 = not cached
  float* store;              // local shard (device pointer; mapped if pinned host)
  uint64_t rows;             // E_t
  int64_t base;              // first lookup of this table in the batch
  int64_t n;                 // lookups of this table in the batch
  uint32_t direct;           // 1: `hash` is direct-mapped (slot = id, rows slots), no probing
  uint32_t pad_;
  uint32_t* idcnt;           // per slot of `hash`: lookups of that id in the batch (tile path, grouped lists)
};

struct Tile {
  uint32_t table;
  uint32_t count;
  int64_t start;
  uint32_t ub_lo, ub_hi;  // tables whose first tile this is (k_compact writes their ubase)
};

// Per-batch device counters, one int array:
//   M[T] ubase[T+1] miss_total tile_counter wire hot_out hot_in err   (err last: survives resets)
// wire: rows pulled from peer shards by the P2P exchange; hot_out / hot_in:
// hot-row gradients sent to other owners / updated hot rows copied from them.
struct Counters {
  int *M, *ubase, *miss_total, *tile_counter, *wire, *hot_out, *hot_in, *err;
};
__host__ __device__ inline Counters counters(int* p, int T) {
  return Counters{p, p + T, p + 2 * T + 1, p + 2 * T + 2, p + 2 * T + 3, p + 2 * T + 4, p + 2 * T + 5, p + 2 * T + 6};
}
inline size_t counters_size(int T) { return 2 * static_cast<size_t>(T) + 7; }

// What a rank sees of a peer for the peer-memory exchange (K4 over NVLink
// loads/stores/atomics): the peer's HBM shard and its published hot-row
// gradient list, and the flag words the peer waits on.
constexpr int kP2PBarriers = 2;  // device barriers per step of the peer-memory exchange

struct PeerView {
  float* store;             // the peer's whole shard (row = shard_off[peer][t] + id / world)
  // hot rows (replicated cache) owned by the peer (cache slot % world == peer):
  const uint32_t* upd_slot; // slots it updated this step ...
  const float* upd_rows;    // ... their new values ...
  const int* upd_cnt;       // ... and how many
  uint32_t* hin_slot;       // its inbox of hit gradients for its slots, one segment per source rank:
  float* hin_grad;          //   [world][cap] slots / gradient rows
  int* hin_cnt;             //   [world] counts
  unsigned* flags;          // the peer's barrier words: [kP2PBarriers * world]
  // pinned-host shards: the owner's inbox of miss-row gradients, one segment
  // per source rank ([world][cap] row indices / gradient rows, [world] counts)
  uint32_t* inbox_idx;
  float* inbox_grad;
  int* inbox_cnt;
  uint32_t* ver;  // pinned-host shards: step generation of each row's last update (prefetch patch)
};

struct Exchange;  // exchange.cu

template <class T>
struct View {
  T* p = nullptr;
  size_t n = 0;
  size_t bytes() const { return n * sizeof(T); }
};
template <class T>
View<T> view(DevBuf<T>& b) {
  return View<T>{b.p, b.n};
}

struct BatchBufs {
  DevBuf<uint32_t> slot_of, inv, uniq, uslot, missq;
  DevBuf<int32_t> usrc;
  DevBuf<uint16_t> utab;
  DevBuf<float> urows, ugrad;
  DevBuf<int> ucount;  // lookups per unique (cluster dedup; k_scatter's fp32 / fp64 split); zeroed by the backward
  DevBuf<double> g64;  // fp64 gradient sums of unique rows (fused SGD; rows spanning transpose chunks); self-cleaning
  DevBuf<unsigned long long> status, tstat;  // tile / table look-back words
  DevBuf<int> ctr;
  DevBuf<int> cnt, off, part;          // backward transpose: occurrences per unique, offsets, scan partials
  DevBuf<uint2> list;                  // lookups grouped by unique: (unique, grad row)
  const uint32_t* indices = nullptr;  // batch held by a pending prefetch
  uint64_t geom_version = 0;
  bool pending = false;               // prefetched, not yet consumed by forward
  bool gathered = false;              // its pinned-host miss gather was launched (ev_pf)
  bool rows_early = false;            // (peer exchange) host rows read before the step barrier: patch them
  uint64_t seq = 0;                   // prefetch order (the smallest pending seq is consumed next)
  cudaEvent_t ev_free = nullptr;      // main-stream work of its last batch done (set reusable)
  cudaEvent_t ev_ded = nullptr;       // its prefetch's dedup done
  cudaEvent_t ev_pf = nullptr;        // its prefetch complete (dedup + host gather)
  bool lists = false;                 // its forward built the unique-grouped gradient lists
  bool counted = false;               // its dedup wrote ucount (cluster kernel)
  bool row_sources = false;           // its dedup wrote per-lookup row sources into slot_of (cluster kernel, fused path)
  bool left_counts = false;           // a batch in this set left per-unique counts / sums to clear
  uint64_t bytes() const {
    return slot_of.bytes() + inv.bytes() + uniq.bytes() + uslot.bytes() + missq.bytes() + usrc.bytes() +
           utab.bytes() + urows.bytes() + ugrad.bytes() + g64.bytes() + ucount.bytes() + status.bytes() + tstat.bytes() + ctr.bytes() +
           cnt.bytes() + off.bytes() + part.bytes() + list.bytes();
  }
};

// One timing slot per kernel of the batch pipeline (ec_tables_profile_read order).
enum { kPhaseInsert = 0, kPhaseCompact, kPhaseInversePartition, kPhaseGather, kPhaseGatherHost, kPhaseExchange,
       kPhasePool, kPhaseScatter, kPhaseApply, kPhaseApplyHost, kPhaseDedupCluster, kPhaseClearSums, kNumPhases };

// Optional per-phase CUDA-event timing on the launching streams.
struct Profiler {
  struct Rec {
    int phase;
    cudaEvent_t a, b;
  };
  bool on = false;
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> free_;
  double ms_[kNumPhases] = {};
  uint64_t calls_[kNumPhases] = {};
  // (phase, start ms, end ms) relative to the first event since the last read
  static constexpr size_t kTimelineCap = 1 << 16;
  std::vector<std::array<double, 3>> timeline;
  cudaEvent_t t0 = nullptr;
  cudaEvent_t take();
  void collect();
  ~Profiler();
};

// NVTX range over the host-side enqueue of one phase / one API call (header-
// only NVTX v3: a no-op unless a tool such as Nsight or ncu --nvtx attaches).
struct NvtxRange {
  explicit NvtxRange(const char* name);
  ~NvtxRange();
};
const char* phase_name(int phase);

struct PhaseScope {
  PhaseScope(Profiler& p, int phase, cudaStream_t st);
  ~PhaseScope();
  NvtxRange nvtx_;
  Profiler& p_;
  int phase_;
  cudaStream_t st_;
  cudaEvent_t a_ = nullptr;
};

struct GraphKey {
  int kind;  // 0 forward, 1 backward, 2 forward of a prefetched batch, 3 backward patching a prefetch, 4 prefetch
  const void* a;
  const void* b;
  const void* c;
  uint32_t lr_bits;
  int set = 0;  // per-batch buffer set the captured kernels point at
  bool operator<(const GraphKey& o) const {
    return std::tie(kind, a, b, c, lr_bits, set) < std::tie(o.kind, o.a, o.b, o.c, o.lr_bits, o.set);
  }
};

struct GraphEntry {
  cudaGraphExec_t exec;
  uint64_t kernels;
};

struct Engine {
  int device = 0;
  uint32_t T = 0, D = 0;
  int storage = EC_STORAGE_HBM;
  int rank = 0, world = 1;
  uint64_t max_n = 0;
  uint32_t max_b = 0;
  std::vector<uint64_t> rows, local_rows, store_off, remap_off, hash_off;
  std::vector<uint32_t> hash_lg;
  std::vector<uint32_t> hash_direct;  // per table: direct-mapped dedup set
  // direct-map a table's dedup set (8 B per row and buffer set) up to this many
  // rows, within a total budget; the cluster dedup kernel needs it
  static constexpr uint64_t kDirectRows = 1ull << 27;
  static constexpr uint64_t kDirectBudget = 16ull << 30;
  static constexpr uint64_t kAutoClusterN = 32768;  // auto cluster dedup up to this many lookups per table

  DevBuf<float> store_dev;
  float* store_host = nullptr;  // pinned, mapped
  uint64_t store_host_bytes = 0;
  bool store_host_mmapped = false;
  int store_host_fd = -1;  // memfd of a shared host shard (world > 1)
  float* store_base = nullptr;  // device-visible base of the shard
  DevBuf<int32_t> remap;
  DevBuf<unsigned long long> hash;
  DevBuf<uint32_t> idcnt;  // parallel to hash: per-id lookup counts (self-cleaning with the slots)
  DevBuf<float> cache;
  DevBuf<uint32_t> cache_ids;
  DevBuf<uint16_t> cache_tab;
  uint64_t cache_k_total = 0;
  std::vector<uint64_t> cache_k;
  uint64_t synth_seed = 0;
  float synth_scale = 0.f;
  bool synth_valid = false;
  bool rows_trained = false;  // a backward or row write ran since the last synthetic init

  // Per-batch state in a ring of kSets buffer sets, so up to kSets-1 next
  // batches can be prefetched (dedup, hit/miss, host-miss gather) while the
  // current one runs.  The View members below point at the selected set.
  static constexpr int kSets = 3;
  BatchBufs bb[kSets];
  int cur = 0;
  uint64_t pf_seq = 0;
  int head_pending() const;  // the pending set the next forward consumes, or -1
  int free_set() const;      // a set neither current nor pending, or -1
  void launch_pending_gather(int s);
  View<uint32_t> slot_of, inv, uniq, uslot, missq;
  View<int32_t> usrc;
  View<uint16_t> utab;
  View<float> urows, ugrad;
  View<double> g64;
  View<int> ucount;
  View<unsigned long long> status;  // decoupled look-back words, one per tile
  View<unsigned long long> tstat;   // one per table (cluster dedup)
  bool cluster_fits = false;        // every table's batch fits one cluster
  bool cluster_ok = false;          // ... and the cluster path is the faster one
  int cluster_items = 1;            // positions per thread of the cluster kernel
  int dedup_mode = 0;               // 0 auto, 1 tile path, 2 cluster path, 3 CTA-per-table path (when they fit)
  bool table_fits = false;          // every table's batch fits one CTA (k_dedup_table)
  View<int> ctr, cnt, off, part;
  int* ctr_host = nullptr;  // pinned staging for ec_lookup_stats
  // ec_lookup_stats_enqueue ring: pinned counter copies + their completion events
  int* ring_host = nullptr;
  cudaEvent_t ring_ev[EC_STATS_SLOTS] = {};
  uint64_t ring_lookups[EC_STATS_SLOTS] = {}, ring_wire_rows[EC_STATS_SLOTS] = {}, ring_wire_bytes[EC_STATS_SLOTS] = {};
  bool ring_full[EC_STATS_SLOTS] = {};
  View<uint2> list;
  int scatter_mode = 0;  // 0 auto (fused when possible), 1 float4 atomics, 2 transpose + segmented reduction
  // dedup by one thread-block cluster per table (K1+K2 in one kernel)
  bool use_table_kernel() const { return table_fits && dedup_mode == 3; }
  // backward reduction by transposition (lookups grouped by unique): auto at
  // >= 32K lookups per table (measured in bwd_scatter)
  bool transpose_regime() const { return scatter_mode == 2 || (scatter_mode == 0 && max_n_batch >= 32768); }
  // the tile dedup path builds the grouped lists in the forward (counts in
  // k_insert, offsets by scan, fill in k_inverse_partition)
  bool lists_in_forward() const { return !use_cluster() && transpose_regime(); }
  bool use_cluster() const {
    return use_table_kernel() || (cluster_ok && dedup_mode == 0) || (cluster_fits && dedup_mode == 2);
  }
  // single rank, atomic-scatter regime (<= 32K lookups per table, e.g. the
  // Kaggle configs): the forward pools straight from the source rows (no K3
  // gather of cached/HBM rows) and the backward scatters -lr * grad straight
  // into them (no ugrad round trip, no K6b launch).  Measured: Kaggle HBM tier
  // 76 -> 64 us per step; but TB (26 x 65K, D=64) 0.42 -> 0.44 ms and cfg1
  // (P=20) 0.23 -> 0.24 ms, where pooling from the compact L2-resident copy of
  // the unique rows beats re-reading every lookup's row at its source.
  bool fused() const { return world == 1 && !in_group && scatter_mode == 0 && max_n_batch < 32768; }
  int64_t max_n_batch = 0;  // largest per-table lookup count of the current geometry
  void select(int i);
  DevBuf<Tile> tiles;
  DevBuf<int4> stiles;                // scatter tiles (table, bag lo, bag hi, -)
  DevBuf<TableDev> tdev_buf;  // kSets copies of the table descriptors, one per batch-buffer set (own hash each)
  View<TableDev> tdev;        // the selected set's copy
  std::vector<TableDev> td_host;
  int ntiles = 0, nstiles = 0, tail_lo = 0;

  // geometry of the last batch
  bool have_geom = false, geom_fixed = true, have_fwd = false;
  std::vector<int64_t> geom_off;
  uint32_t geom_b = 0, geom_p = 0;
  const int64_t* bag_off = nullptr;
  float* out_ptr = nullptr;

  cudaStream_t side = nullptr, side2 = nullptr, pstream = nullptr;
  cudaEvent_t ev_pfcall = nullptr;   // caller's stream at the prefetch call
  cudaEvent_t ev_gate = nullptr;     // caller's stream at the forward that starts a pending gather
  cudaEvent_t ev_b1 = nullptr;       // (peer exchange) the last forward passed its step barrier

  cudaEvent_t ev_part = nullptr, ev_side = nullptr, ev_side2 = nullptr,
              ev_grad = nullptr, ev_patch = nullptr;
  uint64_t geom_version = 0;
  bool consuming_prefetch = false;
  void prefetch(const ec_batch& b, cudaStream_t st);
  void drop_prefetch(cudaStream_t st);
  template <int VEC> void launch_gather_host(cudaStream_t s);

  Profiler prof;
  uint64_t launches = 0;
  void launched() {
    EC_LAUNCH();
    ++launches;
  }

  bool use_graphs = true;
  std::map<GraphKey, GraphEntry> graphs;
  template <class F> void run_maybe_graphed(const GraphKey& key, cudaStream_t st, F&& enqueue);
  void clear_graphs();
  void enqueue_forward(const uint32_t* indices, cudaStream_t st);

  Exchange* ex = nullptr;
  uint64_t last_wire_rows = 0, last_wire_bytes = 0;

  ~Engine();
  void create(const ec_tables_config& c);
  uint64_t device_bytes() const;
  int host_grid() const;
  static bool host_tma();
  void upload_tdev();
  void plan_sets(bool direct_big);
  void alloc_sets();
  void sync_set_remap();
  void set_views();
  void require_direct_sets();
  int host_write_grid() const;
  int row_grid() const;
  void init_synthetic(uint64_t seed, float scale, cudaStream_t st);
  void fill_cache(cudaStream_t st, bool from_store);
  void place_cache(const uint32_t* const* ids, const uint64_t* k);
  void rw_rows(uint32_t t, const uint32_t* ids, uint64_t n, float* buf, bool write);
  void set_geometry(const ec_batch& b, cudaStream_t st);
  void forward(const ec_batch& b, float* out, cudaStream_t st);
  void backward(const float* grad, float lr, cudaStream_t st);
  void read_counters(cudaStream_t st, std::vector<int>& h);
  template <int VEC> void fwd_gather_local(cudaStream_t st);
  template <int VEC> void fwd_pool(cudaStream_t st);
  template <int VEC> void bwd_scatter(const float* grad, cudaStream_t st);
  template <int VEC> void finalize_transpose(cudaStream_t st);
  bool fold_g64 = false;  // k_apply reads the fp64 sums of chunk-spanning rows itself
  bool direct_apply = false;  // k_bwd_reduce applied the rows whose runs fit one chunk
  template <int VEC> void bwd_apply_local(float lr, cudaStream_t st);
  template <int VEC> void enqueue_host_writeback(float lr);
  template <int VEC> void clear_sums(cudaStream_t st);
  void join_host_writes(cudaStream_t st);
  void enqueue_dedup_partition(const uint32_t* indices, cudaStream_t st);
  void gather_for_export();
  void scatter_grads(const float* grad, cudaStream_t st);
  template <int VEC>
  void export_gather();
  float bwd_lr = 0.f;  // learning rate of the backward being enqueued
  template <int ITEMS>
  void launch_dedup_cluster(const uint32_t* indices, cudaStream_t st);
  template <int ITEMS, bool RSRC>
  void launch_dedup_cluster_k(const uint32_t* indices, cudaStream_t st);
  void forward_prologue(const ec_batch& b, float* out, cudaStream_t st);
  void gather_local(cudaStream_t st);
  void pool(cudaStream_t st);
  void scatter_and_apply_local(const float* grad, float lr, cudaStream_t st);

  // multi-GPU (exchange.cu)
  bool in_group = false;  // member of an in-process loopback group
  void ex_init(int W);
  void ex_route(cudaStream_t st);
  void ex_plan();
  void ex_serve(cudaStream_t st);
  void ex_unpack(cudaStream_t st);
  void ex_pack_bwd(cudaStream_t st);
  void ex_apply_bwd(float lr, cudaStream_t st);
  bool comm_ready() const;
  void attach_comm(const uint8_t* id128);
  void destroy_comm();
  uint64_t exch_bytes() const;
  uint64_t geometry_digest() const;  // what every rank of a job must agree on (peer memory is indexed by it)
  void exchange_fwd(cudaStream_t st);
  void exchange_bwd(float lr, cudaStream_t st);
  // peer-memory exchange (exchange.cu)
  bool p2p_on() const;
  const PeerView* p2p_peers() const;
  const int64_t* p2p_shard_off() const;
  void p2p_alloc();
  void p2p_set_peers(const std::vector<PeerView>& v);
  PeerView p2p_self() const;
  void p2p_fwd_begin(cudaStream_t st);
  void p2p_close_open(cudaStream_t st);
  bool p2p_step_open() const;
  void p2p_patch_prefetched(cudaStream_t st);
  template <int VEC> void p2p_patch(cudaStream_t st);
  void p2p_bwd_publish(float lr, cudaStream_t st);
  template <int VEC> void p2p_publish(float lr, cudaStream_t st, int part, int wait_b, int sig_b);
  void p2p_signal(int b, cudaStream_t st);
  void p2p_wait(int b, unsigned epoch, cudaStream_t st);
  void p2p_bwd_finish(float lr, cudaStream_t st);
  void p2p_bwd_owner(float lr, cudaStream_t st);   // (finish, part 1) owners apply misses and their hot rows
  void p2p_bwd_replica(cudaStream_t st);           // (finish, part 2) every replica copies the owners' hot rows
  template <int VEC> void p2p_hot(float lr, cudaStream_t st);
  template <int VEC> void p2p_hot_copy(cudaStream_t st);
  void p2p_hot_alloc();  // owner accumulators, sized by the cache
};

// Instantiate FN<VEC> for the row width (D/4 float4 lanes per row).
#define EC_DISPATCH_VEC(FN, ...)                                                  \
  switch (D / 4) {                                                                \
    case 1: FN<1>(__VA_ARGS__); break;                                            \
    case 2: FN<2>(__VA_ARGS__); break;                                            \
    case 4: FN<4>(__VA_ARGS__); break;                                            \
    case 8: FN<8>(__VA_ARGS__); break;                                            \
    case 16: FN<16>(__VA_ARGS__); break;                                          \
    case 32: FN<32>(__VA_ARGS__); break;                                          \
    default: invalid("dim must be 4, 8, 16, 32, 64 or 128 for the lookup kernels"); \
  }

}  // namespace ec

// Opaque ABI handle (include/embcomm_gpu.h).
struct ec_tables_s {
  ec::Engine e;
};
