/*
 * embcomm_gpu.h — C-ABI of libembcomm_gpu.so, the B200-native (sm_100a)
 * implementation of the embedding-lookup hot path of arXiv 2411.01611 behind
 * the reference library's core/ API surface (/root/reference/proj/core).
 *
 * The reference is a C++20 static library with no FFI.  Each
 * entry point below names the reference interface it replaces
 * (file:line into /root/reference/proj).  Reference spans become
 * (pointer, length); value results become caller-owned POD structs; C++
 * exceptions become status codes.  No torch or C++ types cross this ABI.
 *
 * Conventions
 *   - Every function returns an ec_status.  EC_EINVAL (=2) is the reference's
 *     ValidationError, EC_EINVARIANT (=3) its InvariantError
 *     (core/include/embcomm/error.hpp:10-19; CLI exit codes
 *     tools/src/main.cpp:220-229).  ec_last_error() returns the thread-local
 *     message of the last failure (messages name the offending id/size as the
 *     reference's do, e.g. core/src/distribution.cpp:22-24).
 *   - `stream` arguments are cudaStream_t passed as void* (NULL = legacy
 *     default stream).  Device pointers are marked _dev, host pointers _host.
 *   - Handles are not thread-safe; use one handle per host thread / GPU.
 *   - There is no CPU fallback: GPU entry points fail with EC_ECUDA when no
 *     device is present.
 */
#ifndef EMBCOMM_GPU_H_
#define EMBCOMM_GPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  EC_OK = 0,
  EC_EINVAL = 2,      /* embcomm::ValidationError  (error.hpp:10-13) */
  EC_EINVARIANT = 3,  /* embcomm::InvariantError   (error.hpp:16-19) */
  EC_ECUDA = 4,       /* CUDA runtime / launch failure, or no GPU */
  EC_ENCCL = 5,       /* NCCL failure */
  EC_ENOMEM = 6       /* device / pinned-host allocation failure */
} ec_status;

const char* ec_last_error(void);
const char* ec_version(void);
/* kCostUnitsNote, core/include/embcomm/cost_model.hpp:13-14 */
const char* ec_cost_units_note(void);
/* kRngAlgorithm, core/include/embcomm/rng.hpp:41 */
const char* ec_rng_algorithm(void);

/* ------------------------------------------------------------------ RNG */
/* substream_seed, core/include/embcomm/rng.hpp:33-38 */
uint64_t ec_substream_seed(uint64_t master, uint64_t index);

/* ---------------------------------------------------------- distributions
 * EmbeddingDistribution (core/include/embcomm/distribution.hpp:19-49) and
 * DistributionSpec materialisation (distribution_spec.hpp:36-67).  Host
 * objects; probabilities and rank maps are computed in the reference's exact
 * arithmetic order so downstream fp64 results are bit-identical. */
typedef struct ec_dist_s* ec_dist;
enum { EC_ZIPF = 0, EC_EXPONENTIAL = 1, EC_HALF_NORMAL = 2, EC_EMPIRICAL = 3 };

int ec_dist_from_probabilities(const double* probs_host, uint64_t n, ec_dist* out); /* distribution.cpp:13-55 */
int ec_dist_uniform(uint64_t n, ec_dist* out);                                      /* distribution.cpp:57-60 */
int ec_dist_materialize(int kind, uint64_t size, double shape, ec_dist* out);       /* distribution_spec.cpp:195-203 */
int ec_dist_materialize_extended(int kind, uint64_t size, double shape, int64_t factor,
                                 ec_dist* out);                                     /* distribution_spec.cpp:215-226 */
int ec_default_shape(int kind, double* out);                                        /* distribution_spec.cpp:85-93 */
void ec_dist_destroy(ec_dist d);
uint64_t ec_dist_size(ec_dist d);
int ec_dist_prob(ec_dist d, uint32_t id, double* out);                              /* distribution.cpp:62-68 */
int ec_dist_prob_at_rank(ec_dist d, uint64_t rank, double* out);                    /* :70-75 */
int ec_dist_id_at_rank(ec_dist d, uint64_t rank, uint32_t* out);                    /* :77-82 */
int ec_dist_rank_of(ec_dist d, uint32_t id, uint64_t* out);                         /* :84-90 */
int ec_dist_top_ids(ec_dist d, uint64_t k, uint32_t* out_host);                     /* :92-98 */
int ec_dist_mass_of(ec_dist d, const uint32_t* ids_host, uint64_t n, double* out);  /* :100-104 */
/* ranked probabilities (non-increasing) and rank->id map; either may be NULL */
int ec_dist_export(ec_dist d, double* ranked_probs_host, uint32_t* rank_to_id_host);
/* value semantics of EmbeddingDistribution (distribution.hpp:18, copyable and
 * immutable): an independent copy; and the ranked probabilities in place
 * (ranked_probs(), distribution.hpp:34), valid until ec_dist_destroy */
int ec_dist_clone(ec_dist d, ec_dist* out);
int ec_dist_ranked_view(ec_dist d, const double** ranked_probs);

/* ------------------------------------------------------------ cost model
 * core/include/embcomm/cost_model.hpp:17-64.  Host fp64, reference
 * summation order (a GPU reduction would reorder the sum). */
typedef struct {
  int64_t num_samples;        /* Q */
  int64_t batch_size;         /* b */
  int64_t lookups_per_sample; /* d */
} ec_workload;                /* WorkloadSpec, cost_model.hpp:17-25 (validated: Q>=b>=1, d>=1) */

typedef struct {
  double index_cost;
  double embedding_cost;
  double total;
} ec_cost; /* CostBreakdown, cost_model.hpp:27-32 */

int ec_workload_validate(const ec_workload* w);                                     /* cost_model.cpp:23-34 */
int ec_batch_presence_prob(double p, int64_t b, double* out);                       /* cost_model.cpp:36-46 */
int ec_expected_unique_per_batch(ec_dist d, int64_t b, double* out);                /* cost_model.cpp:61-63 */
int ec_expected_unique_from_rank(ec_dist d, int64_t b, uint64_t first_rank, double* out); /* :48-59 */
int ec_coalesced_batch_cost(ec_dist d, int64_t b, ec_cost* out);                    /* :65-71 */
int ec_baseline_epoch_cost(const ec_workload* w, double* out);                      /* :73-76 */
int ec_coalesced_epoch_cost(ec_dist d, const ec_workload* w, ec_cost* out);         /* :78-86 */
int ec_cached_epoch_cost(ec_dist d, const ec_workload* w, const uint32_t* cache_ids_host,
                         uint64_t k, ec_cost* out);                                 /* :88-111 */

/* ------------------------------------------------- cache placement policy
 * core/include/embcomm/cache_planner.hpp:16-81 (host). */
typedef struct {
  int64_t total_params;                 /* M */
  int64_t activation_params_per_sample; /* a */
  int64_t embedding_params;             /* d_emb */
  double memory_efficiency;             /* (0, 1] */
} ec_device_model;                      /* DeviceModel, cache_planner.hpp:16-24 */

typedef struct {
  uint32_t candidate_id;
  double presence_gain;
  double threshold;
  double delta_comm;
  int32_t recommend;
} ec_marginal; /* MarginalReport, cache_planner.hpp:34-44 */

typedef struct {
  uint64_t cache_size;
  int64_t batch_size;
  ec_cost expected_epoch_cost;
  int32_t feasible;
  int32_t used_scan_fallback;
} ec_cache_plan; /* CachePlan, cache_planner.hpp:55-62; cached ids returned separately */

int ec_device_model_validate(const ec_device_model* m);                             /* cache_planner.cpp:90-112 */
/* *out = -1 when no batch fits (std::nullopt) */
int ec_max_batch_size(const ec_device_model* m, int64_t cache_size, int64_t* out);  /* :114-136 */
int ec_delta_comm(ec_dist d, const ec_device_model* m, int64_t num_samples,
                  int64_t current_cache_size, ec_marginal* out);                    /* :138-186 */
/* cached_ids_host (capacity >= dist size) may be NULL */
int ec_optimal_cache_size_scan(ec_dist d, const ec_device_model* m, const ec_workload* w,
                               ec_cache_plan* out, uint32_t* cached_ids_host);      /* :188-204 */
int ec_optimal_cache_size_search(ec_dist d, const ec_device_model* m, const ec_workload* w,
                                 ec_cache_plan* out, uint32_t* cached_ids_host);    /* :206-289 */
int ec_memory_io_proxy(ec_dist d, const ec_workload* w, const uint32_t* cache_ids_host,
                       uint64_t k, double* out);                                    /* :291-294 */
/* GPU planner sweeps.  Many expected_unique_from_rank
 * evaluations at once: out[i] = sum over ranks >= first_ranks[i] (NULL: 0) of
 * 1-(1-p)^batch_sizes[i], fp64 terms reduced on the device (~1e-12 relative
 * to the host's sequential sum, not bitwise).  ec_cost_curve evaluates the
 * planner's cost of caching the top-k prefix at the Eq. 7 batch size (clamped
 * to Q) for every k in ks (cache_planner.cpp:24-53); infeasible k give batch
 * -1 and NaN costs.  The bit-exact planner is ec_optimal_cache_size_search. */
int ec_expected_unique_many(ec_dist d, const int64_t* batch_sizes_host, const uint64_t* first_ranks_host,
                            uint64_t n, int device, double* out_host);
int ec_cost_curve(ec_dist d, const ec_device_model* m, const ec_workload* w, const int64_t* ks_host, uint64_t n,
                  int device, ec_cost* out_host, int64_t* batch_out_host);
/* Multi-table placement under one row budget: global top-`budget_rows` by
 * access probability across tables (ties: lower table, then the
 * distribution's own rank order).  Per table the chosen set is always a
 * probability-ranked prefix, i.e. dist.top_ids(k_t) (cache_planner.cpp:71-79).
 * Presence 1-(1-p)^n is monotone in p, so for equal per-table batch sizes
 * this maximises expected cached distinct rows. */
int ec_place_topk_global(const ec_dist* dists, uint32_t num_tables, uint64_t budget_rows,
                         uint64_t* k_per_table_host);

/* --------------------------------------------------------- GPU sampler (K0)
 * DiscreteSampler (core/src/simulator.cpp:110-130) on the device: the CDF is
 * built on the host in the reference's Kahan order, uploaded once; draws are
 * the closed form  u_m = (mix64(seed + (m+1)*0x9E3779B97F4A7C15) >> 11) * 2^-53
 * followed by an fp64 upper_bound — bit-identical ids. */
typedef struct ec_sampler_s* ec_sampler;
int ec_sampler_create(ec_dist d, int device, ec_sampler* out);
void ec_sampler_destroy(ec_sampler s);
/* ids_dev[i] = draw #(start+i) of SplitMix64(seed) */
int ec_sample_stream(ec_sampler s, uint64_t seed, uint64_t start, uint64_t count,
                     uint32_t* ids_dev, void* stream);
/* sample_batch (simulator.cpp:132-143): b*d ids sample-major into a HOST
 * buffer; *rng_state is the SplitMix64 state, advanced by b*d draws exactly
 * as the reference's generator would be. */
int ec_sample_batch(ec_sampler s, int64_t b, int64_t d, uint64_t* rng_state,
                    uint32_t* out_host);

/* -------------------------------------------- GPU Monte Carlo simulator
 * SimResult (core/include/embcomm/simulator.hpp:34-48).  Distinct and
 * non-cached distinct counts per (batch, feature column) are computed on the
 * device (K0 + K1 count mode); mean / std-error / cost are folded on the host
 * in the reference's fixed order, so results are bit-identical. */
typedef struct {
  double unique_mean, unique_std_error;       /* unique_per_batch */
  double non_cached_mean, non_cached_std_error; /* non_cached_unique */
  ec_cost measured_epoch_cost;
  double hot_batch_fraction;
} ec_sim_result;

int ec_measure_unique(ec_sampler s, int64_t batch_size, int64_t trials, uint64_t seed,
                      ec_sim_result* out);                                          /* simulator.cpp:145-167 */
int ec_simulate_epoch(ec_sampler s, const ec_workload* w, const uint32_t* cache_ids_host,
                      uint64_t k, int64_t epochs, uint64_t seed, ec_sim_result* out); /* :169-220 */
/* trace replay through the hot/normal schedule (simulator.cpp:222-273) */
int ec_simulate_trace(const uint32_t* ids_host, uint64_t num_samples, int64_t num_features,
                      uint64_t vocab, int64_t batch_size, const uint32_t* cache_ids_host,
                      uint64_t k, int device, ec_sim_result* out);

/* ----------------------------------------------- traces on the GPU (§8f)
 * classify_samples (core/src/trace.cpp:185-204): hot_host[s] = 1 iff every
 * id of sample s is cached.  build_schedule (trace.cpp:206-240) without
 * shuffle: order_host = hot samples then normal samples, stable;
 * *num_hot = number of hot samples. */
int ec_classify_samples(const uint32_t* ids_host, uint64_t num_samples, int64_t num_features,
                        uint64_t vocab, const uint32_t* cache_ids_host, uint64_t k, int device,
                        uint8_t* hot_host);
int ec_schedule_order(const uint32_t* ids_host, uint64_t num_samples, int64_t num_features,
                      uint64_t vocab, const uint32_t* cache_ids_host, uint64_t k, int device,
                      uint32_t* order_host, uint64_t* num_hot);
/* build_schedule(trace, cache, b, shuffle_seed) (trace.cpp:206-240): the same
 * order, and with shuffle != 0 each class permuted by the reference's seeded
 * Fisher-Yates (SplitMix64(substream_seed(seed, 0)) hot, (seed, 1) normal;
 * trace.cpp:211-222) -- bit-identical to the reference's schedule. */
int ec_build_schedule(const uint32_t* ids_host, uint64_t num_samples, int64_t num_features, uint64_t vocab,
                      const uint32_t* cache_ids_host, uint64_t k, int device, int shuffle, uint64_t seed,
                      uint32_t* order_host, uint64_t* num_hot);
/* build_skew_table (core/src/trace.cpp:128-150): access counts of the
 * num_ids trace ids (histogram on the GPU), observed ids sorted by (count
 * desc, id asc) with the running fraction of all accesses; output arrays need
 * capacity min(num_ids, vocab); *num_entries = observed ids. */
int ec_build_skew_table(const uint32_t* ids_host, uint64_t num_ids, uint64_t vocab, int device,
                        uint32_t* ids_out_host, uint64_t* counts_out_host, double* cum_fraction_out_host,
                        uint64_t* num_entries);
/* estimate_distribution (trace.cpp:161-183): P(e) = (count + s) / (total + s*E). */
int ec_estimate_distribution(const uint32_t* entry_ids_host, const uint64_t* entry_counts_host,
                             uint64_t num_entries, uint64_t total_accesses, uint64_t vocab, double smoothing,
                             ec_dist* out);

/* ------------------------------------------ binary trace ingest (§8f row 4)
 * The reference's Trace (core/include/embcomm/trace.hpp:18-30) in a mapped
 * binary container instead of the desk-scale text format (trace.cpp:51-101):
 * 40-byte little-endian header {char magic[8] "ECTRACE1"; uint32 version 1;
 * uint32 0; int64 d; uint64 E; uint64 Q} then Q*d uint32 ids, sample-major.
 * Validation mirrors parse_trace (d >= 1, 1 <= E <= 2^32-1, non-empty, every
 * id < E; errors name the sample's text-format line, EC_EINVAL). */
typedef struct ec_trace_s* ec_trace;
int ec_trace_save_binary(const char* path, const uint32_t* ids_host, uint64_t num_samples, int64_t num_features,
                         uint64_t vocab);
int ec_trace_open_binary(const char* path, ec_trace* out);  /* mapped read-only */
void ec_trace_destroy(ec_trace t);
int ec_trace_info(ec_trace t, uint64_t* num_samples, int64_t* num_features, uint64_t* vocab);
int ec_trace_ids(ec_trace t, const uint32_t** ids_host);  /* valid until ec_trace_destroy */
/* stream-ordered copy between UVA addresses (pinned host <-> device), e.g. a
 * step's ids onto the GPU: cudaMemcpyAsync(cudaMemcpyDefault) in one call */
int ec_copy_async(void* dst, const void* src, uint64_t bytes, void* stream);
/* the same, pinned (mapped) host -> device pulled by `ctas` CTAs' loads: with
 * the cold tier in pinned host memory the ids share the host link with its row
 * reads, and a few CTAs' pull yields to them where a copy-engine burst starves
 * them.  Other address kinds, misaligned ends or ctas <= 0: ec_copy_async. */
int ec_copy_async_pull(void* dst, const void* src, uint64_t bytes, int ctas, void* stream);
/* samples [first, first+count) -> ids_dev (count*d ids) through pinned
 * double-buffered staging on `stream`; returns when the copies are done */
int ec_trace_upload(ec_trace t, uint64_t first, uint64_t count, uint32_t* ids_dev, void* stream);

/* --------------------------------------------------------- lookup engine
 * No reference counterpart (SURVEY.md §2 "★ new"): row-wise sharded fp32
 * tables, a replicated HBM hot-row cache, per-table batch dedup (K1), hit/miss
 * partition (K2), 128-bit row gather from HBM and from pinned host memory on a
 * side stream (K3), unique-only exchange between shards (K4), pooled
 * EmbeddingBag sum through inverse indices (K5) and dedup-then-scatter-add SGD
 * backward into the owning shard and the cache (K6).
 *
 * Dedup domain (SURVEY §7 hard part 1, mapping M1): all lookups of one table
 * in one batch.  Unique ids are kept in FIRST-OCCURRENCE order — the order in
 * which the reference's UniqueCounter first marks them (simulator.cpp:96-98);
 * inverse[i] is the position of lookup i's id in that list.  The number of
 * uniques and of non-cached uniques per table is exactly what
 * simulate_epoch(Trace{d=1}, n, C) / count_batch_unique count. */
typedef struct ec_tables_s* ec_tables;

enum { EC_STORAGE_HBM = 0, EC_STORAGE_HOST = 1 };

typedef struct {
  uint32_t num_tables;
  uint32_t dim;                  /* D, fp32 elements per row: 4, 8, 16, 32, 64 or 128 */
  const uint64_t* rows_host;     /* E_t per table, each in [1, 2^32-1] */
  int32_t storage;               /* cold tier: EC_STORAGE_HBM or EC_STORAGE_HOST (pinned) */
  int32_t rank, world;           /* row sharding: owner(id) = id % world, local row id / world */
  uint64_t max_lookups_per_table;/* workspace sizing: n_t of any batch */
  uint32_t max_batch_size;       /* workspace sizing: bags per table */
  int32_t device;                /* CUDA ordinal */
} ec_tables_config;

int ec_tables_create(const ec_tables_config* cfg, ec_tables* out);
void ec_tables_destroy(ec_tables t);
/* bytes of device / pinned-host memory held */
int ec_tables_memory(ec_tables t, uint64_t* device_bytes, uint64_t* host_bytes);
/* Per-kernel CUDA-event timing of ec_lookup_fwd/bwd (events on the launching
 * streams; CUDA graphs are bypassed while enabled).  Slots (12): 0 k_insert,
 * 1 k_compact (K1), 2 k_inverse_partition (K1 inverse + K2), 3 k_gather (K3
 * HBM), 4 k_gather_host (K3 pinned host, side stream), 5 exchange (K4),
 * 6 k_pool (K5), 7 k_scatter (K6a), 8 k_apply (K6b), 9 k_apply_host (K6b
 * pinned host, side stream), 10 k_dedup_cluster (K1+K2, one cluster per
 * table), 11 k_clear_miss_sums (per-unique counts and heavy rows' fp64
 * sums a set's last batch left, cleared before its next counting dedup).
 * profile_read returns accumulated ms and call counts per slot (12
 * entries) and the number of kernels the engine launched; reset != 0 clears
 * them. */
int ec_tables_profile(ec_tables t, int enable);
/* Timeline of the profiled kernels since the last call: `count` records of
 * (slot, start ms, end ms), times relative to the first recorded launch, on
 * their own streams (up to `cap` written to out[3*i..3*i+2]). */
int ec_tables_profile_timeline(ec_tables t, double* out, uint64_t cap, uint64_t* count);
/* CUDA-graph replay of the per-batch kernel sequence (default on): the first
 * ec_lookup_fwd/bwd with a given (indices, bag offsets, out) / (grad, lr) on a
 * capturable stream is captured, later ones replay it.  Off, or on the legacy
 * stream, under profiling, inside an outer capture or with world > 1, kernels
 * are launched directly. */
int ec_tables_use_graphs(ec_tables t, int enable);
/* Dedup implementation (identical results): 0 (default, auto) one
 * thread-block cluster per table (insert, flags, scan, emit, inverse and
 * hit/miss in one kernel) when the tables fill the GPU (8*T >= SMs) and every
 * table's batch has <= 32768 lookups, else the tile path; 1 forces the tile
 * path (k_insert -> k_compact -> k_inverse_partition); 2 forces the cluster
 * kernel whenever every table's batch has <= 65536 lookups; 3 one CTA per
 * table (k_dedup_table) whenever every batch has <= 16384 lookups.  Modes
 * 2 and 3 need direct-mapped dedup sets (tables up to 2^27 rows). */
int ec_tables_dedup_mode(ec_tables t, int mode);
/* Gradient reduction per unique row (K6a): 1 one float4 atomic per lookup
 * after warp-level pre-aggregation; 2 transpose — lookups grouped by unique
 * (count, scan, fill) and summed in registers, runs inside a 32-entry chunk
 * stored, boundary runs added atomically; 0 (default) picks the transpose when
 * some table has >= 32768 lookups in the batch. */
int ec_tables_scatter_mode(ec_tables t, int mode);
int ec_tables_profile_read(ec_tables t, double* ms_host, uint64_t* calls_host, uint64_t* launches,
                           int reset);
/* Deterministic synthetic weights: row (t, id) element c =
 *   scale * (2 * ((mix64(seed + 0x9E3779B97F4A7C15 * ((t << 40) ^ (id * D + c))) >> 40) * 2^-24) - 1)
 * in fp32; every rank can evaluate any row, so shards and replicated cache
 * rows initialise consistently without communication. */
int ec_tables_init_synthetic(ec_tables t, uint64_t seed, float scale, void* stream);
/* Cache placement: cached_ids[t] lists the k_t ids of table t held in the
 * replicated HBM cache (distinct, in range; typically dist.top_ids(k_t)).
 * Replaces any previous placement; cached rows are (re)initialised from the
 * current authoritative values when world == 1, and from the synthetic init
 * (seed/scale of the last ec_tables_init_synthetic) otherwise. */
int ec_tables_place_cache(ec_tables t, const uint32_t* const* cached_ids_host,
                          const uint64_t* k_host);
/* Authoritative row values (cache copy for cached ids, else the shard) —
 * host copies for tests/checkpointing.  Ids must be owned by this rank unless
 * cached. */
int ec_tables_read_rows(ec_tables t, uint32_t table, const uint32_t* ids_host, uint64_t n,
                        float* out_host);
int ec_tables_write_rows(ec_tables t, uint32_t table, const uint32_t* ids_host, uint64_t n,
                         const float* rows_host);

/* One batch: lookups of table t are indices_dev[table_offsets_host[t] ..
 * table_offsets_host[t+1]); each table has batch_size bags.  Bags are either
 * fixed-size (bag_offsets_dev == NULL: bag s of table t is lookups
 * [s*P, (s+1)*P) of that table, P = pooling) or CSR: bag_offsets_dev has
 * num_tables*batch_size+1 entries, table-major, in global lookup positions. */
typedef struct {
  const uint32_t* indices_dev;
  const int64_t* table_offsets_host;
  const int64_t* bag_offsets_dev;
  uint32_t batch_size;
  uint32_t pooling;
} ec_batch;

/* Forward: out_dev[s, t*D + c] = sum over bag (t, s) of row values.  Runs
 * K1..K5 on `stream` (host misses on an internal side stream joined by an
 * event).  No host synchronisation unless world > 1. */
int ec_lookup_fwd(ec_tables t, const ec_batch* batch, float* out_dev, void* stream);
/* Hot/normal scheduling of a dataset (classify_samples +
 * build_schedule, core/src/trace.cpp:185-240, with one id per table per
 * sample): ids_dev is sample-major [q, num_tables]; a sample is hot iff every
 * id is cached under the current placement.  order_dev (q entries) receives
 * the hot samples then the normal ones, each in original order; *num_hot is
 * the hot count (synchronises `stream`).  ec_tables_gather_batch writes
 * samples order[first .. first+count) as a table-major pooling-1 batch
 * (indices_dev[t*count + i]) ready for ec_lookup_fwd; batches cut inside the
 * hot prefix never touch the cold tier. */
int ec_tables_schedule(ec_tables t, const uint32_t* ids_dev, uint64_t num_samples, uint32_t* order_dev,
                       uint64_t* num_hot, void* stream);
int ec_tables_gather_batch(ec_tables t, const uint32_t* ids_dev, const uint32_t* order_dev, uint64_t first,
                           uint32_t count, uint32_t* indices_dev, void* stream);
/* Start the next batch while the current one finishes (single rank, or a
 * rank on the peer-memory exchange, where the next batch's pinned-host rows
 * are read once the current forward passed its step barrier and the ones the
 * current step updates are re-read after the next barrier): its
 * dedup, hit/miss partition and pinned-host miss gather run on internal
 * streams into a second buffer set, overlapping the current backward; the
 * next ec_lookup_fwd with the same indices_dev consumes them (up to 2 batches
 * may be pending; forwards consume them in prefetch order).  Host-tier rows
 * the current backward updates are refreshed in the prefetched copy, so
 * results equal the unpipelined sequence.  Stream-ordered on `stream`: it
 * starts after the work already enqueued there, so pass the stream that
 * produces indices_dev (e.g. an input-copy stream; passing the compute stream
 * instead serialises the prefetch behind the current forward).  Same
 * geometry as the last forward required. */
int ec_lookup_prefetch(ec_tables t, const ec_batch* batch, void* stream);
/* Make `stream` wait for a pending prefetch and for the deferred host-tier
 * write-back of the last backward (no-op without either). */
int ec_lookup_prefetch_wait(ec_tables t, void* stream);
/* Discard every pending prefetched batch (their buffer sets become free). */
int ec_lookup_prefetch_drop(ec_tables t, void* stream);
/* Backward of the last forward: grad_dev laid out like out_dev; applies
 * w <- w - lr * (sum of grads of every lookup of the row) to the cache copy
 * of cached rows and to the owning shard of the others (K6).  Single rank,
 * pinned-host tier: the host write-back keeps running on an internal stream
 * (overlapping the next forward); every later engine call that needs it
 * orders itself after it, and ec_lookup_prefetch_wait joins it into a
 * caller's stream (a device synchronise also covers it). */
int ec_lookup_bwd(ec_tables t, const float* grad_dev, float lr, void* stream);

typedef struct {
  uint64_t lookups;        /* sum_t n_t (with duplicates) */
  uint64_t unique_rows;    /* sum_t U_t */
  uint64_t hit_rows;       /* sum_t |U_t ∩ C_t| */
  uint64_t miss_rows;      /* sum_t |U_t \ C_t| = model rows (reference embedding units) */
  uint64_t index_units;    /* sum_t n_t (M1: one index unit per lookup) */
  uint64_t model_bytes;    /* miss_rows*D*4 + index_units*4 */
  uint64_t wire_rows;      /* misses owned by another rank (fetched over the exchange) */
  uint64_t wire_bytes;     /* bytes actually sent + received by this rank's exchange */
  uint64_t hot_tables;     /* tables whose batch touched no uncached row */
  uint64_t hot_sync_rows;  /* peer exchange: hot-row gradients sent to other owners + updated hot rows copied
                              from them (the replicated cache's sync; outside the reference's cost model) */
  uint64_t hot_sync_bytes; /* their bytes (slot index + row); included in wire_bytes */
} ec_batch_stats;
/* Synchronises `stream`; per-table arrays (length num_tables) may be NULL. */
int ec_lookup_stats(ec_tables t, void* stream, ec_batch_stats* out, int64_t* unique_per_table_host,
                    int64_t* miss_per_table_host);
/* Asynchronous form for training loops: ec_lookup_stats_enqueue copies the
 * last forward's counters into pinned ring slot `slot` (0..EC_STATS_SLOTS-1)
 * on `stream` without synchronising; ec_lookup_stats_collect waits for that
 * copy only and decodes it like ec_lookup_stats (reference counterpart: the
 * per-batch unique/miss counts of embcomm simulate_epoch). */
#define EC_STATS_SLOTS 4
int ec_lookup_stats_enqueue(ec_tables t, void* stream, int slot);
int ec_lookup_stats_collect(ec_tables t, int slot, ec_batch_stats* out, int64_t* unique_per_table_host,
                            int64_t* miss_per_table_host);
/* Parity exports of the last forward (synchronise): unique ids of table t in
 * first-occurrence order, inverse (positions into that list), per-unique hit
 * flag, and the gathered unique rows. */
int ec_export_unique(ec_tables t, uint32_t table, uint32_t* unique_host, uint64_t cap,
                     uint64_t* count);
int ec_export_inverse(ec_tables t, uint32_t table, uint32_t* inverse_host);
int ec_export_hit(ec_tables t, uint32_t table, uint8_t* hit_host);
int ec_export_rows(ec_tables t, uint32_t table, float* rows_host);

/* ------------------------------------------------- multi-GPU (K4, NCCL)
 * One process per GPU.  Rank 0 calls ec_comm_unique_id and distributes the
 * 128 bytes (e.g. torch.distributed broadcast); every rank then attaches. */
int ec_comm_unique_id(uint8_t* id128_host);
int ec_tables_attach_comm(ec_tables t, const uint8_t* id128_host);

/* Host-side sharding math (no GPU): rows of each table owned by `rank`
 * (owner(id) = id % world), and the per-batch exchange plan of `rank` from the
 * all-gathered count matrix counts[r*(world+1) + o] = requests rank r sends to
 * owner o (o < world) and rank r's cache-hit count (o = world): send/recv
 * counts and offsets per peer, and every rank's hit-list count and offset. */
int ec_shard_rows(const uint64_t* rows_host, uint32_t num_tables, int world, int rank, uint64_t* local_rows_host);
int ec_exchange_plan(const int* counts_host, int world, int rank, int64_t* send_cnt, int64_t* send_off,
                     int64_t* recv_cnt, int64_t* recv_off, int64_t* hot_cnt, int64_t* hot_off);

/* In-process loopback group: `n` ranks (member r has rank r of world n) on one
 * device, driven in lock step with device-to-device copies in place of NCCL.
 * Same routing, owner serve, gradient return and rank-ordered replica update
 * as the NCCL path; used to exercise the sharded data path on one GPU. */
typedef struct ec_group_s* ec_group;
int ec_group_create(ec_tables* members, int n, ec_group* out);
void ec_group_destroy(ec_group g);
int ec_group_lookup_fwd(ec_group g, const ec_batch* batches, float* const* outs_dev, void* stream);
int ec_group_lookup_bwd(ec_group g, const float* const* grads_dev, float lr, void* stream);
/* Switch a group to the peer-memory exchange (enable != 0): remote rows are
 * loaded straight from the owner's shard inside the gather kernel, owner
 * updates are atomics into the owner's rows, hot-row gradient lists are
 * published and applied in rank order, and the ranks meet at device-side
 * barriers (flag words) instead of copies.  Pinned-host shards: every rank
 * reads remote owners' rows from their (shared, memfd-backed) host shards over
 * its own link, and sends miss gradients to the owner's inbox, applied by the
 * owner in rank order.  The same kernels run across processes after
 * ec_tables_p2p_export/import. */
int ec_group_set_p2p(ec_group g, int enable);

/* Multi-process peer-memory exchange (one process per GPU on one NVLink
 * domain).  The reference has no exchange code: it prices one (the E minus C
 * rows of cached_epoch_cost, core/src/cost_model.cpp:88-111) and SURVEY.md
 * 8(e) plans it as NCCL all-to-alls (ec_tables_attach_comm).  This transport
 * replaces those all-to-alls with loads and atomics over NVLink.  export: this rank's peer-visible allocations as
 * CUDA IPC handles (blob == NULL -> *len only); the caller all-gathers the
 * blobs (rank-major, *len bytes each) and passes them to import, after which
 * ec_lookup_fwd/bwd use the peer path (no ec_tables_set_comm needed).  Every
 * rank must call fwd/bwd the same number of times: each step ends at a
 * device-side barrier. */
int ec_tables_p2p_export(ec_tables t, uint8_t* blob, uint64_t cap, uint64_t* len);
int ec_tables_p2p_import(ec_tables t, const uint8_t* blobs, uint64_t blob_len);
/* Back to the transport set by ec_tables_attach_comm (e.g. when some rank's
 * import failed: every rank must use the same transport). */
int ec_tables_p2p_disable(ec_tables t);

#ifdef __cplusplus
}
#endif
#endif /* EMBCOMM_GPU_H_ */
