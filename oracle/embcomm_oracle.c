/*
 * TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.
 *
 * CPU restatement ("oracle") of the embedding-lookup hot path, in plain C.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it, and only as the checker.  The product
 * library (paper_2411_01611_b200/csrc) never links or calls it.
 *
 * Parity status
 *   - Pinned against the compiled reference (oracle/_ref/libembcomm_ref.so,
 *     built from /root/reference by oracle/Makefile) and against the
 *     reference's own known-answer tests (tests/test_oracle.py):
 *       orc_stream_u64 / orc_substream_seed / orc_build_cdf / orc_draw /
 *       orc_sample  (sampler bit-exact vs sample_batch, measure_unique,
 *                    simulate_epoch streams)
 *       orc_count_segments (distinct / non-cached distinct counts bit-exact vs
 *                    simulate_epoch and the trace-replay KAT)
 *   - Restatements with NO reference counterpart (the reference materialises
 *     no sets, rows, pools or gradients) — "parity unpinned"
 *     beyond the counts they must agree with:
 *       orc_dedup (unique set in first-occurrence order + inverse),
 *       orc_partition (hit/miss split), orc_gather, orc_pool, orc_backward_sgd.
 *
 * Citations are file:line into /root/reference/proj.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define GOLDEN 0x9E3779B97F4A7C15ull

/* core/include/embcomm/rng.hpp:16-21 (output mix of SplitMix64::next) */
static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* rng.hpp:33-38 */
uint64_t orc_substream_seed(uint64_t master, uint64_t index) {
  return mix64(master + (index + 1) * GOLDEN);
}

/* m-th output (0-based) of SplitMix64(seed): the state after m+1 steps is
 * seed + (m+1)*GOLDEN (rng.hpp:17), so draws are a closed form of (seed, m). */
uint64_t orc_stream_u64(uint64_t seed, uint64_t m) { return mix64(seed + (m + 1) * GOLDEN); }

/* rng.hpp:24 */
static inline double to_unit(uint64_t x) { return (double)(x >> 11) * 0x1.0p-53; }

/* DiscreteSampler ctor, simulator.cpp:110-123: Kahan running sum over ranked
 * probabilities, last entry forced to exactly 1.0. */
void orc_build_cdf(const double* ranked, uint64_t E, double* cdf) {
  double running = 0.0, carry = 0.0;
  for (uint64_t r = 0; r < E; ++r) {
    const double y = ranked[r] - carry;
    const double t = running + y;
    carry = (t - running) - y;
    running = t;
    cdf[r] = running;
  }
  if (E) cdf[E - 1] = 1.0;
}

/* DiscreteSampler::draw, simulator.cpp:125-130: upper_bound(u), clamp to the
 * last rank, map rank -> id (rank_to_id may be NULL for the identity). */
uint32_t orc_draw(const double* cdf, const uint32_t* rank_to_id, uint64_t E, double u) {
  uint64_t lo = 0, hi = E; /* first index with cdf[i] > u */
  while (lo < hi) {
    const uint64_t mid = lo + (hi - lo) / 2;
    if (cdf[mid] > u) hi = mid; else lo = mid + 1;
  }
  if (lo == E) lo = E - 1;
  return rank_to_id ? rank_to_id[lo] : (uint32_t)lo;
}

/* ids[i] = draw #(start+i) of SplitMix64(seed): sample_batch
 * (simulator.cpp:132-143) and the per-epoch loop of simulate_epoch
 * (simulator.cpp:186-192) consume exactly this stream. */
void orc_sample(const double* cdf, const uint32_t* rank_to_id, uint64_t E, uint64_t seed,
                uint64_t start, uint64_t count, uint32_t* out) {
  for (uint64_t i = 0; i < count; ++i)
    out[i] = orc_draw(cdf, rank_to_id, E, to_unit(orc_stream_u64(seed, start + i)));
}

/* ---- a small open-addressing set used by the restatements ---------------- */
typedef struct {
  uint32_t* keys;
  uint32_t* vals;
  uint64_t mask;
} oset;

static int oset_init(oset* s, uint64_t n) {
  uint64_t cap = 16;
  while (cap < 2 * n + 2) cap <<= 1;
  s->keys = (uint32_t*)malloc(cap * sizeof(uint32_t));
  s->vals = (uint32_t*)malloc(cap * sizeof(uint32_t));
  if (!s->keys || !s->vals) return -1;
  memset(s->keys, 0xFF, cap * sizeof(uint32_t));
  s->mask = cap - 1;
  return 0;
}
static void oset_free(oset* s) { free(s->keys); free(s->vals); }
/* returns pointer to the value slot; *fresh = 1 when newly inserted */
static uint32_t* oset_put(oset* s, uint32_t key, int* fresh) {
  uint64_t h = (key * 0x9E3779B1u) & s->mask;
  for (;;) {
    if (s->keys[h] == key) { *fresh = 0; return &s->vals[h]; }
    if (s->keys[h] == 0xFFFFFFFFu) { s->keys[h] = key; *fresh = 1; return &s->vals[h]; }
    h = (h + 1) & s->mask;
  }
}

/* Per-segment distinct / non-cached-distinct counts.
 * count_batch_unique, simulator.cpp:85-106: for one column, `mark` returns
 * true the first time an id is seen (UniqueCounter, :14-35); the non-cached
 * counter marks only ids with !cached[id] (:99).  Segment j covers
 * ids[off[j] .. off[j+1]) with the given element stride (1 = contiguous).
 * cached[j] may be NULL (no cache) — it is a byte mask over the segment's
 * vocabulary. */
int orc_count_segments(const uint32_t* ids, const uint64_t* off, uint64_t n_seg,
                       const uint8_t* const* cached, int64_t* out_all, int64_t* out_nc) {
  for (uint64_t j = 0; j < n_seg; ++j) {
    const uint64_t n = off[j + 1] - off[j];
    oset s;
    if (oset_init(&s, n)) return -1;
    int64_t all = 0, nc = 0;
    for (uint64_t i = off[j]; i < off[j + 1]; ++i) {
      int fresh;
      oset_put(&s, ids[i], &fresh);
      if (fresh) {
        ++all;
        if (!(cached && cached[j] && cached[j][ids[i]])) ++nc;
      }
    }
    oset_free(&s);
    out_all[j] = all;
    out_nc[j] = nc;
  }
  return 0;
}

/* Dedup restatement (no reference counterpart).
 * Canonical order: the unique ids in the order the reference's UniqueCounter
 * first marks them while walking the segment front to back
 * (simulator.cpp:96-98), i.e. first-occurrence order.  inverse[i] is the
 * position of ids[i] in that list.  Returns U. */
uint64_t orc_dedup(const uint32_t* ids, uint64_t n, uint32_t* unique, uint32_t* inverse) {
  oset s;
  if (oset_init(&s, n)) return (uint64_t)-1;
  uint64_t u = 0;
  for (uint64_t i = 0; i < n; ++i) {
    int fresh;
    uint32_t* v = oset_put(&s, ids[i], &fresh);
    if (fresh) { *v = (uint32_t)u; unique[u++] = ids[i]; }
    inverse[i] = *v;
  }
  oset_free(&s);
  return u;
}

/* Hit/miss partition of a unique list against a cache-slot remap
 * (slot[id] >= 0: cached at that slot; < 0: miss).  Restates cache_mask +
 * the !cached[id] test (simulator.cpp:65-75, :99) on materialised sets.
 * hit[u] = 1/0; returns the miss count (the non-cached distinct count). */
uint64_t orc_partition(const uint32_t* unique, uint64_t U, const int32_t* slot, uint8_t* hit) {
  uint64_t miss = 0;
  for (uint64_t u = 0; u < U; ++u) {
    hit[u] = slot[unique[u]] >= 0;
    miss += !hit[u];
  }
  return miss;
}

/* Row gather: out[u] = table[unique[u]] (rows copied unchanged). */
void orc_gather(const float* table, uint64_t D, const uint32_t* unique, uint64_t U, float* out) {
  for (uint64_t u = 0; u < U; ++u) memcpy(out + u * D, table + (uint64_t)unique[u] * D, D * sizeof(float));
}

/* Sum pooling through inverse indices.  Bag k of the segment covers lookups
 * bag_off[k] .. bag_off[k+1].  out32 accumulates in fp32 in lookup order;
 * out64 (optional) in fp64 — the 1e-5-relative check uses out64. */
void orc_pool(const float* urows, uint64_t D, const uint32_t* inverse, const int64_t* bag_off,
              uint64_t n_bags, float* out32, uint64_t out_stride, double* out64) {
  for (uint64_t k = 0; k < n_bags; ++k) {
    for (uint64_t c = 0; c < D; ++c) {
      float a32 = 0.0f;
      double a64 = 0.0;
      for (int64_t i = bag_off[k]; i < bag_off[k + 1]; ++i) {
        const float v = urows[(uint64_t)inverse[i] * D + c];
        a32 += v;
        a64 += v;
      }
      if (out32) out32[k * out_stride + c] = a32;
      if (out64) out64[k * D + c] = a64;
    }
  }
}

/* Backward restatement: per unique row, the fp64 sum of the pooled-output
 * gradients of every lookup that referenced it (in lookup order), then plain
 * SGD  w <- w - lr * g  applied to the row gathered for it.  grad rows are
 * addressed like the pooled output (bag k at grad[k*grad_stride]).
 * rows_in[u] is the pre-update row, rows_out[u] receives fp32(w - lr*g). */
void orc_backward_sgd(const float* grad, uint64_t grad_stride, uint64_t D,
                      const uint32_t* inverse, const int64_t* bag_off, uint64_t n_bags,
                      uint64_t U, const float* rows_in, float lr, double* ugrad,
                      float* rows_out) {
  memset(ugrad, 0, U * D * sizeof(double));
  for (uint64_t k = 0; k < n_bags; ++k)
    for (int64_t i = bag_off[k]; i < bag_off[k + 1]; ++i)
      for (uint64_t c = 0; c < D; ++c)
        ugrad[(uint64_t)inverse[i] * D + c] += grad[k * grad_stride + c];
  if (rows_out)
    for (uint64_t x = 0; x < U * D; ++x)
      rows_out[x] = (float)((double)rows_in[x] - (double)lr * ugrad[x]);
}
