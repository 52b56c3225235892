"""TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.

ctypes access to the two checkers:

* ``ref``  — the UNMODIFIED reference core compiled from /root/reference by
  oracle/Makefile into ``oracle/_ref/libembcomm_ref.so`` (plus the extern "C"
  shim ``oracle/ref_shim.cpp``).  The built .so travels to the GPU box, so the
  GPU parity tests and bench.py's reference arm call the reference itself.
* ``orc``  — the plain-C restatement ``oracle/embcomm_oracle.c`` (pinned
  against ``ref``; see its header for what is pinned and what is not).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this package, and only as the checker.
The product package ``paper_2411_01611_b200`` never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libembcomm_ref.so")
ORC_SO = os.path.join(HERE, "lib", "libembcomm_oracle.so")

KIND = {"zipf": 0, "exponential": 1, "half_normal": 2}


def build(with_ref: bool | None = None) -> None:
    """Compile the C restatement, and the reference when /root/reference exists."""
    targets = ["oracle"]
    if with_ref is None:
        with_ref = os.path.isdir("/root/reference/proj/core/src")
    if with_ref:
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


u32p = lambda a: _p(a, C.c_uint32)  # noqa: E731
u64p = lambda a: _p(a, C.c_uint64)  # noqa: E731
i64p = lambda a: _p(a, C.c_int64)  # noqa: E731
f64p = lambda a: _p(a, C.c_double)  # noqa: E731
f32p = lambda a: _p(a, C.c_float)  # noqa: E731
u8p = lambda a: _p(a, C.c_uint8)  # noqa: E731
i32p = lambda a: _p(a, C.c_int32)  # noqa: E731


class RefSim(C.Structure):
    _fields_ = [(n, C.c_double) for n in (
        "unique_mean", "unique_se", "nc_mean", "nc_se",
        "index_cost", "embedding_cost", "total", "hot_batch_fraction")]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


_ref = None
_orc = None


def ref_lib():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(f"{REF_SO} missing: run `make -C oracle ref` where /root/reference exists")
        lib = C.CDLL(REF_SO)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_substream_seed.restype = C.c_uint64
        lib.ref_substream_seed.argtypes = [C.c_uint64, C.c_uint64]
        lib.ref_dist_size.restype = C.c_uint64
        lib.ref_dist_size.argtypes = [C.c_void_p]
        lib.ref_dist_free.argtypes = [C.c_void_p]
        lib.ref_dist_export.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        _ref = lib
    return _ref


def orc_lib():
    global _orc
    if _orc is None:
        if not os.path.exists(ORC_SO):
            build(with_ref=False)
        lib = C.CDLL(ORC_SO)
        lib.orc_substream_seed.restype = C.c_uint64
        lib.orc_substream_seed.argtypes = [C.c_uint64, C.c_uint64]
        lib.orc_stream_u64.restype = C.c_uint64
        lib.orc_stream_u64.argtypes = [C.c_uint64, C.c_uint64]
        lib.orc_draw.restype = C.c_uint32
        lib.orc_draw.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_double]
        lib.orc_sample.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64,
                                   C.c_uint64, C.c_uint64, C.c_void_p]
        lib.orc_build_cdf.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p]
        lib.orc_dedup.restype = C.c_uint64
        lib.orc_dedup.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p]
        lib.orc_partition.restype = C.c_uint64
        lib.orc_partition.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p]
        lib.orc_count_segments.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p,
                                           C.c_void_p, C.c_void_p]
        lib.orc_gather.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, C.c_void_p]
        lib.orc_pool.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_uint64,
                                 C.c_void_p, C.c_uint64, C.c_void_p]
        lib.orc_backward_sgd.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p,
                                         C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p,
                                         C.c_float, C.c_void_p, C.c_void_p]
        _orc = lib
    return _orc


def _check(rc):
    if rc != 0:
        raise RefError(rc, ref_lib().ref_last_error().decode())


# ---------------------------------------------------------------- reference
class RefDist:
    """Handle on a reference ``EmbeddingDistribution`` (distribution.hpp:19-49)."""

    def __init__(self, handle):
        self.h = C.c_void_p(handle)

    def __del__(self):
        if getattr(self, "h", None) and _ref is not None:
            _ref.ref_dist_free(self.h)
            self.h = None

    @classmethod
    def parametric(cls, kind: str, size: int, shape: float):
        h = C.c_void_p()
        _check(ref_lib().ref_dist_parametric(C.c_int(KIND[kind]), C.c_uint64(size),
                                              C.c_double(shape), C.byref(h)))
        return cls(h.value)

    @classmethod
    def extended(cls, kind: str, size: int, shape: float, factor: int):
        h = C.c_void_p()
        _check(ref_lib().ref_dist_extended(C.c_int(KIND[kind]), C.c_uint64(size),
                                            C.c_double(shape), C.c_int64(factor), C.byref(h)))
        return cls(h.value)

    @classmethod
    def from_probs(cls, probs):
        p = np.ascontiguousarray(probs, dtype=np.float64)
        h = C.c_void_p()
        _check(ref_lib().ref_dist_from_probs(f64p(p), C.c_uint64(p.size), C.byref(h)))
        return cls(h.value)

    @classmethod
    def uniform(cls, n):
        h = C.c_void_p()
        _check(ref_lib().ref_dist_uniform(C.c_uint64(n), C.byref(h)))
        return cls(h.value)

    @property
    def size(self):
        return int(ref_lib().ref_dist_size(self.h))

    def export(self):
        n = self.size
        p = np.empty(n, np.float64)
        r2i = np.empty(n, np.uint32)
        ref_lib().ref_dist_export(self.h, p.ctypes.data, r2i.ctypes.data)
        return p, r2i

    def top_ids(self, k):
        out = np.empty(k, np.uint32)
        _check(ref_lib().ref_dist_top_ids(self.h, C.c_uint64(k), u32p(out)))
        return out


def ref_substream_seed(master, index):
    return int(ref_lib().ref_substream_seed(master, index))


def ref_sample_batch(dist: RefDist, b, d, rng_seed):
    out = np.empty(b * d, np.uint32)
    _check(ref_lib().ref_sample_batch(dist.h, C.c_int64(b), C.c_int64(d), C.c_uint64(rng_seed),
                                      u32p(out)))
    return out


def ref_measure_unique(dist, b, trials, seed):
    r = RefSim()
    _check(ref_lib().ref_measure_unique(dist.h, C.c_int64(b), C.c_int64(trials),
                                        C.c_uint64(seed), C.byref(r)))
    return r.as_dict()


def ref_simulate_epoch(dist, q, b, d, cache, epochs, seed):
    c = np.ascontiguousarray(cache, dtype=np.uint32)
    r = RefSim()
    _check(ref_lib().ref_simulate_epoch(dist.h, C.c_int64(q), C.c_int64(b), C.c_int64(d),
                                        u32p(c), C.c_uint64(c.size), C.c_int64(epochs),
                                        C.c_uint64(seed), C.byref(r)))
    return r.as_dict()


def ref_simulate_trace(ids, d, vocab, b, cache):
    ids = np.ascontiguousarray(ids, dtype=np.uint32)
    c = np.ascontiguousarray(cache, dtype=np.uint32)
    r = RefSim()
    _check(ref_lib().ref_simulate_trace(u32p(ids), C.c_uint64(ids.size // d), C.c_int64(d),
                                        C.c_uint64(vocab), C.c_int64(b), u32p(c),
                                        C.c_uint64(c.size), C.byref(r)))
    return r.as_dict()


def ref_segment_counts(ids, seg_off, seg_vocab, seg_cache, threads=1, want_all=True):
    """Distinct / non-cached distinct count per segment through the reference's
    simulate_epoch(Trace{d=1}, n, C) (simulator.cpp:222-273)."""
    ids = np.ascontiguousarray(ids, dtype=np.uint32)
    off = np.ascontiguousarray(seg_off, dtype=np.uint64)
    n_seg = off.size - 1
    voc = np.ascontiguousarray(seg_vocab, dtype=np.uint64)
    caches = [np.ascontiguousarray(c if c is not None else [], dtype=np.uint32) for c in seg_cache]
    ptrs = (C.c_void_p * n_seg)(*[c.ctypes.data if c.size else None for c in caches])
    lens = np.array([c.size for c in caches], dtype=np.uint64)
    out_all = np.zeros(n_seg, np.int64)
    out_nc = np.zeros(n_seg, np.int64)
    _check(ref_lib().ref_segment_counts(u32p(ids), u64p(off), C.c_uint64(n_seg), u64p(voc), ptrs,
                                        u64p(lens), C.c_int(threads),
                                        i64p(out_all) if want_all else None, i64p(out_nc)))
    return out_all, out_nc


def ref_cost(fn, *args):
    lib = ref_lib()
    if fn == "batch_presence_prob":
        out = C.c_double()
        _check(lib.ref_batch_presence_prob(C.c_double(args[0]), C.c_int64(args[1]), C.byref(out)))
        return out.value
    if fn == "expected_unique_from_rank":
        dist, b, first = args
        out = C.c_double()
        _check(lib.ref_expected_unique_from_rank(dist.h, C.c_int64(b), C.c_uint64(first), C.byref(out)))
        return out.value
    if fn == "coalesced_batch_cost":
        dist, b = args
        out = np.zeros(3)
        _check(lib.ref_coalesced_batch_cost(dist.h, C.c_int64(b), f64p(out)))
        return tuple(out)
    if fn == "baseline_epoch_cost":
        out = C.c_double()
        _check(lib.ref_baseline_epoch_cost(*[C.c_int64(x) for x in args], C.byref(out)))
        return out.value
    if fn == "coalesced_epoch_cost":
        dist, q, b, d = args
        out = np.zeros(3)
        _check(lib.ref_coalesced_epoch_cost(dist.h, C.c_int64(q), C.c_int64(b), C.c_int64(d), f64p(out)))
        return tuple(out)
    if fn == "cached_epoch_cost":
        dist, q, b, d, cache = args
        c = np.ascontiguousarray(cache, dtype=np.uint32)
        out = np.zeros(3)
        _check(lib.ref_cached_epoch_cost(dist.h, C.c_int64(q), C.c_int64(b), C.c_int64(d), u32p(c),
                                         C.c_uint64(c.size), f64p(out)))
        return tuple(out)
    if fn == "memory_io_proxy":
        dist, q, b, d, cache = args
        c = np.ascontiguousarray(cache, dtype=np.uint32)
        out = C.c_double()
        _check(lib.ref_memory_io_proxy(dist.h, C.c_int64(q), C.c_int64(b), C.c_int64(d), u32p(c),
                                       C.c_uint64(c.size), C.byref(out)))
        return out.value
    raise KeyError(fn)


def ref_max_batch_size(m, a, d_emb, eff, k):
    out = C.c_int64()
    _check(ref_lib().ref_max_batch_size(C.c_int64(m), C.c_int64(a), C.c_int64(d_emb),
                                        C.c_double(eff), C.c_int64(k), C.byref(out)))
    return None if out.value < 0 else out.value


def ref_plan(dist, m, a, d_emb, eff, q, d, search=True):
    plan = np.zeros(4, np.int64)
    cost = np.zeros(3)
    ids = np.zeros(dist.size, np.uint32)
    _check(ref_lib().ref_plan(dist.h, C.c_int64(m), C.c_int64(a), C.c_int64(d_emb), C.c_double(eff),
                              C.c_int64(q), C.c_int64(d), C.c_int(1 if search else 0), i64p(plan),
                              f64p(cost), u32p(ids)))
    return {"cache_size": int(plan[0]), "batch_size": int(plan[1]), "feasible": bool(plan[2]),
            "used_scan_fallback": bool(plan[3]), "cost": tuple(cost),
            "cached_ids": ids[: plan[0]].copy()}


def ref_delta_comm(dist, m, a, d_emb, eff, q, k):
    out = np.zeros(5)
    _check(ref_lib().ref_delta_comm(dist.h, C.c_int64(m), C.c_int64(a), C.c_int64(d_emb),
                                    C.c_double(eff), C.c_int64(q), C.c_int64(k), f64p(out)))
    return {"candidate_id": int(out[0]), "presence_gain": out[1], "threshold": out[2],
            "delta_comm": out[3], "recommend": bool(out[4])}


def ref_load_trace(path):
    """The reference's parse_trace of a text trace file -> (d, vocab, ids)."""
    d, vocab, n = C.c_int64(), C.c_uint64(), C.c_uint64()
    _check(ref_lib().ref_load_trace(os.fsencode(path), C.byref(d), C.byref(vocab), None, C.c_uint64(0),
                                    C.byref(n)))
    ids = np.empty(n.value, np.uint32)
    _check(ref_lib().ref_load_trace(os.fsencode(path), C.byref(d), C.byref(vocab), ids.ctypes.data_as(C.c_void_p),
                                    C.c_uint64(ids.size), C.byref(n)))
    return int(d.value), int(vocab.value), ids


def ref_build_skew_table(ids, d, vocab):
    ids = np.ascontiguousarray(ids, dtype=np.uint32)
    oid = np.zeros(vocab, np.uint32)
    cnt = np.zeros(vocab, np.uint64)
    cum = np.zeros(vocab, np.float64)
    n = C.c_uint64()
    _check(ref_lib().ref_build_skew_table(u32p(ids), C.c_uint64(ids.size // d), C.c_int64(d),
                                          C.c_uint64(vocab), u32p(oid), u64p(cnt), f64p(cum),
                                          C.byref(n)))
    k = n.value
    return oid[:k].copy(), cnt[:k].copy(), cum[:k].copy()


def ref_estimate_distribution(ids, d, vocab, smoothing=0.0):
    ids = np.ascontiguousarray(ids, dtype=np.uint32)
    h = C.c_void_p()
    _check(ref_lib().ref_estimate_distribution(u32p(ids), C.c_uint64(ids.size // d), C.c_int64(d),
                                               C.c_uint64(vocab), C.c_double(smoothing), C.byref(h)))
    return RefDist(h.value)


def ref_classify_samples(ids, d, vocab, cache):
    ids = np.ascontiguousarray(ids, dtype=np.uint32)
    c = np.ascontiguousarray(cache, dtype=np.uint32)
    n = ids.size // d
    hot = np.zeros(n, np.uint8)
    _check(ref_lib().ref_classify_samples(u32p(ids), C.c_uint64(n), C.c_int64(d), C.c_uint64(vocab),
                                          u32p(c), C.c_uint64(c.size), u8p(hot)))
    return hot


def ref_build_schedule(ids, d, vocab, cache, b, shuffle_seed=-1):
    ids = np.ascontiguousarray(ids, dtype=np.uint32)
    c = np.ascontiguousarray(cache, dtype=np.uint32)
    n = ids.size // d
    order = np.zeros(n, np.uint32)
    sizes = np.zeros(n + 2, np.uint64)
    nh = C.c_uint64()
    nb = C.c_uint64()
    _check(ref_lib().ref_build_schedule(u32p(ids), C.c_uint64(n), C.c_int64(d), C.c_uint64(vocab),
                                        u32p(c), C.c_uint64(c.size), C.c_int64(b),
                                        C.c_int64(shuffle_seed), u32p(order), u64p(sizes),
                                        C.byref(nh), C.byref(nb)))
    return order, sizes[: nb.value].copy(), int(nh.value)


# -------------------------------------------------------------- restatement
class Sampler:
    """Restated DiscreteSampler (simulator.cpp:110-130) over exported ranked
    probabilities and the rank->id map."""

    def __init__(self, ranked_probs, rank_to_id=None):
        self.ranked = np.ascontiguousarray(ranked_probs, dtype=np.float64)
        self.E = self.ranked.size
        self.cdf = np.empty(self.E, np.float64)
        orc_lib().orc_build_cdf(self.ranked.ctypes.data, C.c_uint64(self.E), self.cdf.ctypes.data)
        self.r2i = None if rank_to_id is None else np.ascontiguousarray(rank_to_id, dtype=np.uint32)

    def sample(self, seed, start, count):
        out = np.empty(count, np.uint32)
        orc_lib().orc_sample(self.cdf.ctypes.data, None if self.r2i is None else self.r2i.ctypes.data,
                             C.c_uint64(self.E), C.c_uint64(seed), C.c_uint64(start),
                             C.c_uint64(count), out.ctypes.data)
        return out


def substream_seed(master, index):
    return int(orc_lib().orc_substream_seed(master, index))


def count_segments(ids, seg_off, masks=None):
    ids = np.ascontiguousarray(ids, dtype=np.uint32)
    off = np.ascontiguousarray(seg_off, dtype=np.uint64)
    n = off.size - 1
    ptrs = None
    if masks is not None:
        masks = [None if m is None else np.ascontiguousarray(m, dtype=np.uint8) for m in masks]
        ptrs = (C.c_void_p * n)(*[None if m is None else m.ctypes.data for m in masks])
    a = np.zeros(n, np.int64)
    nc = np.zeros(n, np.int64)
    orc_lib().orc_count_segments(ids.ctypes.data, off.ctypes.data, C.c_uint64(n), ptrs,
                                 a.ctypes.data, nc.ctypes.data)
    return a, nc


def dedup(ids):
    ids = np.ascontiguousarray(ids, dtype=np.uint32)
    uniq = np.empty(ids.size, np.uint32)
    inv = np.empty(ids.size, np.uint32)
    U = orc_lib().orc_dedup(ids.ctypes.data, C.c_uint64(ids.size), uniq.ctypes.data, inv.ctypes.data)
    return uniq[:U].copy(), inv


def partition(unique, slot):
    unique = np.ascontiguousarray(unique, dtype=np.uint32)
    slot = np.ascontiguousarray(slot, dtype=np.int32)
    hit = np.empty(unique.size, np.uint8)
    miss = orc_lib().orc_partition(unique.ctypes.data, C.c_uint64(unique.size), slot.ctypes.data,
                                   hit.ctypes.data)
    return hit, int(miss)


def gather(table, unique):
    table = np.ascontiguousarray(table, dtype=np.float32)
    unique = np.ascontiguousarray(unique, dtype=np.uint32)
    D = table.shape[1]
    out = np.empty((unique.size, D), np.float32)
    orc_lib().orc_gather(table.ctypes.data, C.c_uint64(D), unique.ctypes.data,
                         C.c_uint64(unique.size), out.ctypes.data)
    return out


def pool(urows, inverse, bag_off):
    urows = np.ascontiguousarray(urows, dtype=np.float32)
    inverse = np.ascontiguousarray(inverse, dtype=np.uint32)
    bag_off = np.ascontiguousarray(bag_off, dtype=np.int64)
    D = urows.shape[1]
    nb = bag_off.size - 1
    o32 = np.empty((nb, D), np.float32)
    o64 = np.empty((nb, D), np.float64)
    orc_lib().orc_pool(urows.ctypes.data, C.c_uint64(D), inverse.ctypes.data, bag_off.ctypes.data,
                       C.c_uint64(nb), o32.ctypes.data, C.c_uint64(D), o64.ctypes.data)
    return o32, o64


def backward_sgd(grad, inverse, bag_off, rows_in, lr):
    grad = np.ascontiguousarray(grad, dtype=np.float32)
    inverse = np.ascontiguousarray(inverse, dtype=np.uint32)
    bag_off = np.ascontiguousarray(bag_off, dtype=np.int64)
    rows_in = np.ascontiguousarray(rows_in, dtype=np.float32)
    U, D = rows_in.shape
    ug = np.empty((U, D), np.float64)
    out = np.empty((U, D), np.float32)
    orc_lib().orc_backward_sgd(grad.ctypes.data, C.c_uint64(grad.shape[1]), C.c_uint64(D),
                               inverse.ctypes.data, bag_off.ctypes.data, C.c_uint64(bag_off.size - 1),
                               C.c_uint64(U), rows_in.ctypes.data, C.c_float(lr), ug.ctypes.data,
                               out.ctypes.data)
    return ug, out


@dataclass
class _Stat:
    n: int = 0
    s: float = 0.0
    sq: float = 0.0

    def add(self, x):
        self.n += 1
        self.s += x
        self.sq += x * x

    def finish(self):
        if self.n == 0:
            return 0.0, 0.0
        n = float(self.n)
        mean = self.s / n
        se = 0.0
        if self.n > 1:
            var = max(0.0, (self.sq - n * mean * mean) / (n - 1.0))
            se = (var / n) ** 0.5
        return mean, se


def simulate_epoch(sampler: Sampler, q, b, d, cache_mask, epochs, seed):
    """Restated simulate_epoch(dist, …) (simulator.cpp:169-220): the per-epoch
    stream, sample-major batches, per-column counts, fixed-order stats."""
    all_s, nc_s = _Stat(), _Stat()
    emb_total = 0.0
    hot = total = 0
    for e in range(epochs):
        s_e = substream_seed(seed, e)
        ids = sampler.sample(s_e, 0, q * d)
        pos = 0
        remaining = q
        while remaining > 0:
            bi = min(b, remaining)
            remaining -= bi
            batch = ids[pos: pos + bi * d].reshape(bi, d)
            pos += bi * d
            cols = np.ascontiguousarray(batch.T).ravel()
            off = np.arange(d + 1, dtype=np.uint64) * bi
            a, nc = count_segments(cols, off, [cache_mask] * d if cache_mask is not None else None)
            if bi == b:
                for f in range(d):
                    all_s.add(float(a[f]))
                    nc_s.add(float(nc[f]))
            emb_total += float(nc.sum())
            hot += int(nc.sum() == 0)
            total += 1
    um, use = all_s.finish()
    nm, nse = nc_s.finish()
    emb = emb_total / float(epochs)
    return {"unique_mean": um, "unique_se": use, "nc_mean": nm, "nc_se": nse,
            "index_cost": float(q), "embedding_cost": emb, "total": float(q) + emb,
            "hot_batch_fraction": hot / total}


def synthetic_rows(seed: int, scale: float, table: int, ids, dim: int) -> np.ndarray:
    """Restated synthetic row init (include/embcomm_gpu.h, ec_tables_init_synthetic):
    the expected table contents the parity tests compare against."""
    ids = np.asarray(ids, dtype=np.uint64)
    c = np.arange(dim, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = (np.uint64(seed) + np.uint64(0x9E3779B97F4A7C15)
             * ((np.uint64(table) << np.uint64(40)) ^ (ids[:, None] * np.uint64(dim) + c[None, :])))
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        x = x ^ (x >> np.uint64(31))
    f = (x >> np.uint64(40)).astype(np.float32) * np.float32(2.0 ** -24)
    return np.float32(scale) * (np.float32(2.0) * f - np.float32(1.0))
