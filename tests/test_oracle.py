"""Pin the CPU oracle (oracle/embcomm_oracle.c) before trusting it.

* against the committed golden vectors (produced by the compiled reference,
  tests/golden/make_golden.py) — runs anywhere;
* against the compiled reference itself (oracle/_ref) on randomized inputs
  when that library is present.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_vectors.json")))


def _sampler(kind, size, shape):
    return O.Sampler(*_ranked(kind, size, shape))


def _ranked(kind, size, shape):
    """Parametric probabilities restated (distribution_spec.cpp:19-57) with
    libm through Python's math module (numpy's SIMD exp may differ by an
    ulp); the ranking is the identity for parametric kinds."""
    import math
    if kind == "zipf":
        w = [math.pow(float(i + 1), -shape) for i in range(size)]
    elif kind == "exponential":
        w = [math.exp(-shape * float(i + 1) / size) for i in range(size)]
    else:
        den = 2.0 * shape * shape
        w = [math.exp(-((float(i + 1) / size) ** 2) / den) for i in range(size)]
    s = c = 0.0  # Kahan sum (accumulate.hpp:10-20), then normalise
    for v in w:
        y = v - c
        t = s + y
        c = (t - s) - y
        s = t
    return np.array([v / s for v in w]), None


def test_sampler_matches_reference_golden_streams():
    for case in GOLD["sample_batch"]:
        if "probs" in case:
            p = np.array(case["probs"])
            order = sorted(range(p.size), key=lambda i: (-p[i], i))
            s = O.Sampler(p[order], np.array(order, dtype=np.uint32))
        else:
            s = _sampler(case["kind"], case["size"], case["shape"])
        got = s.sample(case["seed"], 0, case["b"] * case["d"])
        assert got.tolist() == case["ids"], case.get("kind", "empirical")


def test_zipf_1m_stream_digest():
    g = GOLD["zipf1m_stream"]
    s = _sampler("zipf", g["size"], g["shape"])
    ids = s.sample(g["rng_seed"], 0, g["b"] * g["d"])
    assert ids[:64].tolist() == g["head"]
    assert hashlib.sha256(ids.tobytes()).hexdigest() == g["sha256"]


def test_substream_seed_matches_rng_hpp():
    # rng.hpp:33-38 restated in C vs. the value the golden generator used
    assert O.substream_seed(20241101, 0) == GOLD["zipf1m_stream"]["rng_seed"]


def test_simulate_epoch_restatement_matches_reference_golden():
    for c in GOLD["simulate_epoch"]:
        s = _sampler(c["kind"], c["size"], c["shape"])
        mask = np.zeros(c["size"], np.uint8)
        mask[: c["k"]] = 1  # parametric: top-k ids are 0..k-1
        got = O.simulate_epoch(s, c["q"], c["b"], c["d"], mask if c["k"] else None, c["epochs"], c["seed"])
        for key, v in c["result"].items():
            assert got[key] == v, (c, key)


def test_m1_counts_match_reference_golden():
    """Per-(table, batch) distinct / non-cached counts at config-1 shape
    (SURVEY §8c protocol) — the quantities the GPU dedup must reproduce."""
    s = _sampler("zipf", 1_000_000, 1.05)
    for c in GOLD["m1_counts"]:
        ids = s.sample(c["rng_seed"], 0, 4096 * 20)
        assert hashlib.sha256(ids.tobytes()).hexdigest() == c["sha256"]
        mask = np.zeros(1_000_000, np.uint8)
        mask[: c["k"]] = 1
        a, nc = O.count_segments(ids, [0, ids.size], [mask])
        assert (int(a[0]), int(nc[0])) == (c["unique"], c["non_cached"])


def test_trace_kat_counts():
    """tests/test_simulator.cpp:156-172: one hot batch (samples 0,2) and one
    normal batch (samples 1,3); embedding units 3."""
    ids = np.array(GOLD["trace_kat"]["ids"], np.uint32).reshape(4, 2)
    normal = ids[[1, 3]]  # columns {0,3} and {2,3}
    cols = np.ascontiguousarray(normal.T).ravel()
    mask = np.array([1, 1, 0, 0], np.uint8)
    a, nc = O.count_segments(cols, [0, 2, 4], [mask, mask])
    assert int(nc.sum()) == GOLD["trace_kat"]["result"]["embedding_cost"] == 3.0


def test_dedup_restatement_properties():
    rng = np.random.default_rng(0)
    for n, E in [(0, 5), (1, 1), (100, 3), (5000, 100000), (81920, 1000)]:
        ids = rng.integers(0, E, n, dtype=np.uint32)
        u, inv = O.dedup(ids)
        assert len(set(u.tolist())) == u.size == len(set(ids.tolist()))
        assert (u[inv[:n]] == ids).all()
        # first-occurrence order: the k-th unique is the k-th new id in scan order
        seen, order = set(), []
        for x in ids.tolist():
            if x not in seen:
                seen.add(x)
                order.append(x)
        assert u.tolist() == order
        a, nc = O.count_segments(ids, [0, n])
        assert int(a[0]) == u.size


def test_pool_and_backward_restatement():
    rng = np.random.default_rng(1)
    D, B, P, E = 8, 16, 5, 40
    table = rng.standard_normal((E, D)).astype(np.float32)
    ids = rng.integers(0, E, B * P, dtype=np.uint32)
    u, inv = O.dedup(ids)
    rows = O.gather(table, u)
    assert (rows == table[u]).all()
    off = np.arange(B + 1, dtype=np.int64) * P
    o32, o64 = O.pool(rows, inv, off)
    np.testing.assert_allclose(o64, table[ids].reshape(B, P, D).sum(1, dtype=np.float64), rtol=1e-12)
    g = rng.standard_normal((B, D)).astype(np.float32)
    ug, new = O.backward_sgd(g, inv, off, rows, 0.1)
    want = np.zeros((u.size, D))
    for i, x in enumerate(inv):
        want[x] += g[i // P]
    np.testing.assert_allclose(ug, want, rtol=1e-12)
    np.testing.assert_allclose(new, rows - 0.1 * want, rtol=1e-6)


# ------------------------------------------------ against the live reference
def test_sampler_vs_reference_randomized(ref):
    rng = np.random.default_rng(11)
    for _ in range(10):
        E = int(rng.integers(1, 3000))
        p = rng.random(E) ** 3
        p /= p.sum()
        d = ref.RefDist.from_probs(p)
        rp, r2i = d.export()
        s = O.Sampler(rp, r2i)
        seed = int(rng.integers(0, 2**63))
        assert (s.sample(seed, 0, 999) == ref.ref_sample_batch(d, 333, 3, seed)).all()


def test_counts_vs_reference_randomized(ref):
    rng = np.random.default_rng(12)
    for _ in range(10):
        E = int(rng.integers(1, 5000))
        n = int(rng.integers(1, 20000))
        ids = rng.integers(0, E, n, dtype=np.uint32)
        k = int(rng.integers(0, E + 1))
        cache = rng.permutation(E)[:k].astype(np.uint32)
        mask = np.zeros(E, np.uint8)
        mask[cache] = 1
        a, nc = O.count_segments(ids, [0, n], [mask])
        ra, rnc = ref.ref_segment_counts(ids, [0, n], [E], [cache])
        assert (a[0], nc[0]) == (ra[0], rnc[0])


def test_measure_unique_restated_vs_reference(ref):
    """test_simulator.cpp:66-85: manual substream replay equals the mean."""
    d = ref.RefDist.parametric("zipf", 32, 1.0)
    s = O.Sampler(*d.export())
    total = 0
    for t in range(4):
        ids = s.sample(O.substream_seed(1234, t), 0, 16)
        total += len(set(ids.tolist()))
    assert ref.ref_measure_unique(d, 16, 4, 1234)["unique_mean"] == total / 4.0
