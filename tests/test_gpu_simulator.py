"""GPU sampler (K0) and Monte Carlo simulator vs the reference: bit-exact ids
and bit-exact SimResult fields (reference goldens + the live compiled
reference, which travels to the GPU box as oracle/_ref)."""
import hashlib
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_vectors.json")))
KIND = {"zipf": 0, "exponential": 1, "half_normal": 2}


def _dist(ec, kind, size, shape):
    return ec.materialize(ec.DistributionSpec.parametric(ec.DistributionKind(KIND[kind]), size, shape))


def _check_sim(got, want):
    assert got.unique_per_batch.mean == want["unique_mean"]
    assert got.unique_per_batch.std_error == want["unique_se"]
    assert got.non_cached_unique.mean == want["nc_mean"]
    assert got.non_cached_unique.std_error == want["nc_se"]
    assert got.measured_epoch_cost.index_cost == want["index_cost"]
    assert got.measured_epoch_cost.embedding_cost == want["embedding_cost"]
    assert got.measured_epoch_cost.total == want["total"]
    assert got.hot_batch_fraction == want["hot_batch_fraction"]


def test_sample_batch_bit_exact(ec):
    for c in GOLD["sample_batch"]:
        if "probs" in c:
            d = ec.EmbeddingDistribution.from_probabilities(c["probs"])
        else:
            d = _dist(ec, c["kind"], c["size"], c["shape"])
        rng = ec.SplitMix64(c["seed"])
        got = ec.sample_batch(d, c["b"], c["d"], rng)
        assert got.tolist() == c["ids"]
        # the generator advanced exactly b*d steps (rng.hpp:17)
        r2 = ec.SplitMix64(c["seed"])
        for _ in range(c["b"] * c["d"]):
            r2.next()
        assert rng.state == r2.state


def test_zipf_1m_stream_digest(ec):
    g = GOLD["zipf1m_stream"]
    d = _dist(ec, "zipf", g["size"], g["shape"])
    ids = ec.sample_batch(d, g["b"], g["d"], ec.SplitMix64(g["rng_seed"]))
    assert hashlib.sha256(ids.tobytes()).hexdigest() == g["sha256"]


def test_sample_batch_point_mass_and_errors(ec):
    d = ec.EmbeddingDistribution.uniform(1)
    assert ec.sample_batch(d, 3, 2, ec.SplitMix64(1)).tolist() == [0] * 6
    with pytest.raises(ec.ValidationError):
        ec.sample_batch(d, 0, 2, ec.SplitMix64(1))


def test_measure_unique_bit_exact(ec):
    for c in GOLD["measure_unique"]:
        got = ec.measure_unique(_dist(ec, c["kind"], c["size"], c["shape"]), c["b"], c["trials"], c["seed"])
        w = c["result"]
        assert got.unique_per_batch.mean == w["unique_mean"]
        assert got.unique_per_batch.std_error == w["unique_se"]
        assert got.non_cached_unique.mean == w["nc_mean"]


def test_simulate_epoch_bit_exact_golden(ec):
    for c in GOLD["simulate_epoch"]:
        d = _dist(ec, c["kind"], c["size"], c["shape"])
        got = ec.simulate_epoch(d, ec.WorkloadSpec(c["q"], c["b"], c["d"]), d.top_ids(c["k"]), c["epochs"], c["seed"])
        _check_sim(got, c["result"])


def test_simulate_epoch_vs_live_reference(ec, ref):
    rng = np.random.default_rng(99)
    for i in range(12):
        E = int(rng.integers(1, 50000))
        if i % 3 == 0:
            p = rng.random(E) ** 4
            p /= p.sum()
            d = ec.EmbeddingDistribution.from_probabilities(p)
            r = ref.RefDist.from_probs(p)
        else:
            shape = float(rng.uniform(0.5, 1.5))
            d = _dist(ec, "zipf", E, shape)
            r = ref.RefDist.parametric("zipf", E, shape)
        b = int(rng.integers(1, 3000))
        q = b * int(rng.integers(1, 20)) + int(rng.integers(0, b))
        dd = int(rng.integers(1, 6))
        k = int(rng.integers(0, E + 1)) if i % 2 else 0
        cache = rng.permutation(E)[:k].astype(np.uint32)
        seed = int(rng.integers(0, 2**63))
        got = ec.simulate_epoch(d, ec.WorkloadSpec(q, b, dd), cache, 2, seed)
        _check_sim(got, ref.ref_simulate_epoch(r, q, b, dd, cache, 2, seed))


def test_simulate_epoch_edges(ec):
    d = _dist(ec, "zipf", 16, 1.0)
    r = ec.simulate_epoch(d, ec.WorkloadSpec(100, 10, 2), d.top_ids(16), 3, 1)
    assert r.measured_epoch_cost.embedding_cost == 0.0 and r.measured_epoch_cost.total == 100.0
    assert r.hot_batch_fraction == 1.0
    u1 = ec.EmbeddingDistribution.uniform(1)
    r = ec.simulate_epoch(u1, ec.WorkloadSpec(100, 10, 1), [], 1, 1)
    assert r.measured_epoch_cost.total == 110.0 and r.unique_per_batch.mean == 1.0
    u8 = ec.EmbeddingDistribution.uniform(8)
    assert ec.simulate_epoch(u8, ec.WorkloadSpec(1000, 4, 2), [], 2, 4).unique_per_batch.mean <= 4.0
    with pytest.raises(ec.ValidationError):
        ec.simulate_epoch(u8, ec.WorkloadSpec(10, 5, 1), [8], 1, 1)


def test_simulate_trace_kat_and_golden(ec):
    k = GOLD["trace_kat"]
    t = ec.Trace(k["d"], k["vocab"], np.array(k["ids"], np.uint32))
    r = ec.simulate_epoch(t, k["b"], k["cache"])
    assert r.measured_epoch_cost.index_cost == 4.0
    assert r.measured_epoch_cost.embedding_cost == 3.0
    assert r.hot_batch_fraction == 0.5
    _check_sim(r, k["result"])

    g = GOLD["trace_large"]
    d = _dist(ec, g["kind"], g["size"], g["shape"])
    ids = ec.sample_batch(d, g["b_gen"], g["d"], ec.SplitMix64(g["seed"]))
    t = ec.Trace(g["d"], g["size"], ids)
    cache = d.top_ids(g["cache_k"])
    _check_sim(ec.simulate_epoch(t, g["batch"], cache), g["result"])
    cls = ec.classify_samples(t, cache)
    hot = np.zeros(t.num_samples(), np.uint8)
    hot[cls.hot] = 1
    assert hot.tolist() == g["hot"]
    sched = ec.build_schedule(t, cache, g["batch"])
    flat = [s for bt in sched.hot_batches + sched.normal_batches for s in bt]
    assert flat == g["schedule_order"]
    assert len(sched.hot_batches) == g["n_hot_batches"]


def test_trace_validation(ec):
    t = ec.Trace(2, 3, np.array([0, 1, 0, 2], np.uint32))
    with pytest.raises(ec.ValidationError):
        ec.classify_samples(t, [3])
    bad = ec.Trace(2, 3, np.array([0, 1, 0, 7], np.uint32))
    with pytest.raises(ec.ValidationError):
        ec.simulate_epoch(bad, 2, [])
    assert ec.classify_samples(t, [0, 1, 2]).hot == [0, 1]
    assert ec.classify_samples(t, []).normal == [0, 1]
    c = ec.classify_samples(t, [0, 1])
    assert (c.hot, c.normal) == ([0], [1])


def test_skew_table_bit_exact(ec, ref):
    """build_skew_table (trace.cpp:128-150): GPU histogram + (count desc, id
    asc) order, cumulative fractions identical to the reference; placement
    from the estimated distribution equals the reference's top_ids."""
    rng = np.random.default_rng(21)
    for E, n, a in [(10, 100, 1.5), (5000, 200000, 1.2), (100000, 50000, 1.05)]:
        ids = (rng.zipf(a, n) - 1).astype(np.uint32) % E
        t = ec.Trace(1, E, ids)
        st = ec.build_skew_table(t)
        oid, cnt, cum = ref.ref_build_skew_table(ids, 1, E)
        assert (st.ids == oid).all() and (st.counts == cnt).all() and (st.cum_fraction == cum).all()
        d = ec.estimate_distribution(st, E, 0.0)
        rd = ref.ref_estimate_distribution(ids, 1, E, 0.0)
        k = min(E, 64)
        assert (d.top_ids(k) == rd.top_ids(k)).all()
    with pytest.raises(ec.ValidationError):
        ec.build_skew_table(ec.Trace(1, 4, np.array([1, 9], np.uint32)))
