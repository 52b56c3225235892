"""Host half of the C-ABI (distributions, cost model, planner) against the
reference: known answers from the reference's own tests, the committed golden
vectors, and — where oracle/_ref is present — the live reference on
randomized inputs.  Every comparison is bit-exact (==) unless the reference
test itself uses a tolerance."""
import json
import os
import re

import numpy as np
import pytest

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_vectors.json")))


def test_library_exports_every_header_symbol(ec):
    """include/embcomm_gpu.h declares exactly what the library exports."""
    import ctypes
    hdr = open(os.path.join(os.path.dirname(__file__), "..", "include", "embcomm_gpu.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    names = set(re.findall(r"\b(ec_[a-z0-9_]+)\s*\(", hdr))
    assert len(names) > 50
    lib = ctypes.CDLL(ec._native.LIB_PATH)
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing
    assert set(ec._native.exported_symbols()) <= names


def test_error_model(ec):
    with pytest.raises(ec.ValidationError):
        ec.EmbeddingDistribution.from_probabilities([])
    with pytest.raises(ec.ValidationError):
        ec.EmbeddingDistribution.from_probabilities([0.5, 0.6])
    with pytest.raises(ec.ValidationError):
        ec.EmbeddingDistribution.from_probabilities([0.5, 0.4999])
    ec.EmbeddingDistribution.from_probabilities([0.5, 0.5 + 0.9e-9])
    with pytest.raises(ec.ValidationError):
        ec.WorkloadSpec(10, 11, 1)
    with pytest.raises(ec.ValidationError):
        ec.batch_presence_prob(1.1, 1)
    with pytest.raises(ec.ValidationError):
        ec.DeviceModel(5, 10, 1)


def test_distribution_kats(ec):
    """tests/test_distribution.cpp:20-47."""
    d = ec.EmbeddingDistribution.from_probabilities([0.2, 0.4, 0.2, 0.2])
    assert [d.id_at_rank(r) for r in range(4)] == [1, 0, 2, 3]
    assert d.rank_of(1) == 0 and d.prob(1) == 0.4
    assert d.top_ids(2).tolist() == [1, 0]
    z = ec.EmbeddingDistribution.from_probabilities([0.0, 1.0, 0.0])
    assert [z.id_at_rank(r) for r in range(3)] == [1, 0, 2]
    u = ec.EmbeddingDistribution.uniform(4)
    assert u.prob(3) == 0.25 and abs(u.mass_of([0, 2]) - 0.5) < 1e-12
    with pytest.raises(ec.ValidationError):
        u.prob(4)
    with pytest.raises(ec.ValidationError):
        u.top_ids(5)
    # tests/test_distribution_spec.cpp: zipf(2, 1) -> (2/3, 1/3)
    z2 = ec.materialize(ec.DistributionSpec.parametric(ec.DistributionKind.zipf, 2, 1.0))
    assert abs(z2.prob(0) - 2 / 3) < 1e-15 and abs(z2.prob(1) - 1 / 3) < 1e-15


def test_cost_model_kats(ec):
    """tests/test_cost_model.cpp:53-197."""
    assert ec.batch_presence_prob(0.0, 100) == 0.0
    assert ec.batch_presence_prob(1.0, 1) == 1.0
    assert abs(ec.batch_presence_prob(0.5, 2) - 0.75) < 1e-12
    assert abs(ec.batch_presence_prob(1e-15, 1000) - 1e-12) < 1e-18
    u4 = ec.EmbeddingDistribution.uniform(4)
    assert abs(ec.expected_unique_per_batch(u4, 2) - 1.75) < 1e-12
    assert ec.coalesced_batch_cost(ec.EmbeddingDistribution.uniform(1), 10).total == 11.0
    assert ec.baseline_epoch_cost(ec.WorkloadSpec(5000, 256, 26)) == 130000.0
    c = ec.coalesced_epoch_cost(ec.EmbeddingDistribution.uniform(2), ec.WorkloadSpec(100, 10, 1))
    assert abs(c.total - 119.98046875) < 1e-9
    spec = ec.WorkloadSpec(40, 4, 1)
    assert ec.cached_epoch_cost(u4, spec, [0, 1, 2, 3]).total == 40.0
    assert abs(ec.cached_epoch_cost(u4, spec, [0]).total - 60.5078125) < 1e-9
    with pytest.raises(ec.ValidationError):
        ec.cached_epoch_cost(u4, spec, [4])


def test_cost_model_golden(ec):
    g = GOLD["cost_model"]
    for p, b, v in g["presence"]:
        assert ec.batch_presence_prob(p, b) == v
    dz = ec.materialize(ec.DistributionSpec.parametric(ec.DistributionKind.zipf, 1_000_000, 1.05))
    assert ec.expected_unique_per_batch(dz, 81920) == g["expected_unique_zipf1m_81920"]
    c = ec.cached_epoch_cost(dz, ec.WorkloadSpec(4096 * 100, 4096, 20), dz.top_ids(10000))
    assert [c.index_cost, c.embedding_cost, c.total] == g["cached_zipf1m_k10000"]


def test_planner_golden(ec):
    """tests/test_cache_planner.cpp:153-163 golden + a larger reference run."""
    g = GOLD["cost_model"]["planner_zipf32"]
    z32 = ec.materialize(ec.DistributionSpec.parametric(ec.DistributionKind.zipf, 32, 1.0))
    p = ec.optimal_cache_size_scan(z32, ec.DeviceModel(2048, 2, 8), ec.WorkloadSpec(10000, 1, 4))
    assert (p.cache_size, p.batch_size, p.feasible) == (g["cache_size"], g["batch_size"], g["feasible"]) == (32, 896, True)
    assert p.expected_epoch_cost.total == 10000.0
    g = GOLD["cost_model"]["planner_zipf200k"]
    d = ec.materialize(ec.DistributionSpec.parametric(ec.DistributionKind.zipf, 200000, 1.05))
    p = ec.optimal_cache_size_search(d, ec.DeviceModel(8_000_000, 300, 64, 0.9), ec.WorkloadSpec(1_000_000, 1, 26))
    assert (p.cache_size, p.batch_size, p.used_scan_fallback) == (g["cache_size"], g["batch_size"],
                                                                   g["used_scan_fallback"])
    assert [p.expected_epoch_cost.index_cost, p.expected_epoch_cost.embedding_cost,
            p.expected_epoch_cost.total] == g["cost"]


def test_max_batch_size_kats(ec):
    """tests/test_cache_planner.cpp:49-71."""
    dm = ec.DeviceModel(1000, 10, 5)
    assert ec.max_batch_size(dm, 0) == 100
    assert ec.max_batch_size(dm, 198) == 1
    assert ec.max_batch_size(dm, 199) is None
    assert ec.max_batch_size(ec.DeviceModel(1000, 10, 5, 0.5), 12) == 44


def test_place_topk_global(ec):
    a = ec.EmbeddingDistribution.from_probabilities([0.5, 0.3, 0.2])
    b = ec.EmbeddingDistribution.from_probabilities([0.4, 0.4, 0.2])
    assert ec.place_topk_global([a, b], 3) == [1, 2]
    assert ec.place_topk_global([a, b], 4) == [2, 2]
    assert ec.place_topk_global([a, b], 100) == [3, 3]


# ------------------------------------------------ against the live reference
def _pair(ref, ec, probs):
    return ref.RefDist.from_probs(probs), ec.EmbeddingDistribution.from_probabilities(probs)


def test_distribution_and_costs_vs_reference_randomized(ref, ec):
    rng = np.random.default_rng(5)
    for i in range(25):
        E = int(rng.integers(1, 400))
        p = rng.random(E)
        if i % 3 == 0:
            p = np.round(p * 4)  # ties
            p[0] += 1
        p /= p.sum()
        r, m = _pair(ref, ec, p)
        rp, r2i = r.export()
        assert (m.ranked_probs() == rp).all() and (m.rank_to_id() == r2i).all()
        b = int(rng.integers(1, 5000))
        assert ec.expected_unique_per_batch(m, b) == ref.ref_cost("expected_unique_from_rank", r, b, 0)
        k = int(rng.integers(0, E + 1))
        assert ec.expected_unique_from_rank(m, b, k) == ref.ref_cost("expected_unique_from_rank", r, b, k)
        q = b * int(rng.integers(1, 50)) + int(rng.integers(0, b))
        d = int(rng.integers(1, 27))
        cache = rng.permutation(E)[:k]
        c = ec.cached_epoch_cost(m, ec.WorkloadSpec(q, b, d), cache)
        assert (c.index_cost, c.embedding_cost, c.total) == ref.ref_cost("cached_epoch_cost", r, q, b, d, cache)
        c = ec.coalesced_epoch_cost(m, ec.WorkloadSpec(q, b, d))
        assert (c.index_cost, c.embedding_cost, c.total) == ref.ref_cost("coalesced_epoch_cost", r, q, b, d)
        assert ec.memory_io_proxy(m, ec.WorkloadSpec(q, b, d), cache) == ref.ref_cost(
            "memory_io_proxy", r, q, b, d, cache)


def test_parametric_materialize_vs_reference(ref, ec):
    for kind, name, size, shape in [(ec.DistributionKind.zipf, "zipf", 100000, 1.05),
                                    (ec.DistributionKind.exponential, "exponential", 5000, 100.0),
                                    (ec.DistributionKind.half_normal, "half_normal", 7000, 0.05),
                                    (ec.DistributionKind.zipf, "zipf", 1000, 2.5)]:
        m = ec.materialize(ec.DistributionSpec.parametric(kind, size, shape))
        r = ref.RefDist.parametric(name, size, shape)
        assert (m.ranked_probs() == r.export()[0]).all()
        me = ec.materialize_extended(ec.DistributionSpec.parametric(kind, size, shape), 5)
        re_ = ref.RefDist.extended(name, size, shape, 5)
        assert (me.ranked_probs() == re_.export()[0]).all()


def test_planner_vs_reference_randomized(ref, ec):
    """Mirrors tests/test_cache_planner.cpp 'search matches scan' over random
    instances, but compares against the reference's own answers."""
    rng = np.random.default_rng(41)
    for i in range(40):
        E = int(rng.integers(2, 65))
        p = rng.random(E) + 0.01
        p /= p.sum()
        r, m = _pair(ref, ec, p)
        a = int(rng.integers(1, 7))
        de = int(rng.integers(1, 41))
        M = a + int(rng.integers(0, 5000))
        q = 1000 + int(rng.integers(0, 20000))
        d = int(rng.integers(1, 9))
        eff = 1.0 if i % 2 else float(rng.uniform(0.3, 1.0))
        for search in (False, True):
            fn = ec.optimal_cache_size_search if search else ec.optimal_cache_size_scan
            if M < a:
                continue
            mine = fn(m, ec.DeviceModel(M, a, de, eff), ec.WorkloadSpec(q, 1, d))
            theirs = ref.ref_plan(r, M, a, de, eff, q, d, search=search)
            assert mine.feasible == theirs["feasible"]
            if not mine.feasible:
                continue
            assert (mine.cache_size, mine.batch_size, mine.used_scan_fallback) == (
                theirs["cache_size"], theirs["batch_size"], theirs["used_scan_fallback"])
            assert (mine.expected_epoch_cost.index_cost, mine.expected_epoch_cost.embedding_cost,
                    mine.expected_epoch_cost.total) == tuple(theirs["cost"])
            assert (mine.cached_ids == theirs["cached_ids"]).all()
        for k in range(0, min(E - 1, 5)):
            if ec.max_batch_size(ec.DeviceModel(M, a, de, eff), k + 1) is None:
                break
            mm = ec.delta_comm(m, ec.DeviceModel(M, a, de, eff), q, k)
            rr = ref.ref_delta_comm(r, M, a, de, eff, q, k)
            assert (mm.candidate_id, mm.presence_gain, mm.threshold, mm.delta_comm, mm.recommend) == (
                rr["candidate_id"], rr["presence_gain"], rr["threshold"], rr["delta_comm"], rr["recommend"])


def test_estimate_distribution_vs_reference(ref, ec):
    """estimate_distribution (trace.cpp:161-183) on the reference's own skew
    table: identical ranked probabilities and rank -> id map."""
    rng = np.random.default_rng(8)
    for smoothing in (0.0, 0.5, 2.0):
        E = int(rng.integers(2, 3000))
        ids = rng.zipf(1.3, 5000).astype(np.uint32) % E
        oid, cnt, cum = ref.ref_build_skew_table(ids, 1, E)
        table = ec.SkewTable(oid, cnt, cum, ids.size)
        mine = ec.estimate_distribution(table, E, smoothing)
        theirs = ref.ref_estimate_distribution(ids, 1, E, smoothing)
        rp, r2i = theirs.export()
        assert (mine.ranked_probs() == rp).all() and (mine.rank_to_id() == r2i).all()
    with pytest.raises(ec.ValidationError):
        ec.estimate_distribution(ec.SkewTable(np.zeros(0, np.uint32), np.zeros(0, np.uint64),
                                              np.zeros(0), 0), 10, 0.0)
