"""GPU planner sweeps vs the bit-exact host planner and
the compiled reference: 1e-12 relative (device reduction order differs)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_expected_unique_many_matches_host(ec, ref):
    d = ec.materialize(ec.DistributionSpec.parametric(ec.DistributionKind.zipf, 1_000_000, 1.05))
    r = ref.RefDist.parametric("zipf", 1_000_000, 1.05)
    bs = np.array([1, 2, 100, 4096, 81920, 10_000_000], np.int64)
    ks = np.array([0, 5, 1000, 0, 10_000, 999_999], np.uint64)
    got = ec.expected_unique_many(d, bs, ks)
    for b, k, g in zip(bs, ks, got):
        want = ref.ref_cost("expected_unique_from_rank", r, int(b), int(k))
        assert abs(g - want) <= 1e-12 * max(1.0, abs(want)), (b, k, g, want)
    assert ec.expected_unique_many(d, [81920])[0] == pytest.approx(ec.expected_unique_per_batch(d, 81920), rel=1e-12)


def test_cost_curve_matches_scan_and_finds_its_minimum(ec, ref):
    E = 20_000
    d = ec.materialize(ec.DistributionSpec.parametric(ec.DistributionKind.zipf, E, 0.9))
    r = ref.RefDist.parametric("zipf", E, 0.9)
    dm = ec.DeviceModel(400_000, 40, 16)
    Q, dd = 1_000_000, 8
    ks = np.arange(0, E + 1, dtype=np.int64)
    costs, bs = ec.cost_curve(d, dm, Q, dd, ks)
    feas = bs > 0
    plan = ec.optimal_cache_size_scan(d, dm, ec.WorkloadSpec(Q, 1, dd))
    theirs = ref.ref_plan(r, 400_000, 40, 16, 1.0, Q, dd, search=False)
    assert plan.cache_size == theirs["cache_size"]
    for k in [0, 1, 17, plan.cache_size, int(ks[feas][-1])]:
        b = ec.max_batch_size(dm, k)
        assert bs[k] == min(b, Q)
        want = ec.WorkloadSpec(Q, int(bs[k]), dd)
        host = ec.cached_epoch_cost(d, want, d.top_ids(k))
        assert costs[k].total == pytest.approx(host.total, rel=1e-12)
    totals = np.array([c.total if f else np.inf for c, f in zip(costs, feas)])
    best = int(np.argmin(totals))
    # the GPU curve's minimum is the scan's plan (or ties it within 1e-12)
    assert totals[best] == pytest.approx(plan.expected_epoch_cost.total, rel=1e-12)
    infeasible = np.where(~feas)[0]
    if infeasible.size:
        assert np.isnan(costs[infeasible[0]].total)
