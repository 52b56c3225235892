"""Hot/normal scheduling on the GPU: per-sample hot flags
and the stable hot-first order equal the reference's classify_samples /
build_schedule on single-table data and a numpy restatement on multi-table
data; hot batches touch no uncached row."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch
    return torch


def test_single_table_matches_reference_schedule(ec, torch, ref):
    E, q, b = 500, 3000, 128
    d = ec.materialize(ec.DistributionSpec.parametric(ec.DistributionKind.zipf, E, 1.1))
    ids = ec.sample_batch(d, q, 1, ec.SplitMix64(77))
    cache = d.top_ids(40)
    tab = ec.EmbeddingTables([E], 8, max_lookups_per_table=b, max_batch_size=b)
    tab.init_synthetic(1, 1.0)
    tab.place_cache([cache])
    order, nh = tab.schedule(torch.from_numpy(ids.view(np.int32)).cuda())
    ref_order, _, _ = ref.ref_build_schedule(ids, 1, E, cache, b)
    hot = ref.ref_classify_samples(ids, 1, E, cache)
    assert nh == int(hot.sum())
    assert (order.cpu().numpy().view(np.uint32) == ref_order).all()
    tab.close()


def test_multi_table_hot_batches_have_no_misses(ec, torch):
    rows, B = [1000, 50, 20000, 7], 256
    T = len(rows)
    dists = [ec.materialize(ec.DistributionSpec.parametric(ec.DistributionKind.zipf, r, 1.2)) for r in rows]
    caches = [d.top_ids(k) for d, k in zip(dists, [200, 50, 2000, 7])]
    q = 16 * B
    ids = np.stack([ec.sample_batch(d, q, 1, ec.SplitMix64(10 + t)) for t, d in enumerate(dists)], 1)
    sample_ids = torch.from_numpy(np.ascontiguousarray(ids).view(np.int32)).cuda()
    tab = ec.EmbeddingTables(rows, 8, max_lookups_per_table=B, max_batch_size=B)
    tab.init_synthetic(2, 1.0)
    tab.place_cache(caches)
    order, nh = tab.schedule(sample_ids)
    cached = [np.isin(np.arange(r), c) for r, c in zip(rows, caches)]
    hot = np.all([cached[t][ids[:, t]] for t in range(T)], axis=0)
    want = np.concatenate([np.where(hot)[0], np.where(~hot)[0]])
    assert nh == int(hot.sum()) and (order.cpu().numpy() == want).all()
    offs = np.arange(T + 1) * B
    for first in range(0, q, B):
        batch = tab.gather_batch(sample_ids, order, first, B)
        sel = want[first:first + B]
        assert (batch.cpu().numpy().reshape(T, B) == ids[sel].T).all()
        tab.forward(batch, offs, B, 1)
        st = tab.stats()
        if first + B <= nh:
            assert st["miss_rows"] == 0  # a hot batch never reaches the cold tier
    tab.close()


@pytest.mark.parametrize("seed", [None, 0, 1, 20241101, (1 << 62) + 7])
@pytest.mark.parametrize("d_feat,q", [(1, 1), (3, 5000), (2, 777)])
def test_build_schedule_shuffle_matches_reference(ec, ref, seed, d_feat, q):
    """build_schedule(trace, cache, b, shuffle_seed) (trace.cpp:206-240): the
    GPU partition plus the seeded per-class Fisher-Yates equal the reference's
    schedule batch for batch (order and batch sizes), including a one-sample
    trace and classes of one sample."""
    E, b = 400, 64
    dist = ec.materialize(ec.DistributionSpec.parametric(ec.DistributionKind.zipf, E, 1.05))
    ids = ec.sample_batch(dist, q, d_feat, ec.SplitMix64(99 + q))
    tr = ec.Trace(d_feat, E, ids)
    cache = dist.top_ids(30)
    s = ec.build_schedule(tr, cache, b, shuffle_seed=seed)
    ref_order, ref_sizes, ref_nh = ref.ref_build_schedule(ids, d_feat, E, cache, b,
                                                          shuffle_seed=-1 if seed is None else seed)
    flat = [x for bt in s.hot_batches + s.normal_batches for x in bt]
    assert flat == ref_order.tolist()
    assert [len(bt) for bt in s.hot_batches + s.normal_batches] == ref_sizes.tolist()
    assert len(s.hot_batches) == ref_nh  # (the shim reports hot batches)
