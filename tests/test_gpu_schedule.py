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
