"""Cache re-placement and row writes while batches are prefetched, and cache
re-placement of row-sharded tables after training (place_cache /
write_rows / init_synthetic invalidate pending prefetches; a multi-rank
re-placement keeps trained values)."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu
RTOL = 1e-5


@pytest.fixture(scope="module")
def torch():
    import torch
    assert torch.cuda.is_available()
    return torch


def _dists(ec, rows, a=1.05):
    return [ec.materialize(ec.DistributionSpec.parametric(ec.DistributionKind.zipf, r, a)) for r in rows]


def _ids(ec, torch, dists, n, seed, rank=None):
    ids = torch.empty(len(dists) * n, dtype=torch.int32, device="cuda")
    for t, d in enumerate(dists):
        s = ec.substream_seed(seed, t) if rank is None else ec.substream_seed(ec.substream_seed(seed, rank), t)
        ec.DiscreteSampler(d).sample_into(ids.data_ptr() + 4 * n * t, s, 0, n)
    torch.cuda.synchronize()
    return ids


@pytest.mark.parametrize("storage", ["host", "hbm"])
@pytest.mark.parametrize("shrink", [True, False])
def test_prefetch_then_place_cache_then_forward(ec, torch, storage, shrink):
    """fwd(A) -> bwd(A) -> prefetch(B) -> place_cache(new) -> fwd(B): the
    prefetched set (cache slots of the old placement) is dropped and B is
    recomputed; outputs equal the run without the prefetch.  A smaller new
    cache would put stale slot numbers out of bounds."""
    rows, D, B, P = [4000, 900, 60], 8, 128, 3
    n = B * P
    dists = _dists(ec, rows)
    old = [d.top_ids(k) for d, k in zip(dists, [400, 100, 30])]
    new = [d.top_ids(k) for d, k in zip(dists, [5, 2, 1] if shrink else [800, 300, 50])]
    offs = np.arange(len(rows) + 1, dtype=np.int64) * n
    a = _ids(ec, torch, dists, n, 1)
    b = _ids(ec, torch, dists, n, 2)
    g = torch.randn(B, len(rows) * D, device="cuda", generator=torch.Generator("cuda").manual_seed(3))

    def run(prefetch):
        tab = ec.EmbeddingTables(rows, D, storage=storage, max_lookups_per_table=n, max_batch_size=B)
        tab.init_synthetic(5, 0.3)
        tab.place_cache(old)
        tab.forward(a, offs, B, P)
        if prefetch:
            tab.prefetch(b, offs, B, P)
        tab.backward(g, 0.25)
        tab.place_cache(new)
        out = tab.forward(b, offs, B, P).clone()
        torch.cuda.synchronize()
        final = [tab.read_rows(t, np.arange(rows[t])) for t in range(len(rows))]
        st = tab.stats(per_table=True)
        tab.close()
        return out.cpu().numpy(), final, st

    o1, f1, s1 = run(False)
    o2, f2, s2 = run(True)
    np.testing.assert_allclose(o2, o1, rtol=RTOL, atol=1e-5 * np.abs(o1).max())
    for x, y in zip(f1, f2):
        np.testing.assert_allclose(y, x, rtol=RTOL, atol=1e-5 * np.abs(x).max())
    assert (s1["miss_per_table"] == s2["miss_per_table"]).all()
    # hit/miss of B follow the new placement
    ids_h = b.cpu().numpy().view(np.uint32)
    for t in range(len(rows)):
        u, _ = O.dedup(ids_h[t * n:(t + 1) * n])
        assert s2["miss_per_table"][t] == int((~np.isin(u, new[t])).sum())


@pytest.mark.parametrize("storage", ["host", "hbm"])
def test_write_rows_after_prefetch(ec, torch, storage):
    """Rows written while a batch that reads them is prefetched: the forward
    sees the written values (the prefetch is dropped and recomputed)."""
    rows, D, B, P = [3000, 500], 8, 64, 2
    n = B * P
    dists = _dists(ec, rows)
    caches = [d.top_ids(k) for d, k in zip(dists, [20, 5])]
    offs = np.arange(len(rows) + 1, dtype=np.int64) * n
    a = _ids(ec, torch, dists, n, 11)
    b = _ids(ec, torch, dists, n, 12)
    tab = ec.EmbeddingTables(rows, D, storage=storage, max_lookups_per_table=n, max_batch_size=B)
    tab.init_synthetic(2, 0.5)
    tab.place_cache(caches)
    tab.forward(a, offs, B, P)
    tab.prefetch(b, offs, B, P)
    ids_h = b.cpu().numpy().view(np.uint32)
    newvals = []
    for t in range(len(rows)):
        u, _ = O.dedup(ids_h[t * n:(t + 1) * n])
        v = np.random.default_rng(t).standard_normal((u.size, D)).astype(np.float32)
        tab.write_rows(t, u, v)  # cached and cold rows alike
        newvals.append((u, v))
    out = tab.forward(b, offs, B, P).cpu().numpy()
    bag = np.arange(B + 1, dtype=np.int64) * P
    for t, (u, v) in enumerate(newvals):
        _, inv = O.dedup(ids_h[t * n:(t + 1) * n])
        _, o64 = O.pool(v, inv[:n], bag)
        np.testing.assert_allclose(out[:, t * D:(t + 1) * D], o64, rtol=RTOL, atol=1e-6)
    tab.close()


def _authoritative(members, rows, world, cached):
    out = []
    for t, r in enumerate(rows):
        vals = np.empty((r, members[0].D), np.float32)
        for i in range(r):
            m = members[0] if i in cached[t] else members[i % world]
            vals[i] = m.read_rows(t, [i])[0]
        out.append(vals)
    return out


@pytest.mark.parametrize("world,storage", [(2, "hbm"), (3, "hbm"), (2, "host")])
def test_group_replace_cache_keeps_trained_rows(ec, torch, world, storage):
    """Row-sharded tables trained for two steps on the peer-memory exchange,
    then re-placed (rows enter and leave the replicated cache): every row's
    value is unchanged bit for bit, and the replicas agree."""
    rows, D, B, P = [700, 90, 13], 8, 32, 4
    n = B * P
    dists = _dists(ec, rows)
    old = [d.top_ids(k) for d, k in zip(dists, [50, 10, 3])]
    new = [d.top_ids(k) for d, k in zip(dists, [120, 4, 6])]
    members = [ec.EmbeddingTables(rows, D, storage=storage, rank=r, world=world, max_lookups_per_table=n,
                                  max_batch_size=B) for r in range(world)]
    for m in members:
        m.init_synthetic(8, 0.2)
    grp = ec.EmbeddingGroup(members, p2p=True)
    for m in members:
        m.place_cache(old)
    offs = np.arange(len(rows) + 1, dtype=np.int64) * n
    for step in range(2):
        ids = [_ids(ec, torch, dists, n, 70 + step, r) for r in range(world)]
        outs = grp.forward(ids, offs, B, P)
        grp.backward([o.clone() for o in outs], 0.05)
    torch.cuda.synchronize()
    before = _authoritative(members, rows, world, [set(map(int, c)) for c in old])
    for m in members:
        m.place_cache(new)
    after = _authoritative(members, rows, world, [set(map(int, c)) for c in new])
    for t in range(len(rows)):
        assert np.array_equal(before[t], after[t]), f"table {t}: values changed by the re-placement"
        for m in members[1:]:
            assert np.array_equal(m.read_rows(t, new[t]), members[0].read_rows(t, new[t])), "replicas differ"
    grp.close()
    for m in members:
        m.close()


def test_group_replace_cache_after_training_without_peer_memory(ec, torch):
    """Without the peer-memory exchange another shard's trained rows are not
    readable: a re-placement that would need them is refused (not silently
    refilled from the synthetic init); before training it is allowed."""
    rows, D, B, P = [500, 40], 8, 16, 2
    n = B * P
    world = 2
    dists = _dists(ec, rows)
    members = [ec.EmbeddingTables(rows, D, rank=r, world=world, max_lookups_per_table=n, max_batch_size=B)
               for r in range(world)]
    for m in members:
        m.init_synthetic(3, 0.1)
    grp = ec.EmbeddingGroup(members, p2p=False)
    for m in members:
        m.place_cache([d.top_ids(5) for d in dists])  # untrained: synthetic values are current
    offs = np.arange(len(rows) + 1, dtype=np.int64) * n
    ids = [_ids(ec, torch, dists, n, 5, r) for r in range(world)]
    outs = grp.forward(ids, offs, B, P)
    grp.backward([o.clone() for o in outs], 0.1)
    torch.cuda.synchronize()
    with pytest.raises(ec.ValidationError):
        members[0].place_cache([d.top_ids(50) for d in dists])
    grp.close()
    for m in members:
        m.close()


def test_p2p_import_rejects_mismatched_geometry(ec, torch):
    """Every rank indexes peers' shards and inboxes from its own geometry:
    blobs exported by a rank with other rows / dim / batch capacity / tier,
    or in the wrong rank slot, are refused before any handle is opened."""
    base = dict(rank=0, world=2, max_lookups_per_table=64, max_batch_size=64)
    a = ec.EmbeddingTables([100, 50], 8, **base)
    good = ec.EmbeddingTables([100, 50], 8, **{**base, "rank": 1})
    bad = [ec.EmbeddingTables([100, 51], 8, **{**base, "rank": 1}),
           ec.EmbeddingTables([100, 50], 16, **{**base, "rank": 1}),
           ec.EmbeddingTables([100, 50], 8, **{**base, "rank": 1, "max_lookups_per_table": 128})]
    for b in bad:
        with pytest.raises(ec.ValidationError, match="geometry"):
            a.p2p_import([a.p2p_export(), b.p2p_export()])
    with pytest.raises(ec.ValidationError, match="exported by rank"):
        a.p2p_import([good.p2p_export(), a.p2p_export()])
    for t in [a, good, *bad]:
        t.close()
