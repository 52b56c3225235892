"""Row-sharded multi-rank data path (K4) on one B200 through the in-process
loopback group: G ranks, owner(id) = id % G, replicated hot cache, the same
route / serve / gradient-return / rank-ordered replica update as the NCCL
path.  Checked against the fp64 oracle (1e-5 relative), the reference's
counts, and replica bit-identity."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu
RTOL, ATOL = 1e-5, 1e-6


@pytest.fixture(scope="module")
def torch():
    import torch
    assert torch.cuda.is_available()
    return torch


def _ids(ec, torch, dists, n, seed, rank):
    T = len(dists)
    ids = torch.empty(T * n, dtype=torch.int32, device="cuda")
    for t, d in enumerate(dists):
        ec.DiscreteSampler(d).sample_into(ids.data_ptr() + 4 * n * t,
                                          ec.substream_seed(ec.substream_seed(seed, rank), t), 0, n)
    torch.cuda.synchronize()
    return ids


def _current_rows(members, t, ids, world, cached):
    """Authoritative values: cache copy (any rank) or the owner's shard."""
    out = np.empty((len(ids), members[0].D), np.float32)
    for k, i in enumerate(ids):
        r = 0 if int(i) in cached else int(i) % world
        out[k] = members[r].read_rows(t, [int(i)])[0]
    return out


@pytest.mark.parametrize("world,storage,p2p", [(2, "hbm", False), (3, "host", False), (4, "hbm", False),
                                               (8, "hbm", False), (2, "hbm", True), (3, "hbm", True),
                                               (4, "hbm", True), (8, "hbm", True), (2, "host", True),
                                               (3, "host", True), (8, "host", True)])
def test_group_forward_backward(ec, torch, ref, world, storage, p2p):
    rows, D, B, P = [5000, 37, 20000, 1], 16, 64, 5
    n = B * P
    seed, scale, lr = 99, 0.1, 0.5
    dists = [ec.materialize(ec.DistributionSpec.parametric(ec.DistributionKind.zipf, r, 1.05)) for r in rows]
    caches = [d.top_ids(min(len(d), k)) for d, k in zip(dists, [40, 3, 200, 0])]
    cached = [set(int(x) for x in c) for c in caches]
    members = [ec.EmbeddingTables(rows, D, storage=storage, rank=r, world=world, max_lookups_per_table=n,
                                  max_batch_size=B) for r in range(world)]
    for m in members:
        m.init_synthetic(seed, scale)
    group = ec.EmbeddingGroup(members, p2p=p2p)
    for m in members:
        m.place_cache(caches)
    offs = np.arange(len(rows) + 1, dtype=np.int64) * n
    bag = np.arange(B + 1, dtype=np.int64) * P

    for step in range(3):
        ids = [_ids(ec, torch, dists, n, 1000 + step, r) for r in range(world)]
        ids_h = [x.cpu().numpy().view(np.uint32) for x in ids]
        # expected pooled outputs from the current authoritative rows
        want = []
        for r in range(world):
            w = np.empty((B, len(rows) * D))
            for t in range(len(rows)):
                u, inv = O.dedup(ids_h[r][offs[t]:offs[t + 1]])
                cur = _current_rows(members, t, u, world, cached[t])
                _, o64 = O.pool(cur, inv[:n], bag)
                w[:, t * D:(t + 1) * D] = o64
            want.append(w)
        outs = group.forward(ids, offs, B, P)
        torch.cuda.synchronize()
        for r in range(world):
            got = outs[r].cpu().numpy()
            for t in range(len(rows)):  # fp32 sums of P rows: absolute bound scales with the table's values
                sl = slice(t * D, (t + 1) * D)
                np.testing.assert_allclose(got[:, sl], want[r][:, sl], rtol=RTOL,
                                           atol=ATOL * max(1.0, np.abs(want[r][:, sl]).max()))
            st = members[r].stats(per_table=True)
            remote = 0
            for t in range(len(rows)):
                seg = ids_h[r][offs[t]:offs[t + 1]]
                u, _ = O.dedup(seg)
                assert (members[r].export_unique(t) == u).all()
                miss = np.array([x for x in u if int(x) not in cached[t]], dtype=np.uint32)
                assert st["miss_per_table"][t] == miss.size
                remote += int((miss % world != r).sum())
                a, nc = ref.ref_segment_counts(seg, [0, n], [rows[t]], [np.asarray(caches[t], np.uint32)])
                assert (a[0], nc[0]) == (u.size, miss.size)  # bit-exact vs the reference
            assert st["wire_rows"] == remote

        # backward: every touched row gets w - lr * (sum of all ranks' grads)
        grads = [torch.randn(B, len(rows) * D, device="cuda") for _ in range(world)]
        before = {}
        acc = {}
        for t in range(len(rows)):
            for r in range(world):
                seg = ids_h[r][offs[t]:offs[t + 1]]
                u, inv = O.dedup(seg)
                g = grads[r].cpu().numpy()[:, t * D:(t + 1) * D]
                ug, _ = O.backward_sgd(np.ascontiguousarray(g), inv[:n], bag, np.zeros((u.size, D), np.float32), lr)
                for k, i in enumerate(u):
                    key = (t, int(i))
                    acc[key] = acc.get(key, 0.0) + ug[k]
                    if key not in before:
                        before[key] = _current_rows(members, t, [i], world, cached[t])[0].astype(np.float64)
        group.backward(grads, lr)
        torch.cuda.synchronize()
        if p2p:  # hot-row sync of this backward: gradients to other owners, their updated rows back
            for m in members:
                st = m.stats()
                assert st["hot_sync_rows"] > 0 and st["hot_sync_bytes"] == st["hot_sync_rows"] * (4 + 4 * D)
        # fp32 atomics sum each row's gradients in a varying order: the bound
        # is 1e-5 relative to the largest updated value
        scale = max(np.abs(before[k] - lr * g).max() for k, g in acc.items())
        for (t, i), gsum in acc.items():
            exp = before[(t, i)] - lr * gsum
            if i in cached[t]:
                reps = [m.read_rows(t, [i])[0] for m in members]
                for rr in reps[1:]:
                    assert (rr == reps[0]).all(), "hot-row replicas diverged"
                got = reps[0]
            else:
                got = members[i % world].read_rows(t, [i])[0]
            np.testing.assert_allclose(got, exp, rtol=RTOL, atol=1e-5 * scale)
    group.close()
    for m in members:
        m.close()


def test_group_rejects_direct_calls(ec, torch):
    ms = [ec.EmbeddingTables([100], 4, rank=r, world=2, max_lookups_per_table=8, max_batch_size=8) for r in range(2)]
    for m in ms:
        m.init_synthetic(1, 1.0)
    g = ec.EmbeddingGroup(ms)
    ids = torch.zeros(8, dtype=torch.int32, device="cuda")
    with pytest.raises(ec.ValidationError):
        ms[0].forward(ids, [0, 8], 8, 1)
    g.close()
    with pytest.raises(ec.ValidationError):  # world 2 without a transport
        ms[0].forward(ids, [0, 8], 8, 1)


def test_group_p2p_forward_only_steps(ec, torch):
    """Evaluation forwards (no backward) release the peers' barriers; a second
    backward of one forward is refused (its updates would race the peers'
    next forward)."""
    world, rows, D, B = 2, [300, 50], 8, 16
    ms = [ec.EmbeddingTables(rows, D, rank=r, world=world, max_lookups_per_table=B, max_batch_size=B)
          for r in range(world)]
    for m in ms:
        m.init_synthetic(3, 1.0)
    g = ec.EmbeddingGroup(ms, p2p=True)
    offs = np.array([0, B, 2 * B], np.int64)
    ids = [torch.randint(0, 50, (2 * B,), dtype=torch.int32, device="cuda") for _ in range(world)]
    first = [o.clone() for o in g.forward(ids, offs, B, 1)]
    for _ in range(3):  # forward-only steps: identical outputs, nothing applied
        again = g.forward(ids, offs, B, 1)
        for a, b in zip(first, again):
            assert torch.equal(a, b)
    g.backward([torch.ones_like(o) for o in first], 0.5)
    with pytest.raises(ec.ValidationError):
        g.backward([torch.ones_like(o) for o in first], 0.5)
    after = g.forward(ids, offs, B, 1)
    torch.cuda.synchronize()
    # every looked-up row moved by -0.5 * (its count over both ranks); pooled
    # outputs (sum pooling, P = 1) shift by exactly that
    for r in range(world):
        for t in range(2):
            col = slice(t * D, (t + 1) * D)
            seg = torch.cat([i[t * B:(t + 1) * B] for i in ids])
            cnt = torch.bincount(seg.long(), minlength=rows[t]).float()
            exp = first[r][:, col] - 0.5 * cnt[ids[r][t * B:(t + 1) * B].long()][:, None]
            torch.testing.assert_close(after[r][:, col], exp, rtol=1e-5, atol=1e-5)
    g.close()
    for m in ms:
        m.close()


def test_p2p_import_validation(ec, torch):
    """ec_tables_p2p_import refuses a single rank, wrong blob sizes, a blob
    count that is not the world size and ranks on different tiers; p2p_disable
    returns a rank to 'no transport'."""
    one = ec.EmbeddingTables([100], 4, max_lookups_per_table=8, max_batch_size=8)
    with pytest.raises(ec.ValidationError):
        one.p2p_import([one.p2p_export()])
    one.close()
    hb = [ec.EmbeddingTables([100], 4, storage="hbm", rank=r, world=2, max_lookups_per_table=8, max_batch_size=8)
          for r in range(2)]
    ho = ec.EmbeddingTables([100], 4, storage="host", rank=1, world=2, max_lookups_per_table=8, max_batch_size=8)
    blobs = [m.p2p_export() for m in hb]
    assert len(blobs[0]) == 12 * 64 + 48
    with pytest.raises(ValueError):
        hb[0].p2p_import(blobs[:1])
    with pytest.raises(ValueError):
        hb[0].p2p_import([blobs[0], blobs[1][:-1]])
    with pytest.raises(ec.ValidationError):  # rank 1 exports a host shard, rank 0 holds HBM
        hb[0].p2p_import([blobs[0], ho.p2p_export()])
    hb[0].p2p_disable()
    ids = torch.zeros(8, dtype=torch.int32, device="cuda")
    with pytest.raises(ec.ValidationError):  # world 2 without a transport
        hb[0].forward(ids, [0, 8], 8, 1)
    for m in hb + [ho]:
        m.close()
