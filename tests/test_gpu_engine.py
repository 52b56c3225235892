"""Lookup engine (K1 dedup, K2 hit/miss, K3 gather, K5 pool, K6 backward) on
the GPU vs the oracle and the compiled reference.

Bar (north_star): unique sets, inverse indices, hit/miss sets and row counts
bit-exact; gathered rows bitwise (rows are copied unchanged); pooled outputs
and updated rows within 1e-5 relative of the fp64 restatement (tolerance
written per assertion, atol covers values that cancel to ~0)."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-5, 1e-6
KAGGLE = [1460, 583, 10131227, 2202608, 305, 24, 12517, 633, 3, 93145, 5683, 8351593, 3194, 27, 14992,
          5461306, 10, 5652, 2173, 4, 7046547, 18, 15, 286181, 105, 142572]


@pytest.fixture(scope="module")
def torch():
    import torch
    assert torch.cuda.is_available()
    return torch


def make_ids(ec, torch, dists, n_per_table, seed):
    """Table t's lookups = draws [0, n_t) of SplitMix64(substream(seed, t)) (K0)."""
    offs = np.concatenate([[0], np.cumsum(n_per_table)]).astype(np.int64)
    ids = torch.empty(int(offs[-1]), dtype=torch.int32, device="cuda")
    for t, d in enumerate(dists):
        if n_per_table[t]:
            ec.DiscreteSampler(d).sample_into(ids.data_ptr() + 4 * int(offs[t]), ec.substream_seed(seed, t), 0,
                                              int(n_per_table[t]))
    torch.cuda.synchronize()
    return ids, offs


def check_batch(ec, tab, ids_host, offs, caches, rows, D, seed, scale, bag_offs=None, P=None, B=None,
                out=None, ref=None):
    """Compare every export of the last forward with the oracle."""
    T = len(rows)
    stats = tab.stats(per_table=True)
    pooled = out.cpu().numpy() if out is not None else None
    for t in range(T):
        seg = ids_host[offs[t]:offs[t + 1]]
        u_o, inv_o = O.dedup(seg)
        u_g = tab.export_unique(t)
        assert (u_g == u_o).all(), f"table {t}: unique set/order"
        assert (tab.export_inverse(t) == inv_o[:seg.size]).all(), f"table {t}: inverse"
        slot = np.full(rows[t], -1, np.int32)
        if len(caches[t]):
            slot[np.asarray(caches[t], np.int64)] = np.arange(len(caches[t]), dtype=np.int32)
        hit_o, miss_o = O.partition(u_o, slot)
        assert (tab.export_hit(t) == hit_o).all(), f"table {t}: hit/miss"
        assert stats["unique_per_table"][t] == u_o.size
        assert stats["miss_per_table"][t] == miss_o
        want_rows = O.synthetic_rows(seed, scale, t, u_o, D)
        assert (tab.export_rows(t) == want_rows).all(), f"table {t}: gathered rows"
        if ref is not None and seg.size:
            a, nc = ref.ref_segment_counts(seg, [0, seg.size], [rows[t]], [np.asarray(caches[t], np.uint32)])
            assert (a[0], nc[0]) == (u_o.size, miss_o), f"table {t}: counts vs reference"
        if pooled is not None:
            if bag_offs is None:
                bo = np.arange(B + 1, dtype=np.int64) * P
            else:
                bo = bag_offs[t * B:(t + 1) * B + 1] - offs[t]
            _, o64 = O.pool(want_rows, inv_o[:seg.size], bo)
            np.testing.assert_allclose(pooled[:, t * D:(t + 1) * D], o64, rtol=RTOL, atol=ATOL)
    return stats


@pytest.mark.parametrize("storage,graphs,mode", [("hbm", False, "auto"), ("host", False, "auto"),
                                                 ("hbm", True, "auto"), ("host", True, "auto"),
                                                 ("hbm", False, "tiles"), ("host", True, "tiles"),
                                                 ("hbm", False, "cluster"), ("host", True, "cluster"),
                                                 ("hbm", False, "table"), ("host", True, "table"),
                                                 # fused path (auto scatter) with the cluster dedup: the
                                                 # pinned-host tier pools through per-lookup row sources
                                                 ("hbm", True, "cluster-fused"), ("host", True, "cluster-fused"),
                                                 ("host", False, "cluster-fused")])
def test_small_fixed_pooling_fwd_bwd(ec, torch, ref, storage, graphs, mode):
    if graphs:  # CUDA-graph capture/replay needs a non-default stream
        with torch.cuda.stream(torch.cuda.Stream()):
            _small_fixed_pooling(ec, torch, ref, storage, True, mode)
    else:
        _small_fixed_pooling(ec, torch, ref, storage, False, mode)


def _small_fixed_pooling(ec, torch, ref, storage, graphs, mode):
    rows, D, B, P = [1000, 37, 5000, 1], 16, 64, 7
    dists = [ec.materialize(ec.DistributionSpec.parametric(ec.DistributionKind.zipf, r, 1.05)) for r in rows]
    caches = [d.top_ids(min(len(d), k)) for d, k in zip(dists, [50, 0, 500, 1])]
    tab = ec.EmbeddingTables(rows, D, storage=storage, max_lookups_per_table=B * P, max_batch_size=B)
    tab.use_graphs(graphs)
    if mode == "cluster-fused":
        tab.dedup_mode("cluster")
        tab.scatter_mode("auto")
    else:
        tab.dedup_mode(mode)
        tab.scatter_mode("atomic" if mode == "tiles" else "transpose")
    seed, scale = 1234, 0.05
    tab.init_synthetic(seed, scale)
    tab.place_cache(caches)
    ids, offs = make_ids(ec, torch, dists, [B * P] * len(rows), 77)
    out = tab.forward(ids, offs, B, P)
    ids_h = ids.cpu().numpy().view(np.uint32)
    st = check_batch(ec, tab, ids_h, offs, caches, rows, D, seed, scale, P=P, B=B, out=out, ref=ref)
    assert st["lookups"] == B * P * len(rows)
    assert st["model_bytes"] == st["miss_rows"] * D * 4 + st["index_units"] * 4

    # backward: SGD on every unique row, checked through read_rows
    g = torch.randn(B, len(rows) * D, device="cuda", dtype=torch.float32)
    lr = 0.25
    tab.backward(g, lr)
    torch.cuda.synchronize()
    gh = g.cpu().numpy()
    for t in range(len(rows)):
        seg = ids_h[offs[t]:offs[t + 1]]
        u, inv = O.dedup(seg)
        w0 = O.synthetic_rows(seed, scale, t, u, D)
        _, want = O.backward_sgd(np.ascontiguousarray(gh[:, t * D:(t + 1) * D]), inv[:seg.size],
                                 np.arange(B + 1, dtype=np.int64) * P, w0, lr)
        got = tab.read_rows(t, u)
        # fp32 sums of several O(1) gradients: absolute error scales with the
        # row magnitude, so atol is 1e-5 of the largest |w| in the table
        np.testing.assert_allclose(got, want, rtol=RTOL, atol=1e-5 * np.abs(want).max())
    # a second batch sees the updated rows and a clean hash table
    ids2, _ = make_ids(ec, torch, dists, [B * P] * len(rows), 78)
    tab.forward(ids2, offs, B, P)
    ids2_h = ids2.cpu().numpy().view(np.uint32)
    for t in range(len(rows)):
        seg = ids2_h[offs[t]:offs[t + 1]]
        u, _ = O.dedup(seg)
        assert (tab.export_unique(t) == u).all()
        assert (tab.export_rows(t) == tab.read_rows(t, u)).all()
    # same buffers, new contents: a replayed graph must see the new ids
    ids.copy_(ids2)
    tab.forward(ids, offs, B, P)
    for t in range(len(rows)):
        u, inv = O.dedup(ids2_h[offs[t]:offs[t + 1]])
        assert (tab.export_unique(t) == u).all()
        assert (tab.export_inverse(t) == inv[:B * P]).all()
    tab.close()


@pytest.mark.parametrize("storage", ["hbm", "host"])
@pytest.mark.parametrize("mode", ["auto", "cluster"])
def test_csr_bags_empty_bags_and_empty_table(ec, torch, storage, mode):
    rows, D, B = [300, 50, 1000], 8, 40
    rng = np.random.default_rng(3)
    lens = [rng.integers(0, 9, B), np.zeros(B, np.int64), rng.integers(0, 4, B)]
    lens[0][:5] = 0
    n = [int(x.sum()) for x in lens]
    offs = np.concatenate([[0], np.cumsum(n)]).astype(np.int64)
    ids_h = np.concatenate([rng.integers(0, r, k) for r, k in zip(rows, n)]).astype(np.uint32)
    bag = np.concatenate([[0], np.cumsum(np.concatenate(lens))]).astype(np.int64)
    tab = ec.EmbeddingTables(rows, D, storage=storage, max_lookups_per_table=max(n), max_batch_size=B)
    tab.dedup_mode(mode)  # cluster: the fused path (pinned-host tier: row sources through CSR bags)
    tab.init_synthetic(5, 1.0)
    w0 = [tab.read_rows(t, np.arange(rows[t])) for t in range(3)]
    caches = [np.arange(10), [], np.arange(0, 1000, 3)]
    tab.place_cache(caches)
    ids = torch.from_numpy(ids_h.view(np.int32)).cuda()
    bag_t = torch.from_numpy(bag).cuda()
    out = tab.forward(ids, offs, B, bag_offsets=bag_t)
    check_batch(ec, tab, ids_h, offs, caches, rows, D, 5, 1.0, bag_offs=bag, B=B, out=out)
    assert (out.cpu().numpy()[:, D:2 * D] == 0).all()  # empty table pools to zeros
    g = torch.randn(B, 3 * D, device="cuda")
    tab.backward(g, 0.5)
    torch.cuda.synchronize()
    gh = g.cpu().numpy()
    for t in range(3):  # CSR bags through the transposed reduction (binary-searched bag of each lookup)
        seg = ids_h[offs[t]:offs[t + 1]]
        if not seg.size:
            continue
        u, inv = O.dedup(seg)
        bo = bag[t * B:(t + 1) * B + 1] - offs[t]
        _, want = O.backward_sgd(np.ascontiguousarray(gh[:, t * D:(t + 1) * D]), inv[:seg.size], bo, w0[t][u], 0.5)
        np.testing.assert_allclose(tab.read_rows(t, u), want, rtol=RTOL, atol=1e-5 * np.abs(want).max())
    tab.close()


def test_out_of_range_id_is_a_validation_error(ec, torch):
    tab = ec.EmbeddingTables([10], 4, max_lookups_per_table=4, max_batch_size=4)
    tab.init_synthetic(1, 1.0)
    ids = torch.tensor([1, 2, 10, 3], dtype=torch.int32, device="cuda")
    tab.forward(ids, [0, 4], 4, 1)
    with pytest.raises(ec.ValidationError):
        tab.stats()
    with pytest.raises(ec.ValidationError):
        tab.place_cache([[11]])
    with pytest.raises(ec.ValidationError):
        tab.forward(ids, [0, 5], 4, 1)
    tab.close()


@pytest.mark.parametrize("storage", ["hbm", "host"])
@pytest.mark.parametrize("mode", ["cluster", "tiles"])
def test_out_of_range_id_pools_a_zero_row(ec, torch, storage, mode):
    """An out-of-range id is skipped (inverse kInvalidSlot, reported as a
    ValidationError by stats) and pools a zero row; every other bag still
    pools its row -- on the fused cluster path too, whose pinned-host tier
    pools through per-lookup row-source words (kNoSource for the bad id)."""
    import numpy as np
    tab = ec.EmbeddingTables([10, 300], 4, storage=storage, max_lookups_per_table=4, max_batch_size=4)
    tab.init_synthetic(1, 1.0)
    tab.place_cache([[1, 2], [5]])
    tab.dedup_mode(mode)
    ids = torch.tensor([1, 2, 10, 3, 5, 299, 7, 300], dtype=torch.int32, device="cuda")
    out = tab.forward(ids, [0, 4, 8], 4, 1).cpu().numpy()
    with pytest.raises(ec.ValidationError):
        tab.stats()
    h = ids.cpu().numpy()
    for t in range(2):
        for s in range(4):
            i = int(h[t * 4 + s])
            got = out[s, t * 4:(t + 1) * 4]
            if i >= [10, 300][t]:
                assert (got == 0).all()
            else:
                np.testing.assert_array_equal(got, tab.read_rows(t, np.array([i], np.uint32))[0])
    tab.close()


@pytest.mark.parametrize("mode", ["auto", "cluster"])
def test_config1_full_size_counts_and_sets(ec, torch, ref, mode):
    """Config 1 (BASELINE.json configs[0]): 8 tables x 1M rows, D=64, b=4096,
    P=20 (n = 81,920 per table); counts bit-exact vs the reference,
    unique/inverse/hit sets bit-exact vs the oracle, three cache sizes."""
    T, E, D, B, P = 8, 1_000_000, 64, 4096, 20
    dist = ec.materialize(ec.DistributionSpec.parametric(ec.DistributionKind.zipf, E, 1.05))
    tab = ec.EmbeddingTables([E] * T, D, max_lookups_per_table=B * P, max_batch_size=B)
    tab.dedup_mode(mode)
    tab.init_synthetic(9, 0.01)
    for k in (0, 10_000, 100_000):
        caches = [dist.top_ids(k)] * T
        tab.place_cache(caches)
        ids, offs = make_ids(ec, torch, [dist] * T, [B * P] * T, 20241101 + k)
        out = tab.forward(ids, offs, B, P)
        check_batch(ec, tab, ids.cpu().numpy().view(np.uint32), offs, caches, [E] * T, D, 9, 0.01, P=P, B=B,
                    out=out, ref=ref)
    tab.close()


@pytest.mark.parametrize("mode", ["auto", "cluster", "table"])
def test_config2_kaggle_shape_host_tier(ec, torch, ref, mode):
    """Config 2 (BASELINE.json configs[1]): 26 Kaggle-cardinality tables, D=16,
    b=16384, P=1, 256 MB HBM cache placed by global top-k probability, cold
    rows in pinned host memory.  Counts vs reference, sets vs oracle, every
    dedup kernel that fits the shape."""
    D, B = 16, 16384
    dists = [ec.materialize(ec.DistributionSpec.parametric(ec.DistributionKind.zipf, r, 1.05)) for r in KAGGLE]
    ks = ec.place_topk_global(dists, (256 << 20) // (D * 4))
    caches = [d.top_ids(k) for d, k in zip(dists, ks)]
    tab = ec.EmbeddingTables(KAGGLE, D, storage="host", max_lookups_per_table=B, max_batch_size=B)
    tab.dedup_mode(mode)
    tab.init_synthetic(3, 0.1)
    tab.place_cache(caches)
    ids, offs = make_ids(ec, torch, dists, [B] * 26, 555)
    out = tab.forward(ids, offs, B, 1)
    st = check_batch(ec, tab, ids.cpu().numpy().view(np.uint32), offs, caches, KAGGLE, D, 3, 0.1, P=1, B=B,
                     out=out, ref=ref)
    assert st["miss_rows"] > 0 and st["hit_rows"] > 0
    tab.close()


def check_sgd(got, w0, g, inv, bag, lr, what, rtol=RTOL):
    """Updated rows vs the fp64 restatement w0 - lr * sum(g) (orc_backward_sgd).

    The bound is 1e-5 relative to the magnitudes summed, |w0| + lr * sum|g|
    per element: the order-of-summation tolerance of a sum (its condition
    number).  Where a row's gradients share a sign (grad = pooled output, as in
    the bench) that is 1e-5 of |w0| + |lr * sum(g)|.  Returns the worst
    err / bound and the worst plain relative error err / |want| over elements
    with |want| >= 1e-3 * max|want| (reported, not asserted: values that
    cancel to ~0 have no meaningful plain relative error)."""
    ug, _ = O.backward_sgd(g, inv, bag, w0, lr)
    uabs, _ = O.backward_sgd(np.abs(g), inv, bag, w0, lr)
    want = w0.astype(np.float64) - lr * ug
    scale = np.abs(w0.astype(np.float64)) + lr * uabs
    err = np.abs(got.astype(np.float64) - want)
    bound = rtol * scale
    bad = err > bound
    if bad.any():
        k = np.argwhere(bad)[0]
        raise AssertionError(f"{what}: {bad.sum()} of {bad.size} elements over 1e-5 relative; first unique "
                             f"{k[0]} got {got[k[0], k[1]]} want {want[k[0], k[1]]} w0 {w0[k[0], k[1]]} "
                             f"bound {bound[k[0], k[1]]}")
    big = np.abs(want) >= 1e-3 * np.abs(want).max() if want.size else np.zeros(0, bool)
    plain = float((err[big] / np.abs(want[big])).max()) if big.any() else 0.0
    return float((err / np.where(bound > 0, bound, 1.0)).max()) if err.size else 0.0, plain


def run_training_step(ec, torch, rows, D, B, P, storage, cache_bytes, seed, lr=0.01, mode=None, scatter=None,
                      init=(4, 0.05)):
    """One bench-style training step on fresh tables: forward, backward with
    grad = the pooled output (loss = 1/2 |pooled|^2), SGD at lr.  Every touched
    row (cache, HBM shard or pinned host) is checked against check_sgd."""
    dists = [ec.materialize(ec.DistributionSpec.parametric(ec.DistributionKind.zipf, r, 1.05)) for r in rows]
    ks = ec.place_topk_global(dists, cache_bytes // (D * 4)) if cache_bytes else [0] * len(rows)
    caches = [d.top_ids(k) for d, k in zip(dists, ks)]
    tab = ec.EmbeddingTables(rows, D, storage=storage, max_lookups_per_table=B * P, max_batch_size=B)
    if mode:
        tab.dedup_mode(mode)
    if scatter:
        tab.scatter_mode(scatter)
    tab.init_synthetic(*init)
    tab.place_cache(caches)
    ids, offs = make_ids(ec, torch, dists, [B * P] * len(rows), seed)
    out = tab.forward(ids, offs, B, P)
    grad = out.clone()
    tab.backward(grad, lr)
    torch.cuda.synchronize()
    ids_h = ids.cpu().numpy().view(np.uint32)
    g = grad.cpu().numpy()
    bag = np.arange(B + 1, dtype=np.int64) * P
    worst, plain = 0.0, 0.0
    for t in range(len(rows)):
        seg = ids_h[offs[t]:offs[t + 1]]
        u, inv = O.dedup(seg)
        w0 = O.synthetic_rows(init[0], init[1], t, u, D)
        w, p = check_sgd(tab.read_rows(t, u), w0, np.ascontiguousarray(g[:, t * D:(t + 1) * D]), inv[:seg.size],
                         bag, lr, f"table {t}")
        worst, plain = max(worst, w), max(plain, p)
    st = tab.stats()
    tab.close()
    print(f"[sgd parity] rows={len(rows)} D={D} B={B} P={P} {storage} mode={mode} scatter={scatter}: "
          f"max err/bound {worst:.3f}, max plain rel err {plain:.2e}")
    return st


@pytest.mark.parametrize("storage", ["host", "hbm"])
def test_config2_kaggle_shape_training_step(ec, torch, storage):
    """One bench-style training step at the Kaggle shape (configs[1]) on the
    fused single-rank path (SGD inside the scatter): every touched row within
    1e-5 relative of the fp64 oracle (check_sgd)."""
    run_training_step(ec, torch, KAGGLE, 16, 16384, 1, storage, 256 << 20, 909)


@pytest.mark.parametrize("D", [4, 32, 128])
@pytest.mark.parametrize("storage,mode,scatter", [("hbm", None, None), ("host", None, None),
                                                  ("hbm", "tiles", "transpose"), ("host", "tiles", "atomic")])
def test_every_row_width_training_step(ec, torch, D, storage, mode, scatter):
    """The row kernels at the widths the other tests do not use (4, 32 and
    128 floats per row: 1, 8 and 32 lanes per row): the fused path (cluster
    dedup, SGD in the scatter), the tile path with the transpose backward
    (SGD of single-chunk rows inside k_bwd_reduce on HBM rows) and the atomic
    scatter with the pinned-host write-back; pooling 4, a small cache."""
    run_training_step(ec, torch, [1000, 37, 50000, 3], D, 512, 4, storage, 100 * D * 4, 31 + D, mode=mode,
                      scatter=scatter)


@pytest.mark.parametrize("cache_bytes", [0, 64 * 16 * 4])
def test_host_tier_heavy_misses_training_step(ec, torch, cache_bytes):
    """Pinned-host misses with thousands of lookups each (no cache, or a
    64-row one, over small Zipf tables): their gradients take the fp64 path
    and are rounded once by k_g64_misses before the host write-back."""
    run_training_step(ec, torch, [1000, 50, 200000, 3], 16, 16384, 1, "host", cache_bytes, 4711)


@pytest.mark.parametrize("mode", ["auto", "tiles", "auto->tiles", "tiles->auto"])
def test_host_tier_heavy_misses_consecutive_steps(ec, torch, mode):
    """Four training steps on the same tables with heavy pinned-host misses:
    every step's updated rows within 1e-5 of the fp64 update from the rows it
    started from -- so the per-unique counts and fp64 sums a step leaves for
    its write-back (cleared before the buffer set's next dedup) never leak
    into a later step.  "tiles": no counts, sums folded by k_g64_misses."""
    rows, D, B, P, lr = [1000, 50, 3, 20000], 16, 16384, 1, 0.01
    dists = [ec.materialize(ec.DistributionSpec.parametric(ec.DistributionKind.zipf, r, 1.05)) for r in rows]
    tab = ec.EmbeddingTables(rows, D, storage="host", max_lookups_per_table=B * P, max_batch_size=B)
    modes = mode.split("->")  # a switch half way: counts / sums one path left must not reach the other
    tab.init_synthetic(4, 0.05)
    bag = np.arange(B + 1, dtype=np.int64) * P
    for step in range(4):
        tab.dedup_mode(modes[min(step // 2, len(modes) - 1)])
        ids, offs = make_ids(ec, torch, dists, [B * P] * len(rows), 300 + step)
        out = tab.forward(ids, offs, B, P)
        torch.cuda.synchronize()
        ids_h = ids.cpu().numpy().view(np.uint32)
        segs = [O.dedup(ids_h[offs[t]:offs[t + 1]]) for t in range(len(rows))]
        w0 = [tab.read_rows(t, u) for t, (u, _) in enumerate(segs)]
        grad = out.clone()
        tab.backward(grad, lr)
        torch.cuda.synchronize()
        g = grad.cpu().numpy()
        for t, (u, inv) in enumerate(segs):
            check_sgd(tab.read_rows(t, u), w0[t], np.ascontiguousarray(g[:, t * D:(t + 1) * D]), inv[:B * P], bag, lr,
                      f"step {step} table {t}")
    tab.close()


@pytest.mark.parametrize("mode", ["cluster", "tiles", "auto"])
def test_many_tables_cross_table_scan(ec, torch, ref, mode):
    """100 tables: the cluster kernel's warp-parallel look-back walks more than
    32 lower tables (several rounds), and k_compact's tile look-back spans 100
    tables' tiles; sizes from 1 to 200K rows, some tables empty in the batch.
    Sets, inverse, hit/miss and rows vs the oracle; then a training step."""
    rng = np.random.default_rng(17)
    rows = [int(x) for x in rng.choice([1, 3, 40, 900, 5000, 70000, 200000], size=100)]
    n = [0 if t % 17 == 5 else int(rng.integers(1, 3000)) for t in range(100)]
    dists = [ec.materialize(ec.DistributionSpec.parametric(ec.DistributionKind.zipf, r, 1.05)) for r in rows]
    caches = [d.top_ids(min(len(d), k)) for d, k in zip(dists, rng.integers(0, 50, size=100))]
    D, B = 8, 1
    offs = np.concatenate([[0], np.cumsum(n)]).astype(np.int64)
    bag = np.concatenate([[0], offs[1:]]).astype(np.int64)
    tab = ec.EmbeddingTables(rows, D, max_lookups_per_table=max(n), max_batch_size=B)
    tab.dedup_mode(mode)
    tab.init_synthetic(6, 0.5)
    tab.place_cache(caches)
    ids, _ = make_ids(ec, torch, dists, n, 1234)
    bag_t = torch.from_numpy(bag).cuda()
    out = tab.forward(ids, offs, B, bag_offsets=bag_t)
    check_batch(ec, tab, ids.cpu().numpy().view(np.uint32), offs, caches, rows, D, 6, 0.5, bag_offs=bag, B=B, ref=ref)
    tab.backward(torch.zeros(B, len(rows) * D, device="cuda"), 0.0)
    tab.close()


@pytest.mark.parametrize("mode", ["cluster", "tiles"])
def test_single_table(ec, torch, ref, mode):
    """One table (no lower tables to look back on; the last table is the
    first): sets, inverse, hit/miss and rows vs the oracle, fused training step."""
    rows, D, B, P = [50000], 16, 5000, 4
    dists = [ec.materialize(ec.DistributionSpec.parametric(ec.DistributionKind.zipf, rows[0], 1.05))]
    caches = [dists[0].top_ids(100)]
    tab = ec.EmbeddingTables(rows, D, max_lookups_per_table=B * P, max_batch_size=B)
    tab.dedup_mode(mode)
    tab.init_synthetic(8, 0.2)
    tab.place_cache(caches)
    ids, offs = make_ids(ec, torch, dists, [B * P], 55)
    out = tab.forward(ids, offs, B, P)
    check_batch(ec, tab, ids.cpu().numpy().view(np.uint32), offs, caches, rows, D, 8, 0.2, P=P, B=B, out=out, ref=ref)
    tab.backward(torch.zeros(B, D, device="cuda"), 0.0)
    tab.close()


def test_dedup_mode_switch_relays_sets_out(ec, torch, ref):
    """Tables sized for the tile path get hashed sets for their large tables;
    forcing the cluster kernel re-lays them out direct-mapped, and going back
    to tiles keeps working: sets, inverse, hit/miss and rows vs the oracle."""
    rows = [3, 24, 5000, 142572, 10131227]
    n_max = 40000  # > the auto-cluster bound: hashed sets for the two large tables
    dists = [ec.materialize(ec.DistributionSpec.parametric(ec.DistributionKind.zipf, r, 1.05)) for r in rows]
    caches = [d.top_ids(k) for d, k in zip(dists, [1, 0, 100, 1000, 20000])]
    D, B, P = 8, 40000, 1
    tab = ec.EmbeddingTables(rows, D, max_lookups_per_table=n_max, max_batch_size=B)
    tab.init_synthetic(4, 0.5)
    tab.place_cache(caches)
    ids, offs = make_ids(ec, torch, dists, [n_max] * len(rows), 77)
    ids_h = ids.cpu().numpy().view(np.uint32)
    for mode in ["auto", "cluster", "tiles", "cluster"]:
        tab.dedup_mode(mode)
        out = tab.forward(ids, offs, B, P)
        check_batch(ec, tab, ids_h, offs, caches, rows, D, 4, 0.5, P=P, B=B, out=out, ref=ref)
        tab.backward(torch.zeros(B, len(rows) * D, device="cuda"), 0.0)
    tab.close()


@pytest.mark.parametrize("scatter", [None, "atomic"])
def test_config1_full_size_training_step(ec, torch, scatter):
    """configs[0] at full size (8 x 1M rows, D=64, b=4096, P=20, no cache, as
    bench --workload cfg1 times it): tile-path dedup, grouped gradient lists and
    k_bwd_reduce (auto), or the atomic scatter; rows within 1e-5 relative."""
    run_training_step(ec, torch, [1_000_000] * 8, 64, 4096, 20, "hbm", 0, 20241101, scatter=scatter)


def test_config3_terabyte_shape_training_step(ec, torch):
    """configs[2]'s per-rank shape at full size (26 TB tables, 188M rows in
    HBM, D=64, b=65536, 1 GB cache), as bench --workload tb times it: every
    touched cache and shard row within 1e-5 relative of the oracle."""
    run_training_step(ec, torch, TB_ROWS, 64, 65536, 1, "hbm", 1 << 30, 7331, init=(5, 0.02))


TB_ROWS = [39884406, 39043, 17289, 7420, 20263, 3, 7120, 1543, 63, 38532951, 2953546, 403346, 10, 2208, 11938,
           155, 4, 976, 14, 39979771, 25641295, 39664984, 585935, 12972, 108, 36]


@pytest.mark.parametrize("mode", ["auto", "cluster"])
def test_config3_terabyte_shape_one_rank(ec, torch, ref, mode):
    """Config 3's per-rank shape (BASELINE.json configs[2] at G=1): 26
    Criteo-Terabyte-cardinality tables (188M rows, 48 GB at D=64) in HBM,
    b=65536, P=1, 1 GB hot cache by global top-k.  Counts bit-exact vs the
    reference, sets / rows / pooled vs the oracle, on the tile path (auto at
    this size) and the cluster kernel at its widest (16 items per thread)."""
    D, B = 64, 65536
    dists = [ec.materialize(ec.DistributionSpec.parametric(ec.DistributionKind.zipf, r, 1.05)) for r in TB_ROWS]
    ks = ec.place_topk_global(dists, (1 << 30) // (D * 4))
    caches = [d.top_ids(k) for d, k in zip(dists, ks)]
    tab = ec.EmbeddingTables(TB_ROWS, D, storage="hbm", max_lookups_per_table=B, max_batch_size=B)
    tab.dedup_mode(mode)
    tab.init_synthetic(5, 0.02)
    tab.place_cache(caches)
    ids, offs = make_ids(ec, torch, dists, [B] * 26, 7331)
    out = tab.forward(ids, offs, B, 1)
    st = check_batch(ec, tab, ids.cpu().numpy().view(np.uint32), offs, caches, TB_ROWS, D, 5, 0.02, P=1, B=B,
                     out=out, ref=ref)
    assert st["miss_rows"] > 0 and st["hit_rows"] > 0
    tab.close()


def test_async_stats_ring_matches_sync_stats(ec, torch):
    """ec_lookup_stats_enqueue/collect (pinned ring, no sync at enqueue)
    decode each batch's counters exactly like the synchronous ec_lookup_stats,
    also when collected after later batches ran; bad slots are errors."""
    rows, D, B, P = [5000, 300, 7], 8, 256, 2
    dists = [ec.materialize(ec.DistributionSpec.parametric(ec.DistributionKind.zipf, r, 1.1)) for r in rows]
    tab = ec.EmbeddingTables(rows, D, storage="host", max_lookups_per_table=B * P, max_batch_size=B)
    tab.place_cache([d.top_ids(k) for d, k in zip(dists, [50, 20, 0])])
    offs = np.arange(len(rows) + 1, dtype=np.int64) * B * P
    want = []
    for j in range(4):
        ids = make_ids(ec, torch, dists, [B * P] * len(rows), 900 + j)[0]
        tab.forward(ids, offs, B, P)
        tab.stats_enqueue(j)
        want.append(tab.stats(per_table=True))
    for j in range(4):
        got = tab.stats_collect(j, per_table=True)
        for k, v in want[j].items():
            assert np.array_equal(np.asarray(got[k]), np.asarray(v)), (j, k)
    with pytest.raises(Exception):
        tab.stats_collect(0)  # already collected
    with pytest.raises(Exception):
        tab.stats_enqueue(4)
    tab.close()


@pytest.mark.parametrize("storage,graphs,depth", [("host", False, 1), ("host", True, 1), ("hbm", True, 1),
                                                 ("host", False, 2), ("host", True, 2), ("hbm", True, 2)])
def test_prefetch_pipeline_matches_sequential(ec, torch, storage, graphs, depth):
    """fwd(j) -> prefetch(j+depth) -> bwd(j) gives the same outputs and final
    rows as the unpipelined fwd/bwd sequence: cold rows updated by bwd(j) that
    batch j+1 already gathered are refreshed; a batch prefetched two ahead
    gathers its host rows only after every earlier write-back."""
    rows, D, B, P = [3000, 800, 50], 8, 128, 3
    dists = [ec.materialize(ec.DistributionSpec.parametric(ec.DistributionKind.zipf, r, 1.0)) for r in rows]
    caches = [d.top_ids(k) for d, k in zip(dists, [30, 10, 5])]
    n = B * P
    offs = np.arange(len(rows) + 1, dtype=np.int64) * n
    nb = 6
    batches = [make_ids(ec, torch, dists, [n] * len(rows), 500 + j)[0] for j in range(nb)]
    grads = [torch.randn(B, len(rows) * D, device="cuda") for _ in range(nb)]

    def run(pipelined):
        tab = ec.EmbeddingTables(rows, D, storage=storage, max_lookups_per_table=n, max_batch_size=B)
        tab.use_graphs(graphs)
        tab.init_synthetic(4, 0.2)
        tab.place_cache(caches)
        outs = []
        for j in range(nb):
            o = tab.forward(batches[j], offs, B, P)
            outs.append(o.clone())
            if pipelined:
                # keep `depth` batches in flight: after batch 0, prefetch up to j+depth
                for k in range(j + 1 if j == 0 else j + depth, min(nb, j + depth + 1)):
                    tab.prefetch(batches[k], offs, B, P)
            tab.backward(grads[j], 0.5)
        torch.cuda.synchronize()
        final = [tab.read_rows(t, np.arange(rows[t])) for t in range(len(rows))]
        st = tab.stats(per_table=True)
        tab.close()
        return [o.cpu().numpy() for o in outs], final, st

    def body():
        o1, f1, s1 = run(False)
        o2, f2, s2 = run(True)
        # both runs sum gradients with float atomics (order-of-summation
        # noise compounds over the steps); a stale prefetched row would be
        # off by lr*grad = O(0.1), five orders above this bound
        for a, b in zip(o1, o2):
            np.testing.assert_allclose(b, a, rtol=RTOL, atol=1e-5 * np.abs(a).max())
        for a, b in zip(f1, f2):
            np.testing.assert_allclose(b, a, rtol=RTOL, atol=1e-5 * np.abs(a).max())
        assert (s1["miss_per_table"] == s2["miss_per_table"]).all()

    if graphs:
        with torch.cuda.stream(torch.cuda.Stream()):
            body()
    else:
        body()


def test_skew_sweep_distributions(ec, torch, ref):
    """BASELINE configs[3] distributions at small scale: uniform, Zipf 0.8/1.2
    and a power law over a permuted id space (non-identity rank -> id map in
    the sampler and in top-k placement); ids bit-exact vs the reference
    sampler, counts vs the reference, sets vs the oracle."""
    rows, D, B, P = [5000, 20000, 3000, 800], 8, 256, 4
    rng = np.random.default_rng(7)
    dists, rdists = [], []
    for t, r in enumerate(rows):
        if t == 0:
            p = np.full(r, 1.0 / r)
        elif t == 3:
            w = np.arange(1, r + 1, dtype=np.float64) ** -0.95
            p = np.empty(r)
            p[rng.permutation(r)] = w / w.sum()
        else:
            a = 0.8 if t == 1 else 1.2
            w = np.arange(1, r + 1, dtype=np.float64) ** -a
            p = w / w.sum()
        dists.append(ec.EmbeddingDistribution.from_probabilities(p))
        rdists.append(ref.RefDist.from_probs(p))
    caches = [d.top_ids(len(d) // 10) for d in dists]
    for d, rd, c in zip(dists, rdists, caches):
        assert (c == rd.top_ids(len(c))).all()  # placement == reference top_ids
    tab = ec.EmbeddingTables(rows, D, max_lookups_per_table=B * P, max_batch_size=B)
    tab.init_synthetic(11, 0.3)
    tab.place_cache(caches)
    ids, offs = make_ids(ec, torch, dists, [B * P] * len(rows), 4242)
    ids_h = ids.cpu().numpy().view(np.uint32)
    for t, rd in enumerate(rdists):
        want = ref.ref_sample_batch(rd, B, P, ec.substream_seed(4242, t))
        assert (ids_h[offs[t]:offs[t + 1]] == want).all(), f"table {t}: sampler ids"
    out = tab.forward(ids, offs, B, P)
    check_batch(ec, tab, ids_h, offs, caches, rows, D, 11, 0.3, P=P, B=B, out=out, ref=ref)
    tab.close()


@pytest.mark.parametrize("mode,n_max", [("cluster", 700), ("cluster", 8192), ("cluster", 16384), ("cluster", 32768),
                                        ("cluster", 65536), ("table", 700), ("table", 9000), ("table", 16384)])
def test_cluster_dedup_every_width(ec, torch, ref, mode, n_max):
    """The cluster kernel at every positions-per-thread width (1..16): tiny
    tables (direct-mapped local set, thousands of repeats of 3 ids), mid-size
    tables (local hash), a 10M-row table, ragged per-table counts and an empty
    table; sets, inverse and hit/miss vs the oracle, counts vs the reference."""
    rows = [3, 24, 5000, 13000, 142572, 10131227, 1000]
    rng = np.random.default_rng(n_max)
    n = [n_max, int(rng.integers(1, n_max)), n_max, 0, int(rng.integers(1, n_max)), n_max, 17]
    dists = [ec.materialize(ec.DistributionSpec.parametric(ec.DistributionKind.zipf, r, 1.05)) for r in rows]
    caches = [d.top_ids(k) for d, k in zip(dists, [1, 0, 100, 5, 1000, 20000, 999])]
    D, B = 8, 1
    offs = np.concatenate([[0], np.cumsum(n)]).astype(np.int64)
    # CSR: one bag per table holding all of its lookups
    bag = np.concatenate([[0], offs[1:]]).astype(np.int64)
    tab = ec.EmbeddingTables(rows, D, max_lookups_per_table=n_max, max_batch_size=B)
    tab.dedup_mode(mode)
    tab.init_synthetic(4, 0.5)
    tab.place_cache(caches)
    ids, _ = make_ids(ec, torch, dists, n, 900 + n_max)
    bag_t = torch.from_numpy(bag).cuda()
    for rep in range(2):  # the second batch sees a clean hash
        out = tab.forward(ids, offs, B, bag_offsets=bag_t)
        check_batch(ec, tab, ids.cpu().numpy().view(np.uint32), offs, caches, rows, D, 4, 0.5, bag_offs=bag, B=B,
                    ref=ref)  # (one bag of up to 64K rows: pooled sums are covered by the other tests)
        tab.backward(torch.zeros(B, len(rows) * D, device="cuda"), 0.0)
    tab.close()


def test_copy_async_and_prefetch_drop(ec, torch):
    """ec_copy_async moves pinned host ids to the device in stream order; a
    dropped prefetch frees its set and the next forward recomputes the batch."""
    rows, D, B = [500, 40], 8, 64
    dists = [ec.materialize(ec.DistributionSpec.parametric(ec.DistributionKind.zipf, r, 1.05)) for r in rows]
    ids, offs = make_ids(ec, torch, dists, [B] * 2, 31)
    host = ids.cpu().pin_memory()
    dev = torch.empty_like(ids)
    s = torch.cuda.Stream()
    ec.copy_async(dev, host, s)
    s.synchronize()
    assert torch.equal(dev, ids)
    with pytest.raises(ec.ValidationError):
        ec.copy_async(dev[:-1], host, s)
    tab = ec.EmbeddingTables(rows, D, max_lookups_per_table=B, max_batch_size=B)
    tab.init_synthetic(1, 0.1)
    ref_out = tab.forward(ids, offs, B, 1).clone()
    ids2, _ = make_ids(ec, torch, dists, [B] * 2, 32)
    tab.prefetch(ids2, offs, B, 1)
    tab.prefetch(ids, offs, B, 1)
    with pytest.raises(ec.ValidationError):
        tab.prefetch(ids2, offs, B, 1)  # two batches already pending
    tab.prefetch_drop()
    out = tab.forward(ids, offs, B, 1)  # recomputed, not consumed out of order
    torch.cuda.synchronize()
    assert torch.equal(out, ref_out)
    u, _ = O.dedup(ids.cpu().numpy().view(np.uint32)[:B])
    assert (tab.export_unique(0) == u).all()
    tab.close()


@pytest.mark.parametrize("nbytes,offset", [(1, 0), (15, 0), (16, 0), (17, 0), (1000, 4), (1703936, 0),
                                           (1703939, 0), (4096, 8)])
def test_copy_async_pull_and_fallback(ec, torch, nbytes, offset):
    """Pinned host -> device runs as the SM pull kernel (16-byte aligned ends:
    int4 body + byte tail), misaligned ones and device -> host through the
    copy engine; every path is byte-exact."""
    g = torch.Generator().manual_seed(nbytes)
    src = torch.randint(0, 256, (nbytes + offset,), dtype=torch.uint8, generator=g).pin_memory()
    dst = torch.zeros(nbytes + offset, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    ec.copy_async(dst[offset:], src[offset:], s, pull_ctas=8)
    s.synchronize()
    assert torch.equal(dst[offset:].cpu(), src[offset:])
    assert int(dst[:offset].sum()) == 0  # nothing written before the destination
    back = torch.zeros(nbytes, dtype=torch.uint8).pin_memory()
    ec.copy_async(back, dst[offset:], s, pull_ctas=8)  # device -> host: copy engine
    s.synchronize()
    assert torch.equal(back, src[offset:])
