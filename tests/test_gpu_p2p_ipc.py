"""Multi-process peer-memory exchange through CUDA IPC (ec_tables_p2p_export /
import), two processes on one B200: the path a one-process-per-GPU job takes
over NVLink, minus the link.  Both ranks' pooled outputs and the owners' /
replicas' rows after two forward+backward steps must match the in-process
loopback group (same routing and rank-ordered hot-row updates; fp32 atomics
reorder non-hot sums, hence the 1e-5 bound).  The processes meet at device-side
barriers only, so a missing signal shows up as the join timeout below."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ROWS, D, B, P, SEED, LR = [5000, 37, 20000], 16, 64, 5, 7, 0.25
STEPS = 3
PROBE = 400  # rows per table read back at the end


def _atol(x):
    """fp32 sums in a different order: the absolute bound scales with the values."""
    return 1e-6 * max(1.0, float(np.abs(x).max()))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _setup(ec, rank, world, storage):
    n = B * P
    dists = [ec.materialize(ec.DistributionSpec.parametric(ec.DistributionKind.zipf, r, 1.05)) for r in ROWS]
    caches = [d.top_ids(min(len(d), k)) for d, k in zip(dists, [40, 3, 200])]
    m = ec.EmbeddingTables(ROWS, D, storage=storage, rank=rank, world=world, max_lookups_per_table=n, max_batch_size=B)
    m.init_synthetic(SEED, 0.1)
    return m, dists, caches


def _batch(ec, torch, dists, rank, step, repeat=False):
    """repeat: the same ids every step (every cold row a step reads was updated
    by the step before: a prefetch read before the barrier is always stale)."""
    n = B * P
    ids = torch.empty(len(dists) * n, dtype=torch.int32, device="cuda")
    for t, d in enumerate(dists):
        ec.DiscreteSampler(d).sample_into(ids.data_ptr() + 4 * n * t,
                                          ec.substream_seed(ec.substream_seed(100 + (0 if repeat else step), rank), t),
                                          0, n)
    g = torch.Generator(device="cuda").manual_seed(1000 * step + rank)
    grad = torch.randn(B, len(dists) * D, device="cuda", generator=g)
    return ids, grad


def _probe(m, rank, world, caches):
    """This rank's owned rows (first PROBE of each table) and its cache replica."""
    out = []
    for t, r in enumerate(ROWS):
        own = [i for i in range(min(r, PROBE * world)) if i % world == rank][:PROBE]
        out.append(m.read_rows(t, own))
        if len(caches[t]):
            out.append(m.read_rows(t, [int(i) for i in caches[t]]))
    return out


def _worker(rank, port, q, storage, prefetch, repeat, WORLD):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        import paper_2411_01611_b200 as ec
        m, dists, caches = _setup(ec, rank, WORLD, storage)
        m.place_cache(caches)
        blobs = [None] * WORLD
        dist.all_gather_object(blobs, m.p2p_export())
        m.p2p_import(blobs)
        dist.barrier()
        offs = np.arange(len(ROWS) + 1, dtype=np.int64) * (B * P)
        outs = []
        batches = [_batch(ec, torch, dists, rank, step, repeat) for step in range(STEPS)]
        for step in range(STEPS):
            ids, grad = batches[step]
            outs.append(m.forward(ids, offs, B, P).cpu().numpy())
            if prefetch and step + 1 < STEPS:  # next batch's dedup overlaps this backward
                m.prefetch(batches[step + 1][0], offs, B, P)
            m.backward(grad, LR)
        torch.cuda.synchronize()
        dist.barrier()
        q.put((rank, outs, _probe(m, rank, WORLD, caches), m.stats()["wire_rows"]))
        dist.barrier()  # keep the exported memory alive until every peer is done
        m.close()
    except Exception as e:  # surfaces in the parent instead of a hang
        q.put((rank, repr(e), None, None))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("storage,prefetch,repeat,WORLD", [("hbm", False, False, 2), ("host", False, False, 2),
                                                           ("hbm", True, False, 2), ("host", True, False, 2),
                                                           ("host", True, True, 2), ("hbm", True, True, 3),
                                                           ("host", True, True, 3)])
def test_p2p_ipc_processes_match_loopback(ec, storage, prefetch, repeat, WORLD):
    import torch
    import torch.multiprocessing as mp
    # expected: the loopback group (staged copies) in this process
    members, dists, caches = zip(*[_setup(ec, r, WORLD, storage) for r in range(WORLD)])
    group = ec.EmbeddingGroup(members)
    for m in members:
        m.place_cache(caches[0])
    offs = np.arange(len(ROWS) + 1, dtype=np.int64) * (B * P)
    want = [[] for _ in range(WORLD)]
    for step in range(STEPS):
        batch = [_batch(ec, torch, dists[0], r, step, repeat) for r in range(WORLD)]
        outs = group.forward([b[0] for b in batch], offs, B, P)
        for r in range(WORLD):
            want[r].append(outs[r].cpu().numpy())
        group.backward([b[1] for b in batch], LR)
    torch.cuda.synchronize()
    want_rows = [_probe(members[r], r, WORLD, caches[0]) for r in range(WORLD)]
    group.close()
    for m in members:
        m.close()

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q, storage, prefetch, repeat, WORLD)) for r in range(WORLD)]
    for p in procs:
        p.start()
    got = {}
    try:
        for _ in range(WORLD):
            rank, outs, rows, wire = q.get(timeout=300)
            assert rows is not None, f"rank {rank}: {outs}"
            got[rank] = (outs, rows, wire)
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    for r in range(WORLD):
        outs, rows, wire = got[r]
        for s in range(STEPS):
            np.testing.assert_allclose(outs[s], want[r][s], rtol=1e-5, atol=_atol(want[r][s]))
        for a, b in zip(rows, want_rows[r]):
            np.testing.assert_allclose(a, b, rtol=1e-5, atol=_atol(b))
        assert wire > 0
