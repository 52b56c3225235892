"""Multi-rank host logic on CPU: world-size-2 gloo process groups (no GPU).

Covers what the N>1 path does on the host: the NCCL unique-id bootstrap
through torch.distributed, the row-shard layout (owner(id) = id % world), and
the per-batch exchange plan computed by the library (ec_exchange_plan) from the
all-gathered request matrix — checked for send/receive symmetry across real
processes, with the request counts coming from the oracle's dedup of each
rank's own batch and the wire model checked against the compiled reference.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle as O
        import paper_2411_01611_b200 as ec
        res = {}
        # 1. NCCL unique-id bootstrap exactly as bench.py does it
        uid = [ec.EmbeddingTables.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ids = [None] * world
        dist.all_gather_object(ids, uid[0])
        res["uid_same"] = all(x == ids[0] for x in ids) and len(ids[0]) == 128

        # 2. shard layout: every row owned exactly once
        rows = [1460, 583, 10131, 3, 1, 27, 7]
        local = torch.tensor(ec.shard_rows(rows, world, rank), dtype=torch.int64)
        allr = [torch.zeros_like(local) for _ in range(world)]
        dist.all_gather(allr, local)
        res["shard_total"] = torch.stack(allr).sum(0).tolist() == rows

        # 3. exchange plan from a real batch: this rank's misses grouped by owner
        T, n, E = 3, 4096, 50_000
        probs = np.array([(i + 1) ** -1.05 for i in range(E)])
        probs /= probs.sum()
        s = O.Sampler(probs)
        cache_k = 500  # top-500 ids cached (ranks == ids for this Zipf)
        counts = np.zeros(world + 1, np.int32)
        miss_total = own_miss = 0
        for t in range(T):
            seg = s.sample(O.substream_seed(O.substream_seed(77, rank), t), 0, n)
            u, _ = O.dedup(seg)
            miss = u[u >= cache_k]
            miss_total += miss.size
            owners = miss % world
            for o in range(world):
                if o != rank:
                    counts[o] += int((owners == o).sum())
            own_miss += int((owners == rank).sum())
            counts[world] += int((u < cache_k).sum())
            if os.path.exists(O.REF_SO):
                _, nc = O.ref_segment_counts(seg, [0, n], [E], [np.arange(cache_k, dtype=np.uint32)])
                assert int(nc[0]) == miss.size  # model rows == reference embedding units
        mat = [torch.zeros(world + 1, dtype=torch.int32) for _ in range(world)]
        dist.all_gather(mat, torch.from_numpy(counts))
        m = torch.stack(mat).numpy()
        plan = ec.exchange_plan(m, world, rank)
        plans = [None] * world
        dist.all_gather_object(plans, {k: v.tolist() for k, v in plan.items()})
        sym = all(plans[r]["send_cnt"][o] == plans[o]["recv_cnt"][r] for r in range(world) for o in range(world))
        offs = all(plans[r]["send_off"] == list(np.concatenate([[0], np.cumsum(plans[r]["send_cnt"])[:-1]]))
                   for r in range(world))
        res["plan_symmetric"] = sym and offs
        res["wire_rows"] = int(sum(plan["send_cnt"]))
        res["wire_expected"] = miss_total - own_miss
        res["hot_same"] = all(plans[r]["hot_cnt"] == plans[0]["hot_cnt"] for r in range(world))
        out_q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_multirank_host_logic(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r, res in results.items():
        assert res["uid_same"], r
        assert res["shard_total"], r
        assert res["plan_symmetric"], r
        assert res["hot_same"], r
        assert res["wire_rows"] == res["wire_expected"], r


def test_plan_validation():
    import paper_2411_01611_b200 as ec
    with pytest.raises(ec.ValidationError):
        ec.exchange_plan(np.array([[1, 2, 0], [0, 0, 0]]), 2, 0)  # self-request
    with pytest.raises(ec.ValidationError):
        ec.shard_rows([5], 2, 2)
