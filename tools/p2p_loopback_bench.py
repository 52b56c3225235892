"""Peer-memory exchange on one GPU: W ranks of a row-sharded job in one process
(ec_group_set_p2p), each with its own batch, stepped through the same kernels a
one-process-per-GPU job runs over NVLink (remote-row loads in the gather,
owner updates by atomics or inboxes, owner-partitioned hot-row sync, device barriers).
On one GPU the W ranks' kernels share the SMs and the "remote" traffic is
local HBM, so this is a functional and overhead probe, not a scaling number.

usage: python tools/p2p_loopback_bench.py [workload] [world] [steps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2411_01611_b200 as ec  # noqa: E402

wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "kaggle_hbm"]
W = int(sys.argv[2]) if len(sys.argv) > 2 else 2
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
torch.cuda.set_device(0)
torch.cuda.set_stream(torch.cuda.Stream())
rows, D, B, P = wl["rows"], wl["dim"], wl["batch"], wl["pooling"]
T = len(rows)
dists = [bench.make_dist(ec, wl, r, t) for t, r in enumerate(rows)]
budget = wl["cache_bytes"] // (D * 4)
ks = ec.place_topk_global(dists, budget) if budget else [0] * T
caches = [d.top_ids(k) for d, k in zip(dists, ks)]


def group(p2p):
    ms = [ec.EmbeddingTables(rows, D, storage=wl["storage"], rank=r, world=W, max_lookups_per_table=B * P,
                             max_batch_size=B) for r in range(W)]
    for m in ms:
        m.init_synthetic(bench.SEED, 0.05)
    g = ec.EmbeddingGroup(ms, p2p=p2p)
    for m in ms:
        m.place_cache(caches)
    return ms, g


ids = [bench.gen_batches(ec, torch, dists, wl, r, 4)[0] for r in range(W)]
offs = np.arange(T + 1, dtype=np.int64) * (B * P)
for p2p in (False, True):
    ms, g = group(p2p)
    st = torch.cuda.current_stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for k in range(steps + 3):
        if k == 3:
            torch.cuda.synchronize()
            ev[0].record(st)
        outs = g.forward([ids[r][k % 4] for r in range(W)], offs, B, P)
        g.backward(outs, bench.LR)
    ev[1].record(st)
    torch.cuda.synchronize()
    ms_step = ev[0].elapsed_time(ev[1]) / steps
    sts = [m.stats() for m in ms]
    wire = sum(x["wire_rows"] for x in sts)
    hot = max(x.get("hot_sync_bytes", 0) for x in sts)
    print(f"{wl['name']}: world {W} on one GPU, {'p2p' if p2p else 'staged copies'}: "
          f"{ms_step:.3f} ms per group step ({ms_step / W:.3f} ms per rank-step), remote rows {wire}, "
          f"max hot-sync bytes per rank {hot}")
    g.close()
    for m in ms:
        m.close()
