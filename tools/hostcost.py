"""Host enqueue cost per pipelined step vs GPU time per step.
usage: python tools/hostcost.py [workload] [steps]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2411_01611_b200 as ec  # noqa: E402

wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "kaggle"]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
torch.cuda.set_device(0)
st = torch.cuda.Stream(priority=-1)
torch.cuda.set_stream(st)
tab, dists, caches, ks = bench.build_tables(ec, torch, wl, 0, 1, 0)
ids, offs = bench.gen_batches(ec, torch, dists, wl, 0, bench.N_BATCHES)
T, D, B, P = len(wl["rows"]), wl["dim"], wl["batch"], wl["pooling"]
out = torch.empty((B, T * D), dtype=torch.float32, device="cuda")
NB = bench.N_BATCHES
cs = torch.cuda.Stream()  # input stream (as in bench.py)
parts = {"forward": [], "prefetch": [], "backward": [], "wait": []}


def step(j, rec=False):
    t0 = time.perf_counter()
    o = tab.forward(ids[j % NB], offs, B, P, out=out)
    t1 = time.perf_counter()
    tab.prefetch(ids[(j + 1) % NB], offs, B, P, stream=cs)
    t2 = time.perf_counter()
    tab.backward(o, bench.LR)
    t3 = time.perf_counter()
    tab.prefetch_wait()
    t4 = time.perf_counter()
    if rec:
        for k, a, b in (("forward", t0, t1), ("prefetch", t1, t2), ("backward", t2, t3), ("wait", t3, t4)):
            parts[k].append((b - a) * 1e6)


for j in range(20):
    step(j)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
h0 = time.perf_counter()
ev[0].record(st)
for j in range(steps):
    step(j, True)
    ev[j + 1].record(st)
h1 = time.perf_counter()
torch.cuda.synchronize()
g = [ev[j].elapsed_time(ev[j + 1]) * 1e3 for j in range(steps)]
print(f"{sys.argv[1:]}: host enqueue {1e6 * (h1 - h0) / steps:.1f} us/step; GPU back-to-back {np.mean(g):.1f} us/step "
      f"(median {np.median(g):.1f}, p90 {np.percentile(g, 90):.1f})")
for k, v in parts.items():
    print(f"  host {k:9s} mean {np.mean(v):6.1f} us  median {np.median(v):6.1f}")
tab.close()
