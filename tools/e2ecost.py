"""Host time per call in bench.py's e2e loop (pinned H2D of ids, forward,
prefetch, backward, async stats).  usage: python tools/e2ecost.py [workload] [steps]"""
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
NB, NS = bench.N_BATCHES, 6
DEPTH = int(os.environ.get("E2E_DEPTH", "2" if wl["storage"] == "host" else "1"))
LA = DEPTH + 2
PULL = int(os.environ.get("E2E_PULL", "8"))
cs = torch.cuda.Stream(priority=int(os.environ.get("E2E_CSPRIO", "0")))
host_ids = ids.cpu().pin_memory()
dev_ids = [torch.empty_like(ids[0]) for _ in range(NS)]
copied = [torch.cuda.Event() for _ in range(NS)]
consumed = [torch.cuda.Event() for _ in range(NS)]
acc = {}
lib = ec._native.lib()
nbytes = ids[0].numel() * 4
dptr = [t.data_ptr() for t in dev_ids]
hptr = [t.data_ptr() for t in host_ids]


def tick(name, t0):
    t1 = time.perf_counter()
    acc.setdefault(name, []).append((t1 - t0) * 1e6)
    return t1


def h2d(k):
    if k >= NS:
        cs.wait_event(consumed[k % NS])
    if PULL:
        lib.ec_copy_async_pull(dptr[k % NS], hptr[k % NB], nbytes, PULL, cs.cuda_stream)
    else:
        lib.ec_copy_async(dptr[k % NS], hptr[k % NB], nbytes, cs.cuda_stream)
    copied[k % NS].record(cs)


DO_H2D = os.environ.get("E2E_H2D", "1") == "1"
READY = os.environ.get("E2E_READY", "1") == "1"
ready = torch.cuda.Stream()


def pf(k):
    if READY:
        ready.wait_event(copied[k % NS])
        tab.prefetch(dev_ids[k % NS], offs, B, P, stream=ready)
    else:
        tab.prefetch(dev_ids[k % NS], offs, B, P, stream=cs)
DO_STATS = os.environ.get("E2E_STATS", "1") == "1"


def run(n, rec):
    tab.prefetch_drop()
    for k in range(min(n, LA)):
        h2d(k)
    for k in range(min(n, DEPTH)):
        pf(k)
    for k in range(n):
        t = time.perf_counter()
        st.wait_event(copied[k % NS])
        t = tick("wait_copy", t) if rec else t
        o = tab.forward(dev_ids[k % NS], offs, B, P, out=out)
        t = tick("forward", t) if rec else t
        consumed[k % NS].record(st)
        if DEPTH and k + DEPTH < n:
            pf(k + DEPTH)
        t = tick("prefetch", t) if rec else t
        if k + LA < n and DO_H2D:
            h2d(k + LA)
        t = tick("h2d", t) if rec else t
        tab.backward(o, bench.LR)
        t = tick("backward", t) if rec else t
        if DO_STATS:
            tab.stats_enqueue(k % 4)
        t = tick("stats_enqueue", t) if rec else t
        if k >= 2 and DO_STATS:
            tab.stats_collect((k - 2) % 4)
        t = tick("stats_collect", t) if rec else t
    tab.prefetch_wait()
    torch.cuda.synchronize()


BG = os.environ.get("E2E_BG", "")  # background H2D copies beside the steps: "ce" or "pull"
bgs = torch.cuda.Stream()
bg_dev = torch.empty_like(ids[0])


def background(n):
    for k in range(n):
        if BG == "ce":
            lib.ec_copy_async(bg_dev.data_ptr(), hptr[k % NB], nbytes, bgs.cuda_stream)
        elif BG == "pull":
            lib.ec_copy_async_pull(bg_dev.data_ptr(), hptr[k % NB], nbytes, 16, bgs.cuda_stream)


tab.backward(tab.forward(ids[0], offs, B, P, out=out), bench.LR)  # geometry for the first prefetch
run(24, False)
if BG:
    torch.cuda.synchronize()
    bg0 = torch.cuda.Event(enable_timing=True)
    bg1 = torch.cuda.Event(enable_timing=True)
    bg0.record(bgs)
    background(steps)
    bg1.record(bgs)
t0 = time.perf_counter()
run(steps, True)
t1 = time.perf_counter()
if BG:
    torch.cuda.synchronize()
    print(f"background {BG}: {steps} copies in {bg0.elapsed_time(bg1) * 1e3 / steps:.1f} us each")
print(f"{sys.argv[1:]} bg={BG} h2d={DO_H2D} stats={DO_STATS} depth={DEPTH} pull={PULL} cs_prio={cs.priority} ready={READY}: e2e wall {1e6 * (t1 - t0) / steps:.1f} us/step")
for k, v in acc.items():
    print(f"  {k:14s} mean {np.mean(v):7.1f}  median {np.median(v):7.1f}  p90 {np.percentile(v, 90):7.1f}")
tab.close()
