"""Per-kernel timeline of pipelined bench steps (profiling on: direct launches,
CUDA events on each kernel's own stream).  usage: python tools/timeline.py [workload] [steps] [prefetch depth]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2411_01611_b200 as ec  # noqa: E402

wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "kaggle"]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
depth = int(sys.argv[3]) if len(sys.argv) > 3 else (2 if wl["storage"] == "host" else 1)
torch.cuda.set_device(0)
torch.cuda.set_stream(torch.cuda.Stream())
tab, dists, caches, ks = bench.build_tables(ec, torch, wl, 0, 1, 0)
ids, offs = bench.gen_batches(ec, torch, dists, wl, 0, bench.N_BATCHES)
T, D, B, P = len(wl["rows"]), wl["dim"], wl["batch"], wl["pooling"]
out = torch.empty((B, T * D), dtype=torch.float32, device="cuda")
flush = torch.empty(bench.FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
NB = bench.N_BATCHES
cs = torch.cuda.Stream()  # input stream (as in bench.py): prefetches order after it only


def step(j, first=False):
    o = tab.forward(ids[j % NB], offs, B, P, out=out)
    for k in (range(1, depth + 1) if first else [depth]):
        tab.prefetch(ids[(j + k) % NB], offs, B, P, stream=cs)
    tab.backward(o, bench.LR)
    tab.prefetch_wait()


for j in range(4):
    step(j, first=j == 0)
torch.cuda.synchronize()
tab.profile(True)
tab.profile_timeline()
for j in range(4, 4 + steps):
    flush.fill_(float(j))
    step(j)
torch.cuda.synchronize()
tl = tab.profile_timeline()
tab.profile(False)
if os.environ.get("TL_ALL"):
    for k, s0, e0 in sorted(tl, key=lambda r: r[1]):
        print(f"  {k:22s} {1e3 * s0:9.1f} .. {1e3 * e0:9.1f} us")
# step boundaries: each step's pool starts its forward
starts = [s for (k, s, e) in tl if k == "k_pool"]
for i in range(len(starts) - 2, len(starts)):
    a = starts[i]
    b = starts[i + 1] if i + 1 < len(starts) else max(e for _, _, e in tl)
    print(f"--- step {i}: pool start {a:.3f} ms")
    for k, s, e in sorted(tl, key=lambda r: r[1]):
        if a - 0.2 <= s < b:
            print(f"  {k:22s} {1e3 * (s - a):8.1f} .. {1e3 * (e - a):8.1f} us  ({1e3 * (e - s):6.1f})")
tab.close()
