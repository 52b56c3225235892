"""bench.py's contract, run for real on the GPU: one JSON line with the keys the
driver reads (N=1), and the N>1 path under torchrun -- two ranks sharing the
one GPU over the peer-memory exchange (gloo plumbing; a functional check of
the multi-rank bench path, its timings are not per-GPU)."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "roofline", "clocks"}


def _json_lines(out):
    return [json.loads(x) for x in out.splitlines() if x.startswith("{")]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_bench_single_gpu_line():
    r = subprocess.run([sys.executable, "bench.py", "--steps", "3", "--warmup", "3", "--no-cpu-baseline",
                        "--schedule-batches", "0", "--workload", "kaggle_hbm"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1
    d = lines[0]
    assert KEYS <= set(d), KEYS - set(d)
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["value"] > 0
    assert {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= set(d["e2e"])
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(d["roofline"])
    assert d["gpu_launches"] > 0
    assert d["gather_roofline"]["kernel"] in ("k_pool", "k_gather") and d["gather_roofline"]["frac"] > 0
    assert d["comm"]["expected_model_rows_per_batch"] > 0
    assert len(d["comm"]["model_rows_per_table_batch0"]) == 26


def _first_traceback(err):
    i = err.find("Traceback")
    return err[i:i + 4000] if i >= 0 else err[-3000:]


def test_bench_two_ranks_peer_exchange():
    # Two ranks time-slice one GPU beside this process's own context, so a
    # launch can be slow; one retry (fresh port) before the failure is reported.
    errs = []
    for _ in range(2):
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
               "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2", "--steps",
               "3", "--warmup", "3", "--no-cpu-baseline", "--schedule-batches", "0", "--workload", "kaggle_hbm"]
        r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
        if r.returncode == 0:
            break
        errs.append(_first_traceback(r.stderr))
    assert r.returncode == 0, "\n----\n".join(errs)
    lines = _json_lines(r.stdout)
    assert len(lines) == 1  # rank 0 only
    d = lines[0]
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert "p2p exchange" in d["config"]["parallelism"]
