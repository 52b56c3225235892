"""Regenerate tests/golden/reference_vectors.json from the compiled reference.

Run here (where /root/reference exists and oracle/_ref is built):
    python tests/golden/make_golden.py
Every value is produced by the UNMODIFIED reference core through
oracle/ref_shim.cpp; the GPU box only reads the committed JSON.
"""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_vectors.json")


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    g = {"generator": "tests/golden/make_golden.py via oracle/_ref/libembcomm_ref.so (reference core)"}

    # 1. sampler streams: sample_batch (core/src/simulator.cpp:132-143)
    samp = []
    for kind, size, shape, b, d, seed in [("zipf", 64, 1.0, 100, 3, 99), ("zipf", 1000, 1.0, 64, 3, 7),
                                          ("exponential", 500, 5.0, 33, 2, 12345),
                                          ("half_normal", 256, 0.3, 17, 5, 2024)]:
        dist = O.RefDist.parametric(kind, size, shape)
        ids = O.ref_sample_batch(dist, b, d, seed)
        samp.append({"kind": kind, "size": size, "shape": shape, "b": b, "d": d, "seed": seed,
                     "ids": ids.tolist()})
    rng = np.random.default_rng(3)
    p = rng.random(40)
    p /= p.sum()
    dist = O.RefDist.from_probs(p)
    samp.append({"probs": p.tolist(), "b": 50, "d": 2, "seed": 5, "ids": O.ref_sample_batch(dist, 50, 2, 5).tolist()})
    g["sample_batch"] = samp

    # 2. large-vocab stream (81,920 draws at zipf(1M, 1.05)), pinned by digest
    dist = O.RefDist.parametric("zipf", 1_000_000, 1.05)
    ids = O.ref_sample_batch(dist, 4096, 20, O.ref_substream_seed(20241101, 0))
    g["zipf1m_stream"] = {"size": 1_000_000, "shape": 1.05, "b": 4096, "d": 20,
                          "rng_seed": O.ref_substream_seed(20241101, 0), "sha256": digest(ids),
                          "head": ids[:64].tolist()}

    # 3. simulate_epoch(dist, …) (simulator.cpp:169-220)
    sims = []
    for kind, size, shape, q, b, d, k, epochs, seed in [
            ("zipf", 16, 1.0, 100, 10, 2, 16, 3, 1),
            ("zipf", 256, 1.0, 10000, 100, 2, 0, 20, 77),
            ("half_normal", 256, 0.3, 10000, 128, 4, 64, 20, 808),
            ("exponential", 128, 5.0, 5000, 64, 3, 10, 5, 31337),
            ("zipf", 100000, 1.05, 20000, 4096, 1, 1000, 2, 424242),
            ("zipf", 1000, 1.2, 777, 50, 3, 25, 2, 9)]:
        dist = O.RefDist.parametric(kind, size, shape)
        r = O.ref_simulate_epoch(dist, q, b, d, dist.top_ids(k), epochs, seed)
        sims.append({"kind": kind, "size": size, "shape": shape, "q": q, "b": b, "d": d, "k": k,
                     "epochs": epochs, "seed": seed, "result": r})
    g["simulate_epoch"] = sims

    # 4. measure_unique (simulator.cpp:145-167)
    mus = []
    for kind, size, shape, b, trials, seed in [("zipf", 32, 1.0, 16, 4, 1234), ("zipf", 1000, 1.0, 256, 200, 20240817),
                                               ("exponential", 4096, 100.0, 1024, 50, 5)]:
        dist = O.RefDist.parametric(kind, size, shape)
        mus.append({"kind": kind, "size": size, "shape": shape, "b": b, "trials": trials, "seed": seed,
                    "result": O.ref_measure_unique(dist, b, trials, seed)})
    g["measure_unique"] = mus

    # 5. trace replay known answer (tests/test_simulator.cpp:156-172) + a larger trace
    g["trace_kat"] = {"ids": [0, 1, 0, 2, 1, 1, 3, 3], "d": 2, "vocab": 4, "b": 2, "cache": [0, 1],
                      "result": O.ref_simulate_trace([0, 1, 0, 2, 1, 1, 3, 3], 2, 4, 2, [0, 1])}
    dist = O.RefDist.parametric("zipf", 500, 1.1)
    tids = O.ref_sample_batch(dist, 3000, 4, 77)
    cache = dist.top_ids(40)
    order, sizes, nh = O.ref_build_schedule(tids, 4, 500, cache, 128)
    g["trace_large"] = {"kind": "zipf", "size": 500, "shape": 1.1, "b_gen": 3000, "d": 4, "seed": 77,
                        "cache_k": 40, "batch": 128, "result": O.ref_simulate_trace(tids, 4, 500, 128, cache),
                        "hot": O.ref_classify_samples(tids, 4, 500, cache).tolist(),
                        "schedule_order": order.tolist(), "n_hot_batches": nh}

    # 6. per-(table, batch) M1 counts at config-1 shape: 2 tables x n = 81,920
    segs = []
    for t in range(2):
        seed_t = O.ref_substream_seed(1105, t)
        ids = O.ref_sample_batch(dist := O.RefDist.parametric("zipf", 1_000_000, 1.05), 4096, 20, seed_t)
        for k in (0, 1000, 50000):
            a, nc = O.ref_segment_counts(ids, [0, ids.size], [1_000_000], [dist.top_ids(k)])
            segs.append({"table": t, "rng_seed": seed_t, "k": k, "unique": int(a[0]), "non_cached": int(nc[0]),
                         "sha256": digest(ids)})
    g["m1_counts"] = segs

    # 7. cost model / planner values (cost_model.cpp, cache_planner.cpp)
    dz = O.RefDist.parametric("zipf", 1_000_000, 1.05)
    cm = {"expected_unique_zipf1m_81920": O.ref_cost("expected_unique_from_rank", dz, 81920, 0),
          "cached_zipf1m_k10000": O.ref_cost("cached_epoch_cost", dz, 4096 * 100, 4096, 20, dz.top_ids(10000)),
          "presence": [[p, b, O.ref_cost("batch_presence_prob", p, b)]
                       for p, b in [(0.0, 100), (1.0, 1), (0.5, 2), (1e-15, 1000), (0.3, 7), (1e-6, 81920)]]}
    z32 = O.RefDist.parametric("zipf", 32, 1.0)
    cm["planner_zipf32"] = O.ref_plan(z32, 2048, 2, 8, 1.0, 10000, 4, search=False)
    cm["planner_zipf32"]["cached_ids"] = cm["planner_zipf32"]["cached_ids"].tolist()
    big = O.ref_plan(O.RefDist.parametric("zipf", 200000, 1.05), 8_000_000, 300, 64, 0.9, 1_000_000, 26)
    big["cached_ids"] = digest(big["cached_ids"])
    cm["planner_zipf200k"] = big
    g["cost_model"] = cm

    with open(OUT, "w") as f:
        json.dump(g, f, indent=0)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
