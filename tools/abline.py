"""One summary line of a bench JSON line on stdin: python bench.py ... | python tools/abline.py label"""
import json, sys
lab = " ".join(sys.argv[1:])
try:
    d = json.loads(sys.stdin.read().strip().splitlines()[-1])
    r, g = d.get("roofline") or {}, d.get("gather_roofline") or {}
    print(lab, "ms", d["ms_per_step"], "med", (d.get("step_ms_dist") or {}).get("median"), "e2e", (d.get("e2e") or {}).get("ms_per_step"),
          r.get("kernel"), "GB/s", r.get("achieved"), "frac", r.get("frac"), "gather", g.get("kernel"), g.get("frac"))
except Exception as e:  # noqa: BLE001
    print(lab, "unreadable", e)
