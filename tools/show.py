"""Print the key numbers of bench JSON lines: python tools/show.py files..."""
import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "unreadable", e)
        continue
    ph = {k: round(v["ms_per_call"] * 1e3, 1) for k, v in (d.get("phases") or {}).items()}
    print(f.split("/")[-1], "ms/step", d.get("ms_per_step"), "e2e ms", (d.get("e2e") or {}).get("ms_per_step"), (d.get("e2e") or {}).get("step_ms_dist"),
          "G/s", round(d["value"] / 1e9, 3), d.get("step_ms_dist"), ph)
