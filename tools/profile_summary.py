"""Summarise ncu outputs into profiles/ (committed evidence).

usage: python tools/profile_summary.py <launches.csv> <full.ncu-rep> <out_prefix>
writes <out_prefix>_launches.md (per-kernel device time from the launch list:
serialized, cold-cache — compare shares), <out_prefix>_ncu_full.md (key raw
metrics per profiled kernel) and <out_prefix>_traffic.json (dram bytes per
launch by kernel, read by bench.py for roofline.traffic)."""
import collections
import csv
import io
import json
import subprocess
import sys

launches, rep, prefix = sys.argv[1:4]

rows = list(csv.reader(open(launches)))
hdr = None
agg = collections.defaultdict(list)
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            name = d["Kernel Name"].split("(")[0].replace("void ", "")
            agg[name].append(float(d["Metric Value"].replace(",", "")))
step_kernels = {k: v for k, v in agg.items() if not any(s in k for s in ("init_shard", "fill_cache", "set_remap",
                                                                           "sample_stream", "FillFunctor", "Fill", "spin_kernel",
                                                                           "direct_copy", "arange", "k_classify",
                                                                           "k_stable_order", "k_scan_", "k_gather_batch",
                                                                           "k_h2d_pull", "k_spin_ns"))}
tot = sum(sum(v) / len(v) for v in step_kernels.values()) or 1.0
with open(prefix + "_launches.md", "w") as f:
    f.write(f"# ncu launch list summary ({launches})\n\n")
    f.write("`ncu --metrics gpu__time_duration.sum --clock-control none` over `bench.py --steps 3 --warmup 3`.\n")
    f.write("Serialised, cold-cache per-launch times: compare shares, not absolutes.\n\n")
    f.write("| kernel | launches | mean ns | min ns | share of step kernels |\n|---|---|---|---|---|\n")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]) / len(kv[1])):
        m = sum(v) / len(v)
        share = (f"{100 * m / tot:.1f}%" if k in step_kernels else
                 "e2e input copy (not a step kernel)" if "k_h2d_pull" in k else
                 "prefetch delay (a one-warp device wait, not work)" if "k_spin_ns" in k else "setup")
        f.write(f"| `{k}` | {len(v)} | {m:.0f} | {min(v):.0f} | {share} |\n")

raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
h, units = rr[0], rr[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sectors_srcunit_tex_op_atom.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
idx = {w: h.index(w) for w in want if w in h}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
traffic = collections.defaultdict(list)
with open(prefix + "_ncu_full.md", "w") as f:
    f.write(f"# ncu --set full summary ({rep})\n\n")
    f.write("| kernel | " + " | ".join(f"{w} [{units[idx[w]]}]" for w in idx) + " |\n")
    f.write("|---|" + "---|" * len(idx) + "\n")
    for r in rr[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "")
        f.write(f"| `{name}` | " + " | ".join(r[i] for i in idx.values()) + " |\n")
        b = 0.0
        for w in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            if w in idx:
                b += float(r[idx[w]].replace(",", "")) * scale.get(units[idx[w]], 1)
        traffic[name.split("<")[0].replace("ec::", "")].append(b)
json.dump({k: sum(v) / len(v) for k, v in traffic.items()}, open(prefix + "_traffic.json", "w"), indent=1)
print("wrote", prefix + "_launches.md", prefix + "_ncu_full.md", prefix + "_traffic.json")
