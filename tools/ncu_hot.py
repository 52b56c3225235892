"""Summarise an ncu report: hottest SASS instructions (stall samples) per kernel.
usage: python tools/ncu_hot.py report.ncu-rep kernel_regex [top]"""
import csv, io, re, subprocess, sys

rep, pat = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks = re.split(r'^"Kernel Name",', out, flags=re.M)
seen = set()
for b in blocks[1:]:
    name = b.split("\n", 1)[0]
    if not re.search(pat, name) or name in seen:
        continue
    seen.add(name)
    rows = list(csv.reader(io.StringIO(b.split("\n", 1)[1])))
    hdr = rows[0]
    si = hdr.index("Warp Stall Sampling (All Samples)")
    src = hdr.index("Source")
    data = [(int(r[si] or 0), r[src].strip(), r[0]) for r in rows[1:] if len(r) > si]
    tot = sum(d[0] for d in data) or 1
    print(f"== {name[:110]}  samples={tot}")
    for s, ins, addr in sorted(data, reverse=True)[:top]:
        print(f"  {100*s/tot:5.1f}%  {addr[-5:]}  {ins[:90]}")
