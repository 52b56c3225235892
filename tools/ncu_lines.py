"""Per-source-line warp-stall samples of one kernel (ncu --print-source cuda,sass).
usage: python tools/ncu_lines.py report.ncu-rep kernel_regex [top]"""
import csv, io, subprocess, sys, collections
rep, pat = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", "regex:" + pat,
                      "-c", "1"], capture_output=True, text=True).stdout
agg = collections.Counter()
src_of = {}
fname = "?"
hdr = None
cur_line = "?"
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 5:
        continue
    try:
        s = int(r[4] or 0)
    except ValueError:
        continue
    if r[0].strip():
        cur_line = r[0]
    key = (fname, cur_line)
    agg[key] += s
    if r[1].strip():
        src_of[key] = r[1].strip()
tot = sum(agg.values()) or 1
print(f"samples={tot}")
for (f, l), s in agg.most_common(top):
    print(f"{100*s/tot:5.1f}%  {f}:{l}  {src_of.get((f, l), '')[:100]}")
