import csv,collections,sys
rows=list(csv.reader(open(sys.argv[1])))
h=None; agg=collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows:
    if "Kernel Name" in r: h=r; continue
    if h and len(r)==len(h):
        d=dict(zip(h,r)); agg[d["Kernel Name"].split("(")[0]][d["Metric Name"]].append(float(d["Metric Value"].replace(",","")))
for k,v in sorted(agg.items(), key=lambda kv:-sum(kv[1]["gpu__time_duration.sum"])):
    t=v["gpu__time_duration.sum"]; rd=v.get("dram__bytes_read.sum",[0]); wr=v.get("dram__bytes_write.sum",[0])
    print(f"{k[:50]:50s} n={len(t):4d} mean_us={sum(t)/len(t)/1e3:8.2f} rdMB={sum(rd)/len(rd)/1e6:7.2f} wrMB={sum(wr)/len(wr)/1e6:7.2f}")
