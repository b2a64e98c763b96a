"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel name."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(list)
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            v = float(d["Metric Value"].replace(",", ""))
            if d["Metric Unit"] == "usecond":
                v *= 1e3
            elif d["Metric Unit"] == "msecond":
                v *= 1e6
            agg[d["Kernel Name"].split("(")[0]].append(v)
tot = sum(sum(v) for v in agg.values())
print(f"{'kernel':44s} {'n':>6s} {'mean_us':>10s} {'min_us':>9s} {'total_ms':>9s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k[:44]:44s} {len(v):6d} {sum(v)/len(v)/1e3:10.2f} {min(v)/1e3:9.2f} {sum(v)/1e6:9.3f} {sum(v)/tot*100:5.1f}%")
