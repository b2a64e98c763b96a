"""Sum an ncu metrics CSV per kernel name: python tools/traffic_sum.py file.csv [n_backward]."""
import collections, csv, json, sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
per = collections.defaultdict(lambda: collections.defaultdict(float))
cnt = collections.Counter()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0]
        v = float(d["Metric Value"].replace(",", ""))
        u = d["Metric Unit"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}.get(u, 1)
        per[name][d["Metric Name"]] += v * scale
        if d["Metric Name"] == "gpu__time_duration.sum":
            cnt[name] += 1
out = {}
for k, m in per.items():
    out[k] = {"launches": cnt[k], "dram_read_bytes": m.get("dram__bytes_read.sum", 0.0),
              "dram_write_bytes": m.get("dram__bytes_write.sum", 0.0), "time_us": m.get("gpu__time_duration.sum", 0.0)}
tot = sum(v["dram_read_bytes"] + v["dram_write_bytes"] for v in out.values())
print(json.dumps({"kernels": out, "total_dram_bytes": tot}, indent=1))
