"""Per-launch ncu counts of the stage kernels for bench.py's roofline fields (profiles/r02_stage_kernels.json):
python tools/stage_kernels.py out.json cfg2=ncu_cfg2.csv cfg4=ncu_cfg4.csv cfg5=ncu_cfg5.csv
Each csv is `ncu --csv --metrics <KEYS>` over a few launches of the window-stencil and expectation kernels
of that workload (tools/profile_round.sh); values are averaged over the captured launches."""
import csv, json, sys

KEYS = {"smsp__inst_executed.sum": "warp_inst_per_launch",
        "dram__bytes_read.sum": "dram_read", "dram__bytes_write.sum": "dram_write",
        "sm__sass_thread_inst_executed_op_fp64_pred_on.sum": "fp64_thread_inst_per_launch",
        "gpu__time_duration.sum": "ncu_duration"}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1,
         "msecond": 1e3, "ms": 1e3,
         "inst": 1, "": 1}


def load(path):
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    hdr = rows[0]
    ki, mi, ui, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
    idi = hdr.index("ID")
    per = {}
    for r in rows[1:]:
        if len(r) <= vi or r[mi] not in KEYS:
            continue
        role = "window" if "window" in r[ki] else "expectation" if "contract" in r[ki] or "ozaki" in r[ki] else None
        if role is None:
            continue
        v = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1)
        per.setdefault(role, {}).setdefault(r[idi], {})[KEYS[r[mi]]] = v
    out = {}
    for role, launches in per.items():
        agg = {}
        for m in launches.values():
            for k, v in m.items():
                agg.setdefault(k, []).append(v)
        d = {k: sum(v) / len(v) for k, v in agg.items()}
        d["dram_bytes_per_launch"] = d.pop("dram_read", 0.0) + d.pop("dram_write", 0.0)
        d["ncu_us"] = d.pop("ncu_duration", None)
        d["launches"] = len(launches)
        out[role] = d
    return out


if __name__ == "__main__":
    res = {}
    for a in sys.argv[2:]:
        cfg, path = a.split("=", 1)
        res[cfg] = load(path)
        res[cfg]["source"] = path.split("/")[-1]
    with open(sys.argv[1], "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))
