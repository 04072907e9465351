"""Aggregate an ncu --metrics launch list (gpu__time_duration, dram bytes, grid size) per kernel.

python scripts/launch_list_agg.py gpurun_out/list.csv [out.json] [note]
Prints per-kernel launches, total ms and DRAM GB/s (bytes / duration, cold-cache ncu replays).
"""
import collections
import csv
import json
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1}


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, mi, vi, ui, idi = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    launches = collections.defaultdict(dict)
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = r[vi].replace(",", "")
        try:
            launches[r[idi]][r[mi]] = float(v) * SCALE.get(r[ui], 1.0)
        except ValueError:
            continue
        launches[r[idi]]["kernel"] = r[ki].split("(")[0]
    return launches


def aggregate(launches):
    agg = collections.defaultdict(lambda: {"launches": 0, "ms": 0.0, "dram_bytes": 0.0})
    for d in launches.values():
        a = agg[d["kernel"]]
        a["launches"] += 1
        a["ms"] += d.get("gpu__time_duration.sum", 0.0) * 1e3
        a["dram_bytes"] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    out = []
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["ms"]):
        gbs = a["dram_bytes"] / (a["ms"] * 1e-3) / 1e9 if a["ms"] else 0.0
        out.append({"kernel": k, "launches": a["launches"], "ms": round(a["ms"], 3),
                    "dram_GB": round(a["dram_bytes"] / 1e9, 3), "dram_GBps": round(gbs, 1)})
    return out


if __name__ == "__main__":
    res = aggregate(load(sys.argv[1]))
    for r in res:
        print(f"{r['kernel']:<50} n={r['launches']:6d} {r['ms']:10.1f} ms {r['dram_GBps']:8.0f} GB/s")
    if len(sys.argv) > 2:
        json.dump({"source": sys.argv[1], "note": sys.argv[3] if len(sys.argv) > 3 else "", "kernels": res},
                  open(sys.argv[2], "w"), indent=1)
