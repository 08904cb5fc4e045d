"""Summarise an ncu --csv launch list into profiles/: per-kernel launch counts, mean
duration and DRAM bytes, plus the traffic file bench.py reads.

usage: python tools/launches_summary.py LAUNCHES.csv OUT_PREFIX [TRAFFIC_JSON]

The step launches alternate one per width group in QftModelState order (groups sorted
by column count: 4096, then 11008 for LLaMA-2-7B), so the i-th step_kernel launch of a
step belongs to group i.
"""
import collections
import csv
import json
import sys


def load(path):
    lines = [l for l in open(path) if not l.startswith("==")]
    rows = list(csv.DictReader(lines))
    per = collections.OrderedDict()
    for r in rows:
        d = per.setdefault(r["ID"], {"name": r["Kernel Name"], "grid": r["Grid Size"],
                                     "block": r["Block Size"]})
        v = r["Metric Value"].replace(",", "")
        d[r["Metric Name"]] = float(v) if v else 0.0
    return list(per.values())


def main():
    src, prefix = sys.argv[1], sys.argv[2]
    traffic_out = sys.argv[3] if len(sys.argv) > 3 else None
    launches = load(src)
    agg = collections.OrderedDict()
    for l in launches:
        a = agg.setdefault(l["name"], {"launches": 0, "time_ns": 0.0, "dram_read": 0.0,
                                       "dram_write": 0.0})
        a["launches"] += 1
        a["time_ns"] += l.get("gpu__time_duration.sum", 0.0)
        a["dram_read"] += l.get("dram__bytes_read.sum", 0.0)
        a["dram_write"] += l.get("dram__bytes_write.sum", 0.0)
    total = sum(a["time_ns"] for a in agg.values()) or 1.0
    with open(prefix + "_launches_summary.txt", "w") as f:
        f.write(f"source: {src}\n{len(launches)} launches, {total / 1e6:.3f} ms total (ncu, serialised, cold)\n")
        for name, a in sorted(agg.items(), key=lambda kv: -kv[1]["time_ns"]):
            n = a["launches"]
            f.write(f"{a['time_ns'] / total * 100:6.2f}%  n={n:5d}  mean {a['time_ns'] / n / 1e6:9.4f} ms"
                    f"  dram/launch {(a['dram_read'] + a['dram_write']) / n / 1e9:8.4f} GB  {name[:90]}\n")
    steps = [l for l in launches if "step_kernel" in l["name"]]
    if traffic_out and steps:
        # the last two step launches are one full step (4096 group, then 11008 group)
        keys = ["cols4096", "cols11008"]
        tail = steps[-len(keys):]
        traffic = {k: l.get("dram__bytes_read.sum", 0.0) + l.get("dram__bytes_write.sum", 0.0)
                   for k, l in zip(keys, tail)}
        traffic["source"] = src
        traffic["kernel_ms"] = {k: l.get("gpu__time_duration.sum", 0.0) / 1e6 for k, l in zip(keys, tail)}
        json.dump(traffic, open(traffic_out, "w"), indent=1)
    print(open(prefix + "_launches_summary.txt").read())


if __name__ == "__main__":
    main()
