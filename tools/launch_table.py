"""Print the last N launches of an ncu --csv launch list (duration, DRAM bytes, GB/s)."""
import csv
import sys
from collections import defaultdict

path, n = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 20
rows = list(csv.reader(open(path)))
i0 = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[i0]
ki, mn, mv, gs, idc = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Grid Size", "ID"))
recs = defaultdict(dict)
for r in rows[i0 + 1:]:
    if len(r) <= mv:
        continue
    recs[int(r[idc])][r[mn]] = float(r[mv].replace(",", ""))
    recs[int(r[idc])]["name"] = r[ki]
    recs[int(r[idc])]["grid"] = r[gs]
for i in sorted(recs)[-n:]:
    r = recs[i]
    t = r["gpu__time_duration.sum"] / 1e3
    b = (r.get("dram__bytes_read.sum", 0) + r.get("dram__bytes_write.sum", 0)) / 1e6
    print(f"{i:6d} {r['name'][:62]:62s} {r['grid']:>12s} {t:9.1f} us {b:9.1f} MB {b / t / 1e3 if t else 0:7.2f} TB/s")
