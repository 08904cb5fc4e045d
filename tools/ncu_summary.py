"""Summarise an ncu --set full report: headline metrics, top stall reasons, and the
executed-instruction mix by opcode (from the SASS source page)."""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_shared_mem",
        "launch__occupancy_limit_registers"]
for r in rows[2:]:
    d = dict(zip(h, r))
    print("kernel", d.get("Kernel Name", "")[:120])
    for k in KEYS:
        print(f"  {k:60s} {d.get(k)}")
    st = [(float(v.replace(",", "")) if v else 0.0, k) for k, v in d.items()
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")]
    for v, k in sorted(st, reverse=True)[:10]:
        print(f"  stall {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):40s} {v:.0f}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = list(csv.reader(io.StringIO(src)))
hdr = None
mix = Counter()
tot = 0
for ln in lines:
    if "Source" in ln and "Instructions Executed" in ln:
        hdr = ln
        continue
    if hdr is None or len(ln) != len(hdr):
        continue
    d = dict(zip(hdr, ln))
    try:
        n = float(d["Instructions Executed"].replace(",", ""))
    except ValueError:
        continue
    op = d["Source"].strip().split()
    if not op:
        continue
    o = op[0] if not op[0].startswith("@") else (op[1] if len(op) > 1 else op[0])
    mix[o.split(".")[0]] += n
    tot += n
if tot:
    print(f"  executed warp-instructions (source page) {tot:.4g}")
    print("  " + "  ".join(f"{k}:{100 * v / tot:.1f}%" for k, v in mix.most_common(24)))
