"""Summarise an ncu report of the step kernel: key metrics, opcode mix, hot blocks, stalls."""
import csv, subprocess, sys
from collections import Counter
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(raw)); hdr = rows[0]; units = rows[1]; idx = {h: i for i, h in enumerate(hdr)}
want = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'smsp__inst_executed.sum', 'launch__grid_size', 'launch__shared_mem_per_block_dynamic',
        'launch__occupancy_limit_shared_mem', 'launch__registers_per_thread']
stall_keys = [h for h in hdr if h.startswith('smsp__average_warp_latency_issue_stalled_') or
              h.startswith('smsp__pcsamp_warps_issue_stalled_')]
for r in rows[2:]:
    print("kernel", r[idx['Kernel Name']][:60])
    for w in want:
        if w in idx: print(f"  {w:60s} {r[idx[w]]} {units[idx[w]]}")
    st = sorted(((float(r[idx[k]] or 0), k) for k in stall_keys if 'pcsamp' in k and not k.endswith('_not_issued')), reverse=True)[:8]
    for v, k in st: print(f"  stall {k.replace('smsp__pcsamp_warps_issue_stalled_','')}: {v:.0f}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(src)); hdr = rows[1]; idx = {h: i for i, h in enumerate(hdr)}
data = []
for r in rows[2:]:
    if len(r) < len(hdr) or r[0].startswith('Kernel'): break
    data.append(r)
tot = sum(float(r[idx['Instructions Executed']] or 0) for r in data)
cnt = Counter()
for r in data:
    t = r[idx['Source']].split()
    if not t: continue
    op = t[1] if t[0].startswith('@') else t[0]
    cnt[op.split('.')[0]] += float(r[idx['Instructions Executed']] or 0)
print("total warp-instr (first kernel)", tot)
print("  ".join(f"{op}:{c/tot*100:.1f}%" for op, c in cnt.most_common(24)))
ex = [float(r[idx['Instructions Executed']] or 0) for r in data]
blocks = []; cur = None
for i, e in enumerate(ex):
    if cur and abs(e - cur[2]) <= 0.02 * max(e, 1): cur[1] = i; cur[3] += e
    else:
        if cur: blocks.append(cur)
        cur = [i, i, e, e]
blocks.append(cur); blocks.sort(key=lambda b: -b[3])
for b in blocks[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
    print(f"  lines {b[0]}-{b[1]} ({b[1]-b[0]+1}) exec {b[2]:.3g} share {b[3]/tot*100:.1f}%  {data[b[0]][idx['Source']][:50]}")
