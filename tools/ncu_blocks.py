import csv, subprocess, sys
from collections import defaultdict
rep = sys.argv[1]
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(src)); hdr = rows[1]; idx = {h: i for i, h in enumerate(hdr)}
data = []
for r in rows[2:]:
    if len(r) < len(hdr) or r[0].startswith('Kernel'): break
    data.append(r)
ex = [float(r[idx['Instructions Executed']] or 0) for r in data]
tot = sum(ex)
ref = float(sys.argv[2])   # executions of the per-vector body
buckets = defaultdict(float)
for e in ex:
    if e == 0: continue
    ratio = e / ref
    key = round(ratio, 1) if ratio < 4 else round(ratio)
    buckets[key] += e
print(f"total {tot:.4g} warp-instr;  per-vector-iteration units (exec/ref -> share, instr-equiv per vector):")
for k in sorted(buckets, key=lambda k: -buckets[k])[:15]:
    print(f"  ratio {k:>6}: share {buckets[k]/tot*100:5.1f}%  = {buckets[k]/ref:7.1f} warp-instr per vector-iteration")
print(f"  ALL: {tot/ref:.1f} warp-instr per vector-iteration (16 elements/lane)")
