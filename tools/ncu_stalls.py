"""Top SASS lines of an ncu report by warp-stall samples: python tools/ncu_stalls.py REP [N]"""
import csv, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(src)); hdr = rows[1]; idx = {h: i for i, h in enumerate(hdr)}
data = []
for r in rows[2:]:
    if len(r) < len(hdr) or r[0].startswith('Kernel'): break
    data.append(r)
key = [h for h in hdr if h.startswith('Warp Stall Sampling (All')][0]
tot = sum(float(r[idx[key]] or 0) for r in data)
top = sorted(range(len(data)), key=lambda i: -float(data[i][idx[key]] or 0))[:n]
for i in sorted(top):
    v = float(data[i][idx[key]] or 0)
    print(f"{i:5d} {v/tot*100:5.1f}%  {data[i][idx['Source']].strip()[:80]}")
