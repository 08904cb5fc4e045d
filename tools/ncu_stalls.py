"""Top SASS lines of an ncu report by warp-stall samples, with the dominant reasons:
python tools/ncu_stalls.py REP [N]"""
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
reasons = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
f = lambda r, k: float(r[idx[k]] or 0)
tot = sum(f(r, key) for r in data)
top = sorted(range(len(data)), key=lambda i: -f(data[i], key))[:n]
for i in sorted(top):
    r = data[i]
    rs = sorted(((f(r, k), k[6:]) for k in reasons), reverse=True)[:2]
    why = " ".join(f"{k}:{v/max(f(r,key),1)*100:.0f}%" for v, k in rs if v)
    print(f"{i:5d} {f(r,key)/tot*100:5.1f}%  {r[idx['Source']].strip()[:60]:60s} {why}")
agg = {k[6:]: sum(f(r, k) for r in data) / tot * 100 for k in reasons}
print("all:", " ".join(f"{k}:{v:.1f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1]) if v > 0.5))
