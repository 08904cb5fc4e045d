"""Summarise a gpu_round.sh capture into profiles/: launch-list shares (ncu, serialised,
cold caches), per-kernel DRAM bytes, full-set summaries of the rows kernel, traffic json.
usage: python tools/make_profiles.py TAG"""
import collections, csv, json, os, shutil, subprocess, sys
tag = sys.argv[1]
G, P = "gpurun_out", "profiles"
for f in ("bench", "bench_ref", "sweep", "b13"):
    src = os.path.join(G, f"{f}_{tag}.json")
    if os.path.exists(src):
        shutil.copy(src, os.path.join(P, f"{f}_{tag}.json"))
# launch list
rows = list(csv.reader(open(os.path.join(G, f"launches_all_{tag}.csv"))))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(r)
ix = {h: i for i, h in enumerate(hdr)}
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
tscale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
bscale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
ids = set()
for r in data:
    name = r[ix["Kernel Name"]]
    m, u = r[ix["Metric Name"]], r[ix["Metric Unit"]]
    v = float(r[ix["Metric Value"]].replace(",", ""))
    ids.add(r[ix["ID"]])
    if m == "gpu__time_duration.sum":
        agg[name][0] += 1
        agg[name][1] += v * tscale.get(u, 1.0)
    elif m.startswith("dram__bytes"):
        agg[name][2] += v * bscale.get(u, 1.0)
tot = sum(v[1] for v in agg.values())
lines = [f"source: {G}/launches_all_{tag}.csv (ncu --metrics gpu__time_duration.sum,dram__bytes_*"
         " --clock-control none; one bench command: setup + 3 warm-up + 2 timed steps)",
         f"{len(ids)} launches, {tot:.2f} ms total (serialised, cold caches)"]
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:16]:
    lines.append(f"{v[1] / tot * 100:6.2f}%  n={v[0]:5d}  mean {v[1] / max(v[0], 1):9.4f} ms  "
                 f"dram/launch {v[2] / max(v[0], 1) / 1e9:8.3f} GB  {k[:90]}")
open(os.path.join(P, f"{tag}_launches_summary.txt"), "w").write("\n".join(lines) + "\n")
print("\n".join(lines[:8]))
traffic = {}
for k, v in agg.items():
    if "rows_kernel<128" in k:
        traffic["cols4096"] = v[2] / max(v[0], 1)
    elif "rows_kernel<384" in k:
        traffic["cols11008"] = v[2] / max(v[0], 1)
traffic["source"] = f"profiles/{tag}_launches_summary.txt (rows_kernel DRAM read+write per launch)"
json.dump(traffic, open(os.path.join(P, "traffic_r01.json"), "w"), indent=1)
# full-set summary
rep = os.path.join(G, f"prof_{tag}.ncu-rep")
if os.path.exists(rep):
    out = subprocess.run([sys.executable, "tools/ncu_summary.py", rep, "6"], capture_output=True,
                         text=True).stdout
    st = subprocess.run([sys.executable, "tools/ncu_stalls.py", rep, "12"], capture_output=True,
                        text=True).stdout
    open(os.path.join(P, f"{tag}_rows_kernel_ncu_full.txt"), "w").write(
        f"source: {rep} (ncu --set full --clock-control none, rows_kernel launches of both width "
        "classes)\n" + out + "\nstall hot spots (first kernel):\n" + st)
    print(out[:1500])
