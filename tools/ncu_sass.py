import csv, subprocess, sys
rep, a, b = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(src)); hdr = rows[1]; idx = {h: i for i, h in enumerate(hdr)}
data = []
for r in rows[2:]:
    if len(r) < len(hdr) or r[0].startswith('Kernel'): break
    data.append(r)
for i in range(a, b + 1):
    print(i, data[i][idx['Instructions Executed']], data[i][idx['Source']][:88])
