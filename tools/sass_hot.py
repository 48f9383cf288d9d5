"""Per-region instruction counts of one ncu capture (diagnostics).
    python tools/sass_hot.py rep.ncu-rep [start end]"""
import csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]; data = rows[2:]
ie = h.index("Instructions Executed"); ss = h.index("Warp Stall Sampling (All Samples)")
vals = [int(r[ie]) if r[ie].isdigit() else 0 for r in data]
if len(sys.argv) > 3:
    for i in range(int(sys.argv[2]), int(sys.argv[3])):
        print(i, data[i][1].strip()[:70], vals[i], data[i][ss])
    sys.exit()
print("total warp instructions", sum(vals))
runs = []; s = 0
for i in range(1, len(vals) + 1):
    if i == len(vals) or vals[i] != vals[s]:
        runs.append((s, i - 1, vals[s], (i - s) * vals[s], sum(int(data[k][ss] or 0) for k in range(s, i)))); s = i
for a, b, v, t, smp in sorted(runs, key=lambda x: -x[3])[:12]:
    print(f"{a:5d}-{b:5d} x{v:8d} = {t:9d} instr, {smp:5d} samples  {data[a][1].strip()[:50]}")
