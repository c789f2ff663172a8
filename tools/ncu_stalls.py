"""Per-region warp-stall shares of one ncu report (--page source sass): python tools/ncu_stalls.py REP [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
r = list(csv.reader(io.StringIO(txt)))
h = r[1]
idx = {k: i for i, k in enumerate(h)}
rows = [x for x in r[2:] if len(x) >= len(h) - 1]
k = "Warp Stall Sampling (All Samples)"
tot = sum(float(x[idx[k]] or 0) for x in rows) or 1
acc = 0
for i, x in enumerate(rows):
    s = float(x[idx[k]] or 0)
    acc += s
    if s / tot > 1.0 / top or any(t in x[1] for t in ("UTCIMMA", "UTCBAR", "BAR.SYNC", "TRYWAIT", "LDTM")):
        print(f"{i:5d} {s / tot * 100:5.1f} {acc / tot * 100:5.1f}  {x[1][:70]:70s} exec {x[idx['Instructions Executed']]}")
