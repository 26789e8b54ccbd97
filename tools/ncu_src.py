"""Summarise an ncu source page (cuda,sass view): stall samples per CUDA source line."""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
agg = defaultdict(lambda: [0, 0, ""])
fname, hdr = None, None
for row in rows:
    if row and row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row and row[0] == "Line No":
        hdr = row
        continue
    if hdr and len(row) >= 8 and row[0].isdigit():
        try:
            s = int(row[4] or 0)
            ie = int(row[7] or 0)
        except ValueError:
            continue
        key = (fname, int(row[0]))
        agg[key][0] += s
        agg[key][1] += ie
        agg[key][2] = row[1].strip()[:90]
tot = sum(v[0] for v in agg.values()) or 1
for (f, l), (s, ie, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100 * s / tot:5.1f}% {f}:{l:<5} inst={ie:>11}  {src}")
