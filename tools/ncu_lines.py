"""Aggregate an ncu report's SASS stall samples by CUDA source line.
usage: python tools/ncu_lines.py report.ncu-rep [top]"""
import collections
import csv
import io
import subprocess
import sys


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
agg = collections.defaultdict(lambda: [0.0, 0.0, collections.Counter(), ""])
cur, hdr, last = None, None, None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    if r[0]:
        last = (cur, int(r[0]), r[1].strip()[:80])
    a = agg[last]
    a[0] += f(r[4])
    a[1] += f(r[7])
    a[3] = last[2]
    for k, v in zip(hdr, r):
        if k.startswith("stall_") and "Not Issued" not in k:
            a[2][k] += f(v)
tot = sum(v[0] for v in agg.values())
print("total samples", tot)
for key, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{int(v[0]):6d} {v[0] / tot * 100:5.1f}% {v[1] / 1e6:7.2f}M {key[0]}:{key[1]} {v[3][:60]} "
          f"{dict((k[6:], int(c)) for k, c in v[2].most_common(3))}")
