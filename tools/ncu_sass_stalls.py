"""Per-SASS-instruction stall breakdown from an ncu report: top instructions by
samples and the stall-reason totals split by opcode class."""
import csv
import subprocess
import sys
from collections import Counter, defaultdict

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
idx = {k: i for i, k in enumerate(hdr)}
reasons = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k]
by_op = defaultdict(Counter)
tot = Counter()
top = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    src = r[idx["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    top.append((s, r[idx["Address"]][-5:], src[:70]))
    for k in reasons:
        v = int(r[idx[k]] or 0)
        by_op[op][k] += v
        tot[k] += v
T = sum(tot.values()) or 1
print("reason totals:", ", ".join(f"{k[6:]} {100 * v / T:.1f}%" for k, v in tot.most_common(10)))
ops = sorted(by_op.items(), key=lambda kv: -sum(kv[1].values()))[:12]
for op, c in ops:
    s = sum(c.values())
    print(f"{op:10s} {100 * s / T:5.1f}%  " + ", ".join(f"{k[6:]} {100 * v / T:.1f}" for k, v in c.most_common(4)))
print("top instructions:")
for s, a, src in sorted(top, reverse=True)[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(f"{100 * s / T:5.2f}% {a} {src}")
