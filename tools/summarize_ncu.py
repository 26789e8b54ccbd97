"""Write the committed ncu summaries under profiles/ from gpurun_out/ captures.

usage: python tools/summarize_ncu.py <round-tag>
Reads gpurun_out/<tag>_launches_bench.csv, <tag>_corr_full.ncu-rep and
<tag>_ba_full.ncu-rep; writes profiles/<tag>_launches.csv (own kernels only),
profiles/<tag>_ncu_summary.md and profiles/corr_traffic.json.
"""
import csv
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
out_dir = ROOT / "profiles" / (tag[:2] if tag.startswith("r2") else "")
out_dir.mkdir(exist_ok=True)
src = ROOT / "gpurun_out"

# ---- launch list ----
rows = [r for r in csv.reader(l for l in open(src / f"{tag}_launches_bench.csv") if not l.startswith("=="))]
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
own = [(r[ki], float(r[vi]), r[ui]) for r in rows[1:] if "pvo_dev" in r[ki]]
with open(out_dir / f"{tag}_launches.csv", "w") as f:
    f.write("kernel,duration_ns\n")
    for k, v, u in own:
        f.write(f"{k.split('(')[0].split('::')[-1]},{v * (1000 if u == 'us' else 1):.0f}\n")
per = defaultdict(list)
for k, v, u in own:
    per[k.split("(")[0].split("::")[-1]].append(v * (1000 if u == "us" else 1))


def raw(rep, names):
    txt = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv", "--print-units", "base"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(txt.splitlines()))
    hh, vv = r[0], r[2]
    return {n: vv[hh.index(n)] for n in names if n in hh}


COUNTERS = {"dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "lts_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
            "fma_pipe_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_elapsed",
            "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
            "smem_wavefronts_pct": "l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed",
            "kernel_us": "gpu__time_duration.sum"}


def corr_counters(rep, tag):
    """The correlation kernel's ncu utilisation counters (one --set full launch),
    as bench.py reports them under roofline.ncu."""
    d = raw(rep, list(COUNTERS.values()))
    out = {k: float(d[v].replace(",", "")) for k, v in COUNTERS.items() if v in d}
    if "kernel_us" in out:
        out["kernel_us"] /= 1000.0  # base unit ns
    out["source"] = f"{out_dir.relative_to(ROOT)}/{tag}_ncu_summary.md ({Path(rep).name})"
    return out


M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
     "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
     "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_elapsed",
     "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
     "sm__warps_active.avg.pct_of_peak_sustained_active", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
lines = [f"# ncu summary ({tag})", "", "## Launch list (own kernels, `--metrics gpu__time_duration.sum`, cold/serialised)", "",
         "`bench.py` also times the flow provider's `propose` once per run (its `propose_ms` field): its kernels",
         "(`measure_gram_kernel`, `measure_exact_kernel`, the per-slot `gram25_kernel` maps) are listed but are not",
         "part of the benchmark step (Gram + tile preparation + correlation + BA); the step share column excludes them.", "",
         "| kernel | launches | mean us | share | step share |", "|---|---|---|---|---|"]
tot = sum(sum(v) for v in per.values())
NOT_STEP = ("measure_kernel", "measure_gram_kernel", "measure_exact_kernel", "gram25_kernel")  # propose(), not the step
step_tot = sum(sum(v) for k, v in per.items() if k not in NOT_STEP)
for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
    ss = "—" if k in NOT_STEP else f"{100 * sum(v) / step_tot:.1f}%"
    lines.append(f"| {k} | {len(v)} | {sum(v) / len(v) / 1000:.1f} | {100 * sum(v) / tot:.1f}% | {ss} |")
traffic = None
names = sorted(f.name[len(tag) + 1:-len(".ncu-rep")] for f in src.glob(f"{tag}_*_full.ncu-rep"))
traffic_by_cfg = {}
counters_by_cfg = {}
for name in names:
    rep = src / f"{tag}_{name}.ncu-rep"
    if not rep.exists():
        continue
    d = raw(rep, M)
    lines += ["", f"## `--set full` capture: {name}", "", "| metric | value |", "|---|---|"]
    lines += [f"| {k} | {v} |" for k, v in d.items()]
    if name.startswith("corr"):
        def mb(x):
            x = x.replace(",", "")
            return float(x)
        rd = raw(rep, ["dram__bytes_read.sum", "dram__bytes_write.sum"])
        # raw page units vary (Mbyte/Gbyte); ask ncu for bytes explicitly
        txt = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv", "--print-units", "base"],
                             capture_output=True, text=True).stdout
        r = list(csv.reader(txt.splitlines()))
        hh, vv = r[0], r[2]
        traffic = mb(vv[hh.index("dram__bytes_read.sum")]) + mb(vv[hh.index("dram__bytes_write.sum")])
        cfg = name.split("_")[1] if name.count("_") >= 2 else "c2"
        traffic_by_cfg[cfg] = traffic
        counters_by_cfg[cfg] = corr_counters(rep, tag)
(out_dir / f"{tag}_ncu_summary.md").write_text("\n".join(lines) + "\n")
if traffic_by_cfg:
    traffic_by_cfg["source"] = f"{tag}_corr*_full.ncu-rep (dram__bytes_read.sum + dram__bytes_write.sum, one launch)"
    traffic_by_cfg["counters"] = counters_by_cfg
    (ROOT / "profiles" / "corr_traffic.json").write_text(json.dumps(traffic_by_cfg) + "\n")
print("\n".join(lines))
print("traffic", traffic)
