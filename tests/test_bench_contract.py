"""bench.py's reference arm on CPU: it runs the reference's own code
(oracle/_ref) over every edge of the window, prints the contract's JSON line
with the same `config` as the GPU arm, and never maps the product library."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent

PROBE = r"""
import sys, json
sys.argv = ["bench.py", "--impl", "reference", "--config", "c1", "--steps", "2", "--warmup", "1"]
sys.path.insert(0, ".")
import bench
bench.main()
maps = open("/proc/self/maps").read()
libs = sorted({l.split()[-1] for l in maps.splitlines() if l.endswith(".so") and "/repo/" in l})
print("MAPPED " + json.dumps(libs))
print("MODULES " + json.dumps(sorted(m for m in sys.modules if m.startswith("paper_2208_04726_b200"))))
"""


def test_reference_arm_clean_and_unextrapolated():
    r = subprocess.run([sys.executable, "-c", PROBE], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = r.stdout.splitlines()
    line = json.loads(next(l for l in lines if l.startswith("{")))
    mapped = json.loads(next(l for l in lines if l.startswith("MAPPED "))[7:])
    modules = json.loads(next(l for l in lines if l.startswith("MODULES "))[8:])
    assert modules == []
    assert not any("libpvo_b200" in m for m in mapped), mapped
    assert line["impl"] == "reference" and line["steps"] == 2 and line["warmup"] == 1
    assert line["cpu_baseline"]["kind"] in ("reference", "port")
    assert "extrapolat" not in line["cpu_baseline"]["sample"]
    import bench
    import pvo_synth as synth

    w = synth.generate("c1", seed=0, features=False)
    assert line["config"] == bench.workload_config("c1", w, line["config"]["edges_per_gpu"], 1)
    assert line["config"]["edges_per_gpu"] == 6144
    assert line["ms_per_step"] == pytest.approx(line["config"]["edges_per_gpu"] / line["value"] * 1e3)
