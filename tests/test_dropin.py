"""The drop-in operator layer, exercised by the reference's OWN tests.

oracle/ref_build.py links the reference's unit tests (proj/tests/test_*.cpp,
unmodified) against the reference's sources MINUS camera.cpp, correlation.cpp
and bundle_adjust.cpp, plus paper_2208_04726_b200/dropin/*.cpp — the
operators those files define (reproject_patch, reprojection_jacobians,
correlate, correlate_at, correlate_at_cubic, build_target, schur_solve,
gauss_newton_step, optimize_window, BAProblem::validate,
NormalEquations::dump), re-implemented with the reference's signatures over
the C-ABI — and libpvo_b200.so.  On the GPU box the reference's camera,
bundle_adjust and correlation test cases therefore run the sm_100a kernels.
Without a GPU the same binary must fail loudly (no CPU fallback).
"""
from __future__ import annotations

import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
BIN = ROOT / "oracle" / "_ref" / "pvo_dropin_tests"

pytestmark = pytest.mark.skipif(not BIN.exists(), reason="oracle/_ref/pvo_dropin_tests not built "
                                                          "(needs /root/reference: python oracle/ref_build.py)")

# suites whose cases call the replaced operators (directly or through PatchGraph / the providers)
OPERATOR_SUITES = "se3,camera,patch_graph,bundle_adjust,features"


def _run(args, timeout=900):
    r = subprocess.run([str(BIN), *args], capture_output=True, text=True, timeout=timeout)
    cases = dict(re.findall(r"^\[case\] [^/]+ / (.*): (PASS|FAIL)$", r.stdout, flags=re.M))
    m = re.search(r"test cases: (\d+) run, (\d+) failed; checks: (\d+), (\d+) failed", r.stdout)
    assert m, r.stdout[-2000:] + r.stderr[-2000:]
    return r, cases, [int(v) for v in m.groups()]


def test_dropin_links_no_reference_operator():
    # the replaced reference translation units are not in the binary: their
    # functions resolve to the drop-in objects (which call into libpvo_b200.so)
    nm = subprocess.run(["nm", "-C", str(BIN)], capture_output=True, text=True, check=True).stdout
    undefined = {ln.split()[-1] for ln in nm.splitlines() if " U pvo_" in ln}
    for sym in ("pvo_reproject_patches", "pvo_reprojection_jacobians", "pvo_correlate", "pvo_correlate_points",
                "pvo_gauss_newton_step", "pvo_schur_solve", "pvo_ba_window"):
        assert sym in undefined, sym
    ldd = subprocess.run(["ldd", str(BIN)], capture_output=True, text=True).stdout
    assert "libpvo_b200.so" in ldd and "not found" not in ldd


def test_dropin_fails_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    r, cases, (run, failed, _, _) = _run(["-ts=camera"], timeout=120)
    assert failed > 0 and "pvo_b200: CUDA error" in r.stdout + r.stderr


@pytest.mark.gpu
def test_reference_operator_suites_on_gpu():
    r, cases, (run, failed, checks, _) = _run([f"-ts={OPERATOR_SUITES}"])
    failing = sorted(n for n, v in cases.items() if v == "FAIL")
    assert failed == 0 and r.returncode == 0, (failing, r.stdout[-6000:])
    assert run >= 60 and checks > 50000, (run, checks)
