"""The parity anchor: the reference's own code (oracle/_ref).

oracle/ref_build.py compiles /root/reference/proj/src/*.cpp and the
reference's unit tests unmodified against in-repo shims for the libraries this
image lacks (oracle/ref_shim/: Eigen 3 subset, doctest, nlohmann::json,
libpng stub).  These CPU tests check that

* the reference's own test suites pass on that build (so the shims carry the
  arithmetic the reference relies on), and
* the restatement (oracle/pvo_oracle.cpp) agrees with the reference on the
  benchmark configurations: graph and window problem bit-exact, correlation
  and provider measurements bit-exact, BA within 1e-8.

pyoracle prefers the reference build, so every other oracle comparison in
tests/ (the ported KATs, the GPU parity tests) runs against the reference
itself whenever oracle/_ref exists.
"""
from __future__ import annotations

import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

import oracle.pyoracle as orc
import pvo_synth as synth

ROOT = Path(__file__).resolve().parent.parent
TESTS_BIN = ROOT / "oracle" / "_ref" / "pvo_ref_tests"

pytestmark = pytest.mark.skipif(orc.lib_ref is None or not TESTS_BIN.exists(),
                                reason="oracle/_ref not built (needs /root/reference: python oracle/ref_build.py)")

# End-to-end pipeline cases (pipeline state machine: out of scope)
# that fail on this build.  Their outcome is unchanged under -O1 / -O3
# -march=x86-64-v3 -ffp-contract=fast builds of the same sources (identical
# values to 1e-9), so they are not rounding artefacts of the shim; no hot-path
# suite fails.  See DESIGN.md §4.
KNOWN_PIPELINE_FAILURES = {
    "fast motion keeps every keyframe",
    "oracle pipeline tracks the simulator to sub-centiunit ATE",
}


def _run_suites(suites: str):
    r = subprocess.run([str(TESTS_BIN), f"-ts={suites}"], capture_output=True, text=True, timeout=600)
    cases = dict(re.findall(r"^\[case\] [^/]+ / (.*): (PASS|FAIL)$", r.stdout, flags=re.M))
    m = re.search(r"test cases: (\d+) run, (\d+) failed; checks: (\d+), (\d+) failed", r.stdout)
    assert m, r.stdout[-2000:] + r.stderr[-2000:]
    return r, cases, [int(v) for v in m.groups()]


def test_reference_hot_path_suites_pass():
    r, cases, (run, failed, checks, _) = _run_suites("se3,camera,patch_graph,bundle_adjust,features")
    assert failed == 0 and r.returncode == 0, r.stderr[-4000:]
    assert run >= 60 and checks > 50000, (run, checks)


def test_reference_support_suites_pass():
    r, cases, (run, failed, _, _) = _run_suites("simulator,trajectory")
    assert failed == 0 and run >= 20, r.stderr[-4000:]


def test_reference_pipeline_suite():
    r, cases, (run, failed, _, _) = _run_suites("pipeline")
    failing = {name for name, v in cases.items() if v == "FAIL"}
    assert run == len(cases) >= 15
    assert failing <= KNOWN_PIPELINE_FAILURES, failing


@pytest.mark.parametrize("cfg", ["c1", "c3", "c2"])
def test_restatement_matches_reference(cfg):
    w = synth.generate(cfg, seed=11)
    gr = synth.build_graph(w, orc.PatchGraph)  # orc.PatchGraph runs on the reference build
    with orc.using("restated"):
        gs = synth.build_graph(w, orc.PatchGraph)
        ps = gs.window_problem(w.cfg["window"])
        es = gs.edges()
    pr = gr.window_problem(w.cfg["window"])
    for a, b in zip(gr.edges(), es):
        assert np.array_equal(a, b)
    for k in pr:
        assert np.array_equal(pr[k], ps[k]), k
    # correlation + provider measurement on a seeded edge sample: bit-exact
    rng = np.random.default_rng(3)
    E = len(pr["e_patch"])
    sel = np.sort(rng.choice(E, size=min(E, 96), replace=False))
    prob = synth.window_arrays(w, pr)
    coords = np.empty((len(sel), 9, 2))
    for i, e in enumerate(sel):
        k = pr["e_patch"][e]
        coords[i], _ = orc.reproject_patch(pr["poses"][pr["patch_src"][k]], pr["poses"][pr["e_pose"][e]], w.K,
                                           pr["patch_x"][k], pr["patch_y"][k], pr["depth"][k])
    frames = prob["pose_frames"][pr["e_pose"][sel]]
    args = (pr["e_patch"][sel], frames, coords, prob["patch_feats"], w.level0, w.level1)
    c_ref = orc.correlate_batch(*args, threads=8)
    m_ref = orc.measure_batch(pr["e_patch"][sel], frames, coords[:, 4], None, prob["patch_feats"], w.level0,
                              w.level1, threads=8)
    with orc.using("restated"):
        c_res = orc.correlate_batch(*args, threads=8)
        m_res = orc.measure_batch(pr["e_patch"][sel], frames, coords[:, 4], None, prob["patch_feats"], w.level0,
                                  w.level1, threads=8)
    assert np.array_equal(c_ref, c_res)
    for a, b in zip(m_ref, m_res):
        assert np.array_equal(a, b)
    # optimize_window's 2 iterations on the window problem
    b_ref = orc.ba_window(pr, w.K, iterations=2)
    with orc.using("restated"):
        b_res = orc.ba_window(pr, w.K, iterations=2)
    assert np.abs(b_ref["poses"] - b_res["poses"]).max() <= 1e-8
    assert np.abs(b_ref["depth"] - b_res["depth"]).max() <= 1e-8 * max(1.0, np.abs(b_ref["depth"]).max())
    assert np.allclose(b_ref["residual_norms"], b_res["residual_norms"], rtol=1e-9)
