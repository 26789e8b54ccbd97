"""Golden fixtures (tests/golden/).  golden_ref_v1.npz holds the REFERENCE's
own outputs (its sources compiled into oracle/_ref by oracle/ref_build.py);
golden_v1.npz the restatement's.  CPU suite: each backend reproduces its file
bit for bit, and the restatement agrees with the reference (bit-exact
correlation / measurement / features, 1e-8 BA).  GPU suite: the B200 path
matches the reference's golden outputs within the parity tolerances, without
any oracle in the loop.  See tests/golden/cases.py for the cases."""
from pathlib import Path

import numpy as np
import pytest

from tests.golden import cases

GOLDEN = Path(__file__).resolve().parent / "golden" / "golden_v1.npz"
GOLDEN_REF = Path(__file__).resolve().parent / "golden" / "golden_ref_v1.npz"
EXACT = ["corr_out", "measure_delta", "measure_weight", "measure_flags", "feat_level0", "feat_level1", "feat_crops"]


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLDEN_REF)


@pytest.fixture(scope="module")
def golden_restated():
    return np.load(GOLDEN)


def test_golden_inputs_are_stable(golden):
    c = cases.corr_case()
    assert str(golden["corr_inputs_sha"]) == cases.digest(*c.values())
    _, prob = cases.ba_case()
    assert str(golden["ba_inputs_sha"]) == cases.digest(*[prob[k] for k in sorted(prob)])
    f = cases.features_case()
    assert str(golden["feat_inputs_sha"]) == cases.digest(*f.values())


def test_oracle_reproduces_golden(golden_restated):
    import oracle.pyoracle as orc
    from tests.golden.make_golden import build

    with orc.using("restated"):
        fresh = build()
    for k in golden_restated.files:
        assert np.array_equal(fresh[k], golden_restated[k]), k


def test_reference_reproduces_golden(golden):
    import oracle.pyoracle as orc
    from tests.golden.make_golden import build

    if orc.lib_ref is None:
        pytest.skip("oracle/_ref not built (no /root/reference here)")
    with orc.using("reference"):
        fresh = build()
    for k in golden.files:
        assert np.array_equal(fresh[k], golden[k]), k


def test_restatement_pinned_to_reference(golden, golden_restated):
    for k in EXACT:
        assert np.array_equal(golden[k], golden_restated[k]), k
    for k in ["ba_poses", "ba_depth", "ba_norms"]:
        ref, res = golden[k], golden_restated[k]
        assert np.abs(ref - res).max() <= 1e-8 * max(1.0, np.abs(ref).max()), k


@pytest.mark.gpu
def test_gpu_matches_golden(golden):
    import paper_2208_04726_b200 as pvo
    from tests.helpers import pose_parity
    from tests.test_gpu_parity import _gnorm_for_batch, _measure_report, corr_violations

    ctx = pvo.Context(0)
    try:
        c = cases.corr_case()
        F, H0, W0, D = c["level0"].shape
        _, H1, W1, _ = c["level1"].shape
        ctx.frames_reserve(F, W0, H0, W1, H1, D)
        for f in range(F):
            ctx.frames_upload(f, c["level0"][f], c["level1"][f])
        out = pvo.correlate_batch(c["e_patch"], c["e_frame"], c["coords"], c["feats"], ctx=ctx)
        assert corr_violations(out, golden["corr_out"], _gnorm_for_batch(c["feats"], c["e_patch"])) == 0
        assert np.all(out[3] == 0) and np.all(out[10] == 0)  # far outside the frame: all zero padding
        d, w, fl = pvo.measure_batch(c["e_patch"], c["e_frame"], c["coords"][:, 4, :], c["feats"], ctx=ctx)
        flips, off = _measure_report("golden measure", d, w, fl, golden["measure_delta"], golden["measure_weight"],
                                     golden["measure_flags"])
        assert flips == 0 and off == 0
        w_, prob = cases.ba_case()
        pr = pvo.BAProblem(prob["poses"], prob["fixed"].astype(bool), prob["patch_src"], prob["patch_x"],
                           prob["patch_y"], prob["depth"], prob["e_patch"], prob["e_pose"], prob["e_target"],
                           prob["e_weight"], w_.K)
        sol = pvo.ba_window(pr, iterations=2, ctx=ctx)
        dt, dq = pose_parity(sol.poses, golden["ba_poses"])
        assert dt.max() <= 1e-6 and dq.max() <= 1e-6
        assert np.allclose(sol.inverse_depths, golden["ba_depth"], rtol=1e-6, atol=1e-9)
        assert np.allclose(sol.residual_norms, golden["ba_norms"], rtol=1e-6)
        fcase = cases.features_case()
        l0, l1 = golden["feat_level0"], golden["feat_level1"]
        ctx.frames_reserve(1, l0.shape[1], l0.shape[0], l1.shape[1], l1.shape[0], l0.shape[2])
        ctx.frames_extract(0, fcase["image"], base_channels=1)
        g0, g1 = ctx.frames_download(0)
        assert np.array_equal(g0, l0) and np.array_equal(g1, l1)
        assert np.array_equal(ctx.crop_patches(0, fcase["cents"]), golden["feat_crops"])
    finally:
        ctx.close()
