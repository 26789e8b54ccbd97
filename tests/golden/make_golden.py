"""Regenerate the golden fixtures (see cases.py):

* golden_ref_v1.npz - outputs of the REFERENCE's own code (oracle/_ref,
  built from /root/reference/proj/src by oracle/ref_build.py): the golden
  vectors the GPU suite checks the product against;
* golden_v1.npz     - the same cases through the restatement (oracle drift check).

    python tests/golden/make_golden.py
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import oracle.pyoracle as orc  # noqa: E402
from tests.golden import cases  # noqa: E402


def build() -> dict:
    out = {}
    c = cases.corr_case()
    out["corr_inputs_sha"] = np.array(cases.digest(*c.values()))
    out["corr_out"] = orc.correlate_batch(c["e_patch"], c["e_frame"], c["coords"], c["feats"], c["level0"],
                                          c["level1"])
    centers = c["coords"][:, 4, :]
    d, wt, fl = orc.measure_batch(c["e_patch"], c["e_frame"], centers, None, c["feats"], c["level0"], c["level1"])
    out["measure_delta"], out["measure_weight"], out["measure_flags"] = d, wt, fl
    w, prob = cases.ba_case()
    out["ba_inputs_sha"] = np.array(cases.digest(*[prob[k] for k in sorted(prob)]))
    ref = orc.ba_window(prob, w.K, iterations=2)
    out["ba_poses"], out["ba_depth"] = ref["poses"], ref["depth"]
    out["ba_norms"] = np.asarray(ref["residual_norms"], np.float64)
    f = cases.features_case()
    out["feat_inputs_sha"] = np.array(cases.digest(*f.values()))
    l0, l1 = orc.extract_features(f["image"], base_channels=1)
    out["feat_level0"], out["feat_level1"] = l0, l1
    out["feat_crops"] = orc.crop_patches(f["px"], f["py"], l0, l1)
    return out


if __name__ == "__main__":
    here = Path(__file__).resolve().parent
    with orc.using("restated"):
        np.savez_compressed(here / "golden_v1.npz", **build())
    with orc.using("reference"):
        np.savez_compressed(here / "golden_ref_v1.npz", **build())
    for name in ("golden_v1.npz", "golden_ref_v1.npz"):
        print(here / name, (here / name).stat().st_size, "bytes")
