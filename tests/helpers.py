"""Shared test helpers: seeded random twists/poses (proj/tests/helpers.hpp:9-27)."""
import numpy as np

import oracle.pyoracle as orc


def random_unit(rng):
    v = rng.standard_normal(3)
    while np.linalg.norm(v) < 1e-6:
        v = rng.standard_normal(3)
    return v / np.linalg.norm(v)


def random_twist(rng, trans_scale, max_angle):
    trans = trans_scale * rng.standard_normal(3)
    rot = rng.uniform() * max_angle * random_unit(rng)
    return np.concatenate([trans, rot])


def random_pose(rng, trans_scale=1.0, max_angle=2.5):
    return orc.se3_exp(random_twist(rng, trans_scale, max_angle))


def pose_parity(a, b):
    """max |dt| and max |dq| with the quaternion sign fixed."""
    a, b = np.asarray(a).reshape(-1, 7), np.asarray(b).reshape(-1, 7)
    sgn = np.sign((a[:, :4] * b[:, :4]).sum(1, keepdims=True))
    sgn[sgn == 0] = 1
    dq = np.abs(a[:, :4] - sgn * b[:, :4]).max(1)
    dt = np.abs(a[:, 4:] - b[:, 4:]).max(1)
    return dt, dq


def smooth_features(rng, H, W, D):
    """Blurred, unit-norm random feature grid (the synth generator's recipe)."""
    import pvo_synth as synth

    return synth.make_level0(rng, 1, H, W, D)[0]
