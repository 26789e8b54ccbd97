"""B200-native (sm_100a) DPVO geometric hot path: patch reprojection,
normalised patch-to-frame correlation and sparse Gauss-Newton bundle
adjustment, behind the reference's operator API (see include/pvo_capi.h).

Importing the package loads the in-tree ``libpvo_b200.so``; it raises if the
library has not been built (there is no CPU fallback).
"""
from .api import (  # noqa: F401
    IDENTITY,
    BAProblem,
    Batch,
    BASolution,
    Context,
    CudaError,
    DegenerateProblem,
    DeviceGraph,
    NormalEquations,
    Patch,
    PatchGraph,
    ReprojectionJacobians,
    Unsupported,
    Window,
    WindowOptions,
    ba_window,
    build_target,
    compose,
    correlate,
    correlate_at,
    correlate_at_cubic,
    correlate_batch,
    correlate_points,
    grid_cache_stats,
    default_context,
    gauss_newton_step,
    inverse,
    measure_batch,
    optimize_window,
    reproject_patch,
    reproject_patches,
    reprojection_jacobians,
    reprojection_jacobians_batch,
    retract,
    schur_solve,
    se3_exp,
    se3_log,
    window_problem_read,
)
from ._capi import lib  # noqa: F401

__all__ = [n for n in dir() if not n.startswith("_")]
