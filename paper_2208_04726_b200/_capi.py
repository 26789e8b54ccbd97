"""ctypes declarations of the C-ABI in include/pvo_capi.h.

Loads the in-tree ``libpvo_b200.so`` (built by ``build.py``).  There is no
fallback: if the library is missing the import raises, and every compute
entry returns PVO_CUDA_ERROR without an sm_100 device.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_LIB_PATH = Path(__file__).resolve().parent / "libpvo_b200.so"

PVO_OK = 0
PVO_INVALID_ARGUMENT = 1
PVO_DEGENERATE = 2
PVO_DOMAIN_ERROR = 3
PVO_OUT_OF_RANGE = 4
PVO_CUDA_ERROR = 5
PVO_UNSUPPORTED = 6
PVO_HOST = 0
PVO_DEVICE = 1

i32, i64, f64, vp = C.c_int, C.c_int64, C.c_double, C.c_void_p
P = vp  # every array argument is passed as a raw address

# name -> (restype, argtypes)
SIGNATURES = {
    "pvo_version": (i32, []),
    "pvo_last_error": (C.c_char_p, []),
    "pvo_status_string": (C.c_char_p, [i32]),
    "pvo_ctx_create": (i32, [i32, C.POINTER(vp)]),
    "pvo_ctx_destroy": (i32, [vp]),
    "pvo_ctx_set_stream": (i32, [vp, vp]),
    "pvo_ctx_synchronize": (i32, [vp]),
    "pvo_ctx_kernel_launches": (i64, [vp]),
    "pvo_ctx_last_timing": (i32, [vp, P, P]),
    "pvo_ctx_ba_attempts": (i32, [vp, P]),
    "pvo_ctx_set_tracing": (i32, [vp, i32]),
    "pvo_ctx_set_timing": (i32, [vp, i32]),
    "pvo_ctx_ba_phase_cycles": (i32, [vp, P]),
    "pvo_se3_exp": (i32, [P, P]),
    "pvo_se3_log": (i32, [P, P]),
    "pvo_se3_compose": (i32, [P, P, P]),
    "pvo_se3_inverse": (i32, [P, P]),
    "pvo_se3_retract": (i32, [P, P, P]),
    "pvo_reproject_patches": (i32, [vp, i32, i32, P, P, P, P, P, P, P, P]),
    "pvo_reprojection_jacobians": (i32, [vp, i32, i32, P, P, P, P, P, P, P, P]),
    "pvo_correlate": (i32, [vp, i32, i32, P, P, P, i32, i32, P, i32, i32, P, P]),
    "pvo_correlate_points": (i32, [vp, i32, i32, P, P, i32, i32, P, i32, P]),
    "pvo_grid_cache_stats": (i32, [vp, P, P, P, P]),
    "pvo_grid_cache_clear": (i32, [vp]),
    "pvo_frames_reserve": (i32, [vp, i32, i32, i32, i32, i32, i32]),
    "pvo_frames_upload": (i32, [vp, i32, P, P, i32]),
    "pvo_frames_refresh": (i32, [vp, i32]),
    "pvo_frames_device_ptrs": (i32, [vp, P, P]),
    "pvo_correlate_batch": (i32, [vp, i32, i32, i32, P, P, P, P, P, i32]),
    "pvo_gauss_newton_step": (i32, [vp, i32, P, P, i32, i32, P, P, P, P, P, i32, P, P, P, P, P, f64,
                                    P, P, P, P, P, P, P]),
    "pvo_schur_solve": (i32, [vp, i32, i32, P, P, P, P, P, P, P]),
    "pvo_ba_window": (i32, [vp, i32, P, P, i32, i32, P, P, P, P, i32, P, P, P, P, P, i32, i32, i32, f64,
                            i32, i32, P, P, P, P]),
    "pvo_window_load": (i32, [vp, i32, P, P, P, i32, i32, P, P, P, P, P, i32, P, P, P, P, P, i32, i32, i32]),
    "pvo_window_set_state": (i32, [vp, P, P, i32]),
    "pvo_window_iteration": (i32, [vp, i32, f64, P, i32]),
    "pvo_window_correlate": (i32, [vp, P, i32]),
    "pvo_window_ba": (i32, [vp, i32, f64]),
    "pvo_window_read": (i32, [vp, P, P, P, P]),
    "pvo_window_corr_ptr": (i32, [vp, P]),
    "pvo_frames_extract": (i32, [vp, i32, P, i32, i32, i32, i32]),
    "pvo_crop_patches": (i32, [vp, i32, i32, P, P, i32]),
    "pvo_frames_download": (i32, [vp, i32, P, P]),
    "pvo_measure_batch": (i32, [vp, i32, i32, i32, P, P, P, P, P, P, P, P]),
    "pvo_window_propose": (i32, [vp, P, P, P]),
    "pvo_measure_replayed": (i32, [vp, P]),
    "pvo_dgraph_create": (i32, [vp, P, i32, i32, i32, i32, C.POINTER(vp)]),
    "pvo_dgraph_destroy": (i32, [vp]),
    "pvo_dgraph_reserve": (i32, [vp, i32, i32, i32]),
    "pvo_dgraph_add_frame": (i32, [vp, f64, P, i32, P]),
    "pvo_dgraph_add_patches": (i32, [vp, i32, i32, P, P, P, P]),
    "pvo_dgraph_connect": (i32, [vp, i32, P]),
    "pvo_dgraph_remove_frame": (i32, [vp, i32]),
    "pvo_dgraph_set_revisions": (i32, [vp, i32, P, P, P, P]),
    "pvo_dgraph_counts": (i32, [vp, P, P, P]),
    "pvo_dgraph_keyframe": (i32, [vp, f64, P, P, P]),
    "pvo_dgraph_edges": (i32, [vp, P, P, P, P]),
    "pvo_dgraph_frames": (i32, [vp, P, P]),
    "pvo_dgraph_patches": (i32, [vp, P, P, P]),
    "pvo_window_load_dgraph": (i32, [vp, vp, i32, i32, P, P, P]),
    "pvo_dgraph_store_window": (i32, [vp, vp, i32, i32]),
    "pvo_window_problem_read": (i32, [vp, P, P, P, P, P, P, P, P, P, P, P]),
    "pvo_oracle_seed": (i32, [vp, C.c_uint64]),
    "pvo_window_oracle_propose": (i32, [vp, P, P, f64, f64, P, P]),
    "pvo_batch_load": (i32, [vp, i32, P, P, P, P, P, P, i32, P, P, P, P, P, P, P, P, P, P, i32, i32]),
    "pvo_batch_reset": (i32, [vp]),
    "pvo_batch_iteration": (i32, [vp, i32, f64, P, i32]),
    "pvo_batch_read": (i32, [vp, P, P, P, P]),
    "pvo_batch_norm_stride": (i32, []),
    "pvo_graph_create": (i32, [P, i32, i32, i32, C.POINTER(vp)]),
    "pvo_graph_destroy": (i32, [vp]),
    "pvo_graph_add_frame": (i32, [vp, f64, P, P]),
    "pvo_graph_add_patches": (i32, [vp, i32, i32, P, P, P]),
    "pvo_graph_connect": (i32, [vp, i32, P]),
    "pvo_graph_remove_frame": (i32, [vp, i32]),
    "pvo_graph_set_revision": (i32, [vp, i32, i32, P, P]),
    "pvo_graph_set_pose": (i32, [vp, i32, P]),
    "pvo_graph_set_inverse_depth": (i32, [vp, i32, f64]),
    "pvo_graph_num_frames": (i32, [vp]),
    "pvo_graph_num_patches": (i32, [vp]),
    "pvo_graph_num_edges": (i32, [vp]),
    "pvo_graph_edges": (i32, [vp, P, P, P, P]),
    "pvo_graph_frames": (i32, [vp, P, P]),
    "pvo_graph_patches": (i32, [vp, P, P, P]),
    "pvo_graph_active_edges": (i32, [vp, i32, P, P, P]),
    "pvo_graph_build_target": (i32, [vp, i32, i32, P]),
    "pvo_graph_window_problem": (i32, [vp, i32, P, P, P, P, P, P, P, P, P, P, P, P, P, P, P]),
    "pvo_optimize_window": (i32, [vp, vp, i32, i32, i32, f64, P, P, P]),
}


def load(path: Path | str | None = None) -> C.CDLL:
    # PVO_LIB: an alternative build of the same library (A/B kernel variants)
    p = Path(path or os.environ.get("PVO_LIB") or _LIB_PATH)
    if not p.exists():
        raise ImportError(
            f"{p} is missing: build the sm_100a library first "
            "(python paper_2208_04726_b200/build.py); there is no CPU fallback"
        )
    lib = C.CDLL(str(p))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = load()
