"""Loader + ctypes signatures of libdynsurf_b200.so (include/dynsurf_b200.h).

The library is built in-tree (paper_1904_13073_b200/lib/) by
`__graft_entry__.build()` / `make -C paper_1904_13073_b200`. There is no
Python or CPU fallback: importing this module without the built library
raises ImportError, and every compute call on a machine without a CUDA device
fails with CudaError.
"""
from __future__ import annotations

import ctypes as C
import os

from . import errors

PKG = os.path.dirname(os.path.abspath(__file__))
# DS_LIB_PATH: load another build of the library (A/B timing of two builds)
LIB_PATH = os.environ.get("DS_LIB_PATH") or os.path.join(PKG, "lib", "libdynsurf_b200.so")

CONFIG_FIELDS = [
    ("node_sigma", C.c_double), ("knn_k", C.c_int32), ("node_neighbor_k", C.c_int32),
    ("lambda_", C.c_double), ("max_gn_iters", C.c_int32), ("_pad0", C.c_int32),
    ("delta_distance", C.c_double), ("delta_normal", C.c_double), ("epsilon", C.c_double),
    ("delta_stable", C.c_double), ("t_low_confid", C.c_int32), ("delta_recent", C.c_int32),
    ("delta_nn", C.c_double), ("supersample_factor", C.c_int32),
    ("compressive_check", C.c_int32), ("depth_min", C.c_double), ("depth_max", C.c_double),
    ("bilateral_filter", C.c_int32), ("_pad1", C.c_int32),
    ("bilateral_sigma_space", C.c_double), ("bilateral_sigma_depth", C.c_double),
    ("reinit_energy_threshold", C.c_double), ("reinit_append_threshold", C.c_int32),
    ("reinit_window", C.c_int32), ("periodic_reinit_interval", C.c_int32),
    ("_pad2", C.c_int32), ("delta_distance_reinit", C.c_double),
    ("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
    ("width", C.c_int32), ("height", C.c_int32),
    # device-only
    ("pcg_max_iters", C.c_int32), ("max_surfels", C.c_int32), ("pcg_tol", C.c_double),
    ("max_nodes", C.c_int32), ("profile", C.c_int32),
]


class DsConfig(C.Structure):
    _fields_ = CONFIG_FIELDS


class DsSolverReport(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("correspondences", C.c_int32),
                ("initial_energy", C.c_double), ("final_energy", C.c_double),
                ("mean_residual", C.c_double)]


class DsRigidResult(C.Structure):
    _fields_ = [("pose", C.c_double * 12), ("correspondences", C.c_int32),
                ("low_confidence", C.c_int32), ("mean_residual", C.c_double)]


class DsFusionOutcome(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("fused", "appended", "removed",
                                          "compressive_rejected", "low_support_rejected",
                                          "new_nodes", "degenerate_warps", "_pad")]


class DsFrameStats(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("frame", "skipped", "valid_pixels", "surfel_count",
                                          "node_count", "reinit", "reinit_removed", "_pad")] + [
        ("rigid", DsRigidResult), ("solver", DsSolverReport), ("fusion", DsFusionOutcome),
        ("pose", C.c_double * 12),
    ] + [(n, C.c_double) for n in ("depth_ms", "rigid_ms", "solve_ms", "fusion_ms",
                                   "reinit_ms", "total_ms")] + [
        (n, C.c_int32) for n in ("lm_attempts", "pcg_iterations", "gn_blocks",
                                 "kernel_launches")]


P = C.c_void_p
I32 = C.c_int32
PI32 = C.POINTER(C.c_int32)
PD = C.POINTER(C.c_double)

# name -> argtypes (all return ds_status / int32 unless listed in _RESTYPE)
SIGNATURES = {
    "ds_default_config": [C.POINTER(DsConfig)],
    "ds_last_error": [],
    "ds_version": [],
    "ds_validate_config": [C.POINTER(DsConfig)],
    "ds_create": [C.POINTER(DsConfig), I32, P, C.POINTER(P)],
    "ds_destroy": [P],
    "ds_synchronize": [P],
    "ds_join_deferred": [P],
    "ds_capacity": [P, PI32, PI32, PI32],
    "ds_process_frame": [P, P, I32, I32, I32, C.POINTER(DsFrameStats)],
    "ds_process_frame_device": [P, P, I32, I32, I32, C.POINTER(DsFrameStats)],
    "ds_is_initialized": [P, PI32, PI32],
    "ds_reset": [P],
    "ds_upload_model": [P, I32] + [P] * 11,
    "ds_model_size": [P, PI32],
    "ds_download_model": [P] + [P] * 11,
    "ds_upload_nodes": [P, I32] + [P] * 5,
    "ds_num_nodes": [P, PI32],
    "ds_download_nodes": [P] + [P] * 5,
    "ds_set_pose": [P, P],
    "ds_get_pose": [P, P],
    "ds_frame_maps": [P, P, I32, I32, I32, PI32],
    "ds_download_frame": [P] + [P] * 6,
    "ds_upload_frame": [P, I32, I32, I32] + [P] * 6,
    "ds_init_warp_field": [P],
    "ds_compute_node_edges": [P],
    "ds_forward_warp": [P, PI32],
    "ds_render_index_map": [P, P, I32, P],
    "ds_render_model_maps": [P, P, I32, I32, P, P, P, P, P],
    "ds_associate": [P, P, I32, PI32, P, P, P, P, P, P],
    "ds_build_normal_equations": [P, P, I32, I32, PI32, PI32, PD],
    "ds_download_normal_equations": [P, P, P, P, P, P],
    "ds_pcg_solve": [P, C.c_double, I32, C.c_double, P, PI32, PD],
    "ds_check_normal_equations": [P],
    "ds_set_normal_equation_values": [P, P, P],
    "ds_bsr_spmv": [P, P, P, C.c_double, I32, PD],
    "ds_solve_nonrigid": [P, P, I32, I32, C.POINTER(DsSolverReport)],
    "ds_rigid_align": [P, P, P, I32, I32, C.POINTER(DsRigidResult)],
    "ds_apply_fusion": [P, P, I32, C.POINTER(DsFusionOutcome)],
    "ds_fuse_depth": [P, P, I32, PI32, PI32],
    "ds_download_candidates": [P] + [P] * 6,
    "ds_skin_appended": [P, I32] + [P] * 7,
    "ds_remove_mask": [P, P, I32, P],
    "ds_extend_warp_field": [P, I32, P, PI32],
    "ds_update_skinning_incremental": [P, I32],
    "ds_clean_and_reset": [P, P, PI32, PI32],
    "ds_num_kernel_kinds": [],
    "ds_kernel_name": [I32],
    "ds_kernel_stats": [P, I32, C.POINTER(C.c_int64), PD, PD],
    "ds_reset_kernel_stats": [P],
    "ds_set_profiling": [P, I32],
    "ds_total_launches": [P, C.POINTER(C.c_int64)],
    "ds_png_unfilter": [P, C.c_int64, I32, I32, I32, P],
}

_RESTYPE = {
    "ds_default_config": None,
    "ds_last_error": C.c_char_p,
    "ds_kernel_name": C.c_char_p,
}

# The synthetic depth-stream generator (synth.hpp:16-73) is a host-only library
# of its own (synth/lib/libdynsurf_synth.so): generating inputs never maps the
# CUDA library, so the CPU reference arm of bench.py runs without it.
SYNTH_PATH = os.environ.get("DS_SYNTH_LIB_PATH") or os.path.join(
    os.path.dirname(PKG), "synth", "lib", "libdynsurf_synth.so")
SYNTH_SIGNATURES = {
    "ds_synth_scenario": ([C.c_char_p], C.c_int32),
    "ds_synth_scenario_name": ([I32], C.c_char_p),
    "ds_synth_default_frames": ([I32], C.c_int32),
    "ds_synth_render_depth": ([I32, I32, C.POINTER(DsConfig), C.c_double, C.c_uint32, I32, P],
                              C.c_int32),
    "ds_synth_camera_pose": ([I32, I32, I32, P], C.c_int32),
    "ds_synth_surface_distance": ([I32, I32, P, I32], C.c_double),
}

_lib = None


def load():
    """Load the in-tree library (fails loudly if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            f"g.build()'` (no CPU fallback exists for the B200 path)")
    L = C.CDLL(LIB_PATH)
    for name, args in SIGNATURES.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = _RESTYPE.get(name, C.c_int32)
    _lib = L
    return L


_synth = None


def load_synth():
    """Load the in-tree synthetic-scene library (host code only)."""
    global _synth
    if _synth is not None:
        return _synth
    if not os.path.exists(SYNTH_PATH):
        raise ImportError(f"{SYNTH_PATH} is missing: build it with `make -C synth`")
    L = C.CDLL(SYNTH_PATH)
    for name, (args, res) in SYNTH_SIGNATURES.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _synth = L
    return L


def check_synth(status: int) -> None:
    if status != 0:
        raise errors.from_status(status, "synthetic scene generator: invalid argument")


def check(status: int) -> None:
    if status != 0:
        msg = load().ds_last_error().decode(errors="replace")
        raise errors.from_status(status, msg)
