"""ctypes wrapper of oracle/_ref/libdynsurf_ref.so -- TEST INFRASTRUCTURE.

The UNMODIFIED reference (`/root/reference/proj/core/src`, compiled out of
tree against the repo's Eigen / GTest / libpng shims by `make -C oracle ref`,
SURVEY.md 7.1 step 1) behind a small C ABI (`oracle/ref_capi.cpp`):
`dynsurf::Pipeline::process_frame` (pipeline.cpp:74-142) plus read-back of
the surfel model and the warp nodes. Used by the oracle-vs-reference and
device-vs-reference parity tests and by the bench's CPU reference arm; the
product path never loads it. The built library travels to the GPU box with
the repo snapshot; /root/reference does not (it is only needed to build).
"""
import ctypes as C
import os
import subprocess

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SO = os.path.join(REPO, "oracle", "_ref", "libdynsurf_ref.so")
REF_TESTS = os.path.join(REPO, "oracle", "_ref", "ref_tests")
REF_SRC = "/root/reference/proj/core/src"

STAT_KEYS = ("skipped", "valid_pixels", "surfel_count", "node_count", "rigid_correspondences",
             "rigid_mean_residual", "rigid_low_confidence", "solver_iterations",
             "initial_energy", "final_energy", "solver_mean_residual", "solver_correspondences",
             "fused", "appended", "removed", "compressive_rejected", "low_support_rejected",
             "new_nodes", "degenerate_warps", "reinit", "reinit_removed")
N_STATS = len(STAT_KEYS) + 12 + 6

_lib = None


def build() -> bool:
    """Builds oracle/_ref when the reference sources are present (this
    container); returns whether the library exists."""
    if os.path.isdir(REF_SRC):
        subprocess.run(["make", "-s", "-j8", "-C", os.path.join(REPO, "oracle"), "ref"], check=True)
    return os.path.exists(REF_SO)


def available() -> bool:
    return os.path.exists(REF_SO)


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(REF_SO)
        L.dsref_create.restype = C.c_void_p
        L.dsref_create.argtypes = [C.c_char_p, C.c_char_p, C.c_int]
        L.dsref_destroy.argtypes = [C.c_void_p]
        L.dsref_process_frame.restype = C.c_int
        L.dsref_process_frame.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int,
                                          C.c_void_p, C.c_char_p, C.c_int]
        L.dsref_surfel_count.argtypes = [C.c_void_p]
        L.dsref_node_count.argtypes = [C.c_void_p]
        L.dsref_get_model.argtypes = [C.c_void_p] + [C.c_void_p] * 11
        L.dsref_get_nodes.argtypes = [C.c_void_p] + [C.c_void_p] * 4
        L.dsref_dense_solve_count.restype = C.c_longlong
        _lib = L
    return _lib


def config_text(cfg: dict) -> bytes:
    """The repo's config dict (pkg.make_config / oracle_py.make_config keys)
    as the reference's config-file lines (config.cpp key names)."""
    lines = []
    for k, v in cfg.items():
        key = "lambda" if k == "lambda_" else k
        if key in ("pcg_max_iters", "pcg_tol", "profile", "max_surfels", "max_nodes"):
            continue  # B200-side knobs: the reference has no PCG / capacities
        if isinstance(v, bool):
            v = int(v)
        lines.append(f"{key} {repr(float(v)) if isinstance(v, float) else v}")
    return "\n".join(lines).encode()


class RefPipeline:
    """dynsurf::Pipeline of the compiled reference (faithful fp64)."""

    def __init__(self, cfg: dict):
        err = C.create_string_buffer(512)
        self.h = lib().dsref_create(config_text(cfg), err, 512)
        if not self.h:
            raise RuntimeError("reference config: " + err.value.decode())

    def close(self):
        if self.h:
            lib().dsref_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def process_frame(self, depth: np.ndarray, frame_index: int) -> dict:
        d = np.ascontiguousarray(depth, dtype=np.uint16)
        out = np.zeros(N_STATS, np.float64)
        err = C.create_string_buffer(512)
        rc = lib().dsref_process_frame(self.h, d.ctypes.data, d.shape[1], d.shape[0], frame_index,
                                       out.ctypes.data, err, 512)
        if rc != 0:
            raise RuntimeError("reference process_frame: " + err.value.decode())
        st = {k: out[i] for i, k in enumerate(STAT_KEYS)}
        for k in STAT_KEYS:
            if k not in ("rigid_mean_residual", "initial_energy", "final_energy",
                         "solver_mean_residual"):
                st[k] = int(st[k])
        n = len(STAT_KEYS)
        st["pose_R"] = out[n:n + 9].reshape(3, 3).copy()
        st["pose_t"] = out[n + 9:n + 12].copy()
        st["ms"] = dict(zip(("depth", "rigid", "solve", "fusion", "reinit", "total"),
                            out[n + 12:n + 18].tolist()))
        return st

    def model(self) -> dict:
        n = lib().dsref_surfel_count(self.h)
        m = dict(ref_pos=np.zeros((n, 3)), ref_nrm=np.zeros((n, 3)), live_pos=np.zeros((n, 3)),
                 live_nrm=np.zeros((n, 3)), radius=np.zeros(n), confidence=np.zeros(n),
                 t_init=np.zeros(n, np.int32), t_obs=np.zeros(n, np.int32),
                 skin_idx=np.zeros((n, 4), np.int32), skin_w=np.zeros((n, 4)),
                 skin_count=np.zeros(n, np.int32))
        lib().dsref_get_model(self.h, *(m[k].ctypes.data for k in (
            "ref_pos", "ref_nrm", "live_pos", "live_nrm", "radius", "confidence", "t_init",
            "t_obs", "skin_idx", "skin_w", "skin_count")))
        return m

    def nodes(self) -> dict:
        N = lib().dsref_node_count(self.h)
        nd = dict(pos=np.zeros((N, 3)), sigma=np.zeros(N), dq=np.zeros((N, 8)),
                  nbr=np.zeros((N, 8), np.int32))
        lib().dsref_get_nodes(self.h, *(nd[k].ctypes.data for k in ("pos", "sigma", "dq", "nbr")))
        return nd


def set_dense_solver(fn_ptr):
    """Routes the reference's dense LM-step LDLT (solver.cpp:386) to an
    external solver (a ctypes callback: n, a, b, x -> int), None restores it."""
    L = lib()
    L.dsref_set_dense_solver.argtypes = [C.c_void_p]
    L.dsref_set_dense_solver(C.cast(fn_ptr, C.c_void_p) if fn_ptr is not None else None)


def dense_solve_count() -> int:
    return int(lib().dsref_dense_solve_count())
