"""ctypes wrapper of the CPU fp64 oracle (oracle/dynsurf_oracle.h).

TEST INFRASTRUCTURE ONLY: the checker the CUDA product is compared with.
Arrays are numpy, fp64 / int32 / uint8, C-contiguous, in the host layouts
documented in oracle/dynsurf_oracle.h.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(REPO, "oracle")
ORACLE_SO = os.path.join(ORACLE_DIR, "build", "liboracle.so")

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
]


class OrConfig(C.Structure):
    _fields_ = CONFIG_FIELDS


class OrSolverReport(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("correspondences", C.c_int32),
                ("initial_energy", C.c_double), ("final_energy", C.c_double),
                ("mean_residual", C.c_double)]


class OrRigidResult(C.Structure):
    _fields_ = [("pose", C.c_double * 12), ("correspondences", C.c_int32),
                ("low_confidence", C.c_int32), ("mean_residual", C.c_double)]


class OrFusionOutcome(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("fused", "appended", "removed",
                                          "compressive_rejected", "low_support_rejected",
                                          "new_nodes", "degenerate_warps", "_pad")]


class OrFrameStats(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("frame", "skipped", "valid_pixels", "surfel_count",
                                          "node_count", "reinit", "reinit_removed", "_pad")] + [
        ("rigid", OrRigidResult), ("solver", OrSolverReport), ("fusion", OrFusionOutcome),
        ("pose", C.c_double * 12),
    ] + [(n, C.c_double) for n in ("depth_ms", "rigid_ms", "solve_ms", "fusion_ms",
                                   "reinit_ms", "total_ms")]


DEFAULTS = dict(
    node_sigma=0.025, knn_k=4, node_neighbor_k=8, lambda_=5.0, max_gn_iters=10,
    delta_distance=0.001, delta_normal=0.85, epsilon=0.2, delta_stable=10.0,
    t_low_confid=30, delta_recent=2, delta_nn=0.03, supersample_factor=4,
    compressive_check=1, depth_min=0.1, depth_max=5.0, bilateral_filter=0,
    bilateral_sigma_space=4.5, bilateral_sigma_depth=30.0, reinit_energy_threshold=0.005,
    reinit_append_threshold=3000, reinit_window=3, periodic_reinit_interval=0,
    delta_distance_reinit=0.010, fx=0.0, fy=0.0, cx=0.0, cy=0.0, width=0, height=0,
)


def make_config(**kw) -> dict:
    """PipelineConfig{} (config.hpp:11-50) with overrides; `lambda` may be passed as lambda_."""
    cfg = dict(DEFAULTS)
    if "lambda" in kw:
        kw["lambda_"] = kw.pop("lambda")
    for k, v in kw.items():
        if k not in cfg:
            raise KeyError(k)
        cfg[k] = v
    return cfg


def test_config(**kw) -> dict:
    """test_util.hpp:81-89: 160x120, f=140, c=(79.5, 59.5)."""
    base = dict(fx=140.0, fy=140.0, width=160, height=120, cx=79.5, cy=59.5)
    base.update(kw)
    return make_config(**base)


def to_struct(cfg: dict, cls=OrConfig):
    s = cls()
    for name, _ in cls._fields_:
        if name.startswith("_pad"):
            continue
        if name in cfg:
            setattr(s, name, cfg[name])
    return s


_lib = None


def build_oracle() -> str:
    subprocess.run(["make", "-s", "-C", ORACLE_DIR], check=True)
    return ORACLE_SO


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(ORACLE_SO):
        build_oracle()
    L = C.CDLL(ORACLE_SO)
    P = C.c_void_p
    L.or_state_new.restype = P
    L.or_state_new.argtypes = [C.POINTER(OrConfig)]
    L.or_state_free.argtypes = [P]
    L.or_state_set_config.argtypes = [P, C.POINTER(OrConfig)]
    L.or_model_size.argtypes = [P]
    L.or_num_nodes.argtypes = [P]
    L.or_last_error.restype = C.c_char_p
    L.or_pipeline_new.restype = P
    L.or_pipeline_new.argtypes = [C.POINTER(OrConfig), C.c_int32]
    L.or_pipeline_free.argtypes = [P]
    L.or_pipeline_state.restype = P
    L.or_pipeline_state.argtypes = [P]
    L.or_pipeline_process_frame.argtypes = [P, P, C.c_int32, C.c_int32, C.c_int32, P]
    L.or_pipeline_pose.argtypes = [P, P]
    L.or_pipeline_last_reinit.argtypes = [P]
    for fn in ("or_skinning_weight", "or_compute_confidence", "or_compute_radius",
               "or_data_energy", "or_reg_energy", "or_sigma_max3"):
        getattr(L, fn).restype = C.c_double
    L.or_compute_radius.argtypes = [C.c_double, C.c_double, C.c_double]
    L.or_compute_confidence.argtypes = [C.c_double, C.c_double, C.POINTER(OrConfig)]
    L.or_skinning_weight.argtypes = [P, P, C.c_double]
    L.or_voxel_knn.argtypes = [P, C.c_int32, C.c_double, P, C.c_int32, P]
    L.or_voxel_has_point_within.argtypes = [P, C.c_int32, C.c_double, P, C.c_double]
    L.or_bilateral_filter.argtypes = [P, C.c_int32, C.c_int32, C.c_double, C.c_double, P]
    _lib = L
    return L


def ptr(a):
    if a is None:
        return None
    return a.ctypes.data_as(C.c_void_p)


def f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a.reshape(shape) if shape is not None else a


def i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def u8(a):
    return np.ascontiguousarray(a, dtype=np.uint8)


# ------------------------------------------------------------------ geometry
def pose_identity():
    p = np.zeros(12)
    p[[0, 4, 8]] = 1.0
    return p


def pose_from(R, t):
    p = np.zeros(12)
    p[:9] = np.asarray(R, dtype=np.float64).reshape(9)
    p[9:] = t
    return p


def pose_R(p):
    return np.asarray(p[:9]).reshape(3, 3)


def pose_t(p):
    return np.asarray(p[9:12])


def quat_from_rotvec(om):
    q = np.zeros(4)
    lib().or_quat_from_rotvec(ptr(f64(om)), ptr(q))
    return q


def matrix_from_quat(q):
    r = np.zeros(9)
    lib().or_matrix_from_quat(ptr(f64(q)), ptr(r))
    return r.reshape(3, 3)


def quat_from_matrix(R):
    q = np.zeros(4)
    lib().or_quat_from_matrix(ptr(f64(R).reshape(9)), ptr(q))
    return q


def make_se3(axis_angle, translation):
    """test_util.hpp:14-19"""
    return pose_from(matrix_from_quat(quat_from_rotvec(axis_angle)), translation)


def random_se3(rng, max_angle=0.5, max_shift=0.2):
    """test_util.hpp:21-29 (numpy RNG)"""
    axis = rng.uniform(-1, 1, 3)
    if np.linalg.norm(axis) < 1e-6:
        axis = np.array([1.0, 0, 0])
    axis /= np.linalg.norm(axis)
    ang = rng.uniform(0, max_angle)
    sh = rng.uniform(-max_shift, max_shift, 3)
    return make_se3(axis * ang, sh)


def random_point(rng, extent=0.3):
    return rng.uniform(-extent, extent, 3)


def se3_mul(a, b):
    Ra, Rb = pose_R(a), pose_R(b)
    return pose_from(Ra @ Rb, Ra @ pose_t(b) + pose_t(a))


def se3_apply(p, x):
    return pose_R(p) @ np.asarray(x) + pose_t(p)


def se3_inverse(p):
    Rt = pose_R(p).T
    return pose_from(Rt, -(Rt @ pose_t(p)))


def dq_from_se3(pose):
    d = np.zeros(8)
    lib().or_dq_from_se3(ptr(f64(pose)), ptr(d))
    return d


def dq_to_se3(dq):
    p = np.zeros(12)
    lib().or_dq_to_se3(ptr(f64(dq)), ptr(p))
    return p


def dq_mul(a, b):
    o = np.zeros(8)
    lib().or_dq_mul(ptr(f64(a)), ptr(f64(b)), ptr(o))
    return o


def dq_normalized(a):
    o = np.zeros(8)
    lib().or_dq_normalized(ptr(f64(a)), ptr(o))
    return o


def dq_increment(om, dt):
    o = np.zeros(8)
    lib().or_dq_increment(ptr(f64(om)), ptr(f64(dt)), ptr(o))
    return o


def dq_apply(dq, p):
    return se3_apply(dq_to_se3(dq), p)


def blend(dqs, weights):
    dqs = f64(dqs).reshape(-1, 8)
    w = f64(weights)
    o = np.zeros(8)
    ok = lib().or_blend(len(w), ptr(dqs), ptr(w), ptr(o))
    return o if ok else None


def skinning_weight(x, p, sigma):
    return lib().or_skinning_weight(ptr(f64(x)), ptr(f64(p)), sigma)


def se3_increment(om, dt, pose):
    o = np.zeros(12)
    lib().or_se3_increment(ptr(f64(om)), ptr(f64(dt)), ptr(f64(pose)), ptr(o))
    return o


IDENTITY_DQ = np.array([1.0, 0, 0, 0, 0, 0, 0, 0])


# ------------------------------------------------------------------ model
def make_surfel(position, normal=(0, 0, -1), radius=0.004, confidence=1.0, t_init=0):
    """test_util.hpp:36-47"""
    n = np.asarray(normal, dtype=np.float64)
    return dict(pos=np.asarray(position, dtype=np.float64), nrm=n / np.linalg.norm(n),
                radius=float(radius), conf=float(confidence), t_init=int(t_init),
                t_obs=int(t_init))


def model_from_surfels(surfels, skin_idx=None, skin_w=None, skin_count=None):
    n = len(surfels)
    pos = np.array([s["pos"] for s in surfels], dtype=np.float64).reshape(n, 3)
    nrm = np.array([s["nrm"] for s in surfels], dtype=np.float64).reshape(n, 3)
    rad = np.array([s["radius"] for s in surfels], dtype=np.float64)
    conf = np.array([s["conf"] for s in surfels], dtype=np.float64)
    ti = np.array([s["t_init"] for s in surfels], dtype=np.int32)
    to = np.array([s["t_obs"] for s in surfels], dtype=np.int32)
    m = dict(ref_pos=pos.copy(), ref_nrm=nrm.copy(), ref_radius=rad.copy(), ref_conf=conf.copy(),
             ref_t_init=ti.copy(), ref_t_obs=to.copy(), live_pos=pos.copy(), live_nrm=nrm.copy(),
             live_radius=rad.copy(), live_conf=conf.copy(), live_t_init=ti.copy(),
             live_t_obs=to.copy(),
             skin_idx=np.full((n, 8), -1, np.int32) if skin_idx is None else i32(skin_idx),
             skin_w=np.zeros((n, 8)) if skin_w is None else f64(skin_w),
             skin_count=np.zeros(n, np.int32) if skin_count is None else i32(skin_count))
    return m


def plane_surfels(nx, ny, step, z, confidence=20.0):
    """test_util.hpp:67-79"""
    out = []
    for j in range(ny):
        for i in range(nx):
            out.append(make_surfel(((i - (nx - 1) / 2.0) * step, (j - (ny - 1) / 2.0) * step, z),
                                   (0, 0, -1), 0.004, confidence))
    return out


def make_nodes(pos, dq=None, sigma=0.025, nbr=None):
    pos = f64(pos).reshape(-1, 3)
    n = len(pos)
    nodes = dict(pos=pos, sigma=np.full(n, sigma, np.float64),
                 dq=np.tile(IDENTITY_DQ, (n, 1)) if dq is None else f64(dq).reshape(n, 8),
                 nbr=np.full((n, 8), -1, np.int32), nbr_count=np.zeros(n, np.int32))
    if nbr is not None:
        for j, lst in enumerate(nbr):
            nodes["nbr"][j, :len(lst)] = lst
            nodes["nbr_count"][j] = len(lst)
    return nodes


def brute_force_knn(query, points, k):
    """test_util.hpp:49-65 — (d2, index) order."""
    points = np.asarray(points, dtype=np.float64).reshape(-1, 3)
    d = points - np.asarray(query)
    d2 = (d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2]
    order = np.lexsort((np.arange(len(points)), d2))
    return [int(i) for i in order[:k]]


class OracleState:
    """Model + warp field + frame maps (the reference's stage arguments)."""

    def __init__(self, cfg: dict):
        self.cfg = dict(cfg)
        self._c = to_struct(cfg)
        self.h = lib().or_state_new(C.byref(self._c))
        self._own = True

    @classmethod
    def borrow(cls, handle, cfg):
        o = cls.__new__(cls)
        o.cfg = dict(cfg)
        o._c = to_struct(cfg)
        o.h = handle
        o._own = False
        return o

    def __del__(self):
        if getattr(self, "_own", False) and getattr(self, "h", None):
            lib().or_state_free(self.h)
            self.h = None

    def set_mirror(self, on=True):
        lib().or_state_set_mirror(self.h, 1 if on else 0)

    def set_config(self, cfg):
        self.cfg = dict(cfg)
        self._c = to_struct(cfg)
        lib().or_state_set_config(self.h, C.byref(self._c))

    # -- model
    def set_model(self, m):
        n = len(m["ref_pos"])
        a = {k: (i32(v) if v.dtype.kind in "iu" else f64(v)) for k, v in m.items()}
        lib().or_set_model(self.h, n, ptr(a["ref_pos"]), ptr(a["ref_nrm"]), ptr(a["ref_radius"]),
                           ptr(a["ref_conf"]), ptr(a["ref_t_init"]), ptr(a["ref_t_obs"]),
                           ptr(a["live_pos"]), ptr(a["live_nrm"]), ptr(a["live_radius"]),
                           ptr(a["live_conf"]), ptr(a["live_t_init"]), ptr(a["live_t_obs"]),
                           ptr(a["skin_idx"]), ptr(a["skin_w"]), ptr(a["skin_count"]))

    def size(self):
        return lib().or_model_size(self.h)

    def get_model(self):
        n = self.size()
        m = dict(ref_pos=np.zeros((n, 3)), ref_nrm=np.zeros((n, 3)), ref_radius=np.zeros(n),
                 ref_conf=np.zeros(n), ref_t_init=np.zeros(n, np.int32),
                 ref_t_obs=np.zeros(n, np.int32), live_pos=np.zeros((n, 3)),
                 live_nrm=np.zeros((n, 3)), live_radius=np.zeros(n), live_conf=np.zeros(n),
                 live_t_init=np.zeros(n, np.int32), live_t_obs=np.zeros(n, np.int32),
                 skin_idx=np.zeros((n, 8), np.int32), skin_w=np.zeros((n, 8)),
                 skin_count=np.zeros(n, np.int32))
        lib().or_get_model(self.h, *[ptr(m[k]) for k in (
            "ref_pos", "ref_nrm", "ref_radius", "ref_conf", "ref_t_init", "ref_t_obs",
            "live_pos", "live_nrm", "live_radius", "live_conf", "live_t_init", "live_t_obs",
            "skin_idx", "skin_w", "skin_count")])
        return m

    # -- nodes
    def set_nodes(self, nd):
        n = len(nd["pos"])
        lib().or_set_nodes(self.h, n, ptr(f64(nd["pos"])), ptr(f64(nd["sigma"])),
                           ptr(f64(nd["dq"])), ptr(i32(nd["nbr"])), ptr(i32(nd["nbr_count"])))

    def num_nodes(self):
        return lib().or_num_nodes(self.h)

    def get_nodes(self):
        n = self.num_nodes()
        nd = dict(pos=np.zeros((n, 3)), sigma=np.zeros(n), dq=np.zeros((n, 8)),
                  nbr=np.zeros((n, 8), np.int32), nbr_count=np.zeros(n, np.int32))
        lib().or_get_nodes(self.h, ptr(nd["pos"]), ptr(nd["sigma"]), ptr(nd["dq"]),
                           ptr(nd["nbr"]), ptr(nd["nbr_count"]))
        return nd

    # -- frame
    def build_frame(self, depth, frame_index=0):
        d = np.ascontiguousarray(depth, dtype=np.uint16)
        h, w = d.shape
        return lib().or_build_frame(self.h, ptr(d), w, h, frame_index)

    def get_frame(self):
        w, h = self.cfg["width"], self.cfg["height"]
        f = dict(vert=np.zeros((h, w, 3)), nrm=np.zeros((h, w, 3)), conf=np.zeros((h, w)),
                 radius=np.zeros((h, w)), vertex_valid=np.zeros((h, w), np.uint8),
                 valid=np.zeros((h, w), np.uint8))
        vc = C.c_int32()
        lib().or_get_frame(self.h, ptr(f["vert"]), ptr(f["nrm"]), ptr(f["conf"]),
                           ptr(f["radius"]), ptr(f["vertex_valid"]), ptr(f["valid"]), C.byref(vc))
        f["valid_count"] = vc.value
        return f

    def set_frame(self, f, frame_index=0):
        h, w = f["valid"].shape
        lib().or_set_frame(self.h, w, h, frame_index, ptr(f64(f["vert"])), ptr(f64(f["nrm"])),
                           ptr(f64(f["conf"])), ptr(f64(f["radius"])),
                           ptr(u8(f["vertex_valid"])), ptr(u8(f["valid"])))

    # -- stages
    def init_warp_field(self):
        return lib().or_init_warp_field(self.h)

    def compute_node_edges(self, k):
        lib().or_compute_node_edges(self.h, k)

    def forward_warp(self):
        return lib().or_forward_warp(self.h)

    def inverse_warp_surfel(self, i):
        p, n = np.zeros(3), np.zeros(3)
        ok = lib().or_inverse_warp_surfel(self.h, i, ptr(p), ptr(n))
        return (p, n) if ok else None

    def extend_warp_field(self, positions):
        pos = f64(positions).reshape(-1, 3)
        return lib().or_extend_warp_field(self.h, len(pos), ptr(pos))

    def update_skinning_incremental(self, first_new):
        lib().or_update_skinning_incremental(self.h, first_new)

    def render_index_map(self, pose, factor):
        W, H = self.cfg["width"] * factor, self.cfg["height"] * factor
        idx = np.zeros((H, W), np.int32)
        dep = np.zeros((H, W))
        lib().or_render_index_map(self.h, ptr(f64(pose)), factor, ptr(idx), ptr(dep))
        return idx, dep

    def render_model_maps(self, pose, t_now, t_last):
        W, H = self.cfg["width"], self.cfg["height"]
        mm = dict(idx=np.zeros((H, W), np.int32), vert=np.zeros((H, W, 3)),
                  nrm=np.zeros((H, W, 3)), depth=np.zeros((H, W)), valid=np.zeros((H, W), np.uint8))
        lib().or_render_model_maps(self.h, ptr(f64(pose)), t_now, t_last, ptr(mm["idx"]),
                                   ptr(mm["vert"]), ptr(mm["nrm"]), ptr(mm["depth"]),
                                   ptr(mm["valid"]))
        return mm

    def find_correspondences(self, mm, pose):
        H, W = mm["valid"].shape
        cap = W * H
        out = dict(surfel=np.zeros(cap, np.int32), px=np.zeros(cap, np.int32),
                   py=np.zeros(cap, np.int32), v_model=np.zeros((cap, 3)),
                   v_depth=np.zeros((cap, 3)), n_depth=np.zeros((cap, 3)))
        n = lib().or_find_correspondences(
            self.h, ptr(i32(mm["idx"])), ptr(f64(mm["vert"])), ptr(f64(mm["nrm"])),
            ptr(u8(mm["valid"])), W, H, ptr(f64(pose)), cap, ptr(out["surfel"]), ptr(out["px"]),
            ptr(out["py"]), ptr(out["v_model"]), ptr(out["v_depth"]), ptr(out["n_depth"]))
        if n < 0:
            return -n
        return {k: v[:n] for k, v in out.items()}

    def normal_equations(self, pose, t_now, t_last):
        N = self.num_nodes()
        dim = 6 * N
        h = np.zeros((dim, dim))
        g = np.zeros(dim)
        touched = np.zeros((N, N), np.uint8)
        e = C.c_double()
        npairs = C.c_int32()
        st = lib().or_normal_equations(self.h, ptr(f64(pose)), t_now, t_last, ptr(h), ptr(g),
                                       ptr(touched), C.byref(e), C.byref(npairs))
        assert st == 0, lib().or_last_error()
        return dict(h=h, g=g, touched=touched, e_pre=e.value, n_pairs=npairs.value)

    def solve_nonrigid(self, pose, t_now, t_last):
        rep = OrSolverReport()
        st = lib().or_solve_nonrigid(self.h, ptr(f64(pose)), t_now, t_last, C.byref(rep))
        if st != 0:
            raise RuntimeError(f"oracle solve failed {st}: {lib().or_last_error()}")
        return rep

    def rigid_align(self, render_pose, init_pose, t_now, t_last):
        out = OrRigidResult()
        lib().or_rigid_align(self.h, ptr(f64(render_pose)), ptr(f64(init_pose)), t_now, t_last,
                             C.byref(out))
        return out

    def data_energy(self, surfel, v_depth, n_depth):
        return lib().or_data_energy(self.h, len(surfel), ptr(i32(surfel)), ptr(f64(v_depth)),
                                    ptr(f64(n_depth)))

    def reg_energy(self):
        return lib().or_reg_energy(self.h)

    def blend_jacobian(self, i):
        y = np.zeros(3)
        dydb = np.zeros((3, 8))
        nj = np.zeros((8, 3, 6))
        c = lib().or_blend_jacobian(self.h, i, ptr(y), ptr(dydb), ptr(nj))
        if c == 0:
            return None
        return y, dydb, nj[:c]

    def fuse_depth(self, index_map, factor, pose, t_now):
        cap = self.cfg["width"] * self.cfg["height"]
        out = dict(pos=np.zeros((cap, 3)), nrm=np.zeros((cap, 3)), radius=np.zeros(cap),
                   conf=np.zeros(cap), px=np.zeros(cap, np.int32), py=np.zeros(cap, np.int32))
        nc = C.c_int32()
        fused = lib().or_fuse_depth(self.h, ptr(i32(index_map)), factor, ptr(f64(pose)), t_now,
                                    cap, C.byref(nc), ptr(out["pos"]), ptr(out["nrm"]),
                                    ptr(out["radius"]), ptr(out["conf"]), ptr(out["px"]),
                                    ptr(out["py"]))
        return fused, {k: v[:nc.value] for k, v in out.items()}

    def skin_appended(self, x, node_live):
        idx = np.zeros(8, np.int32)
        w = np.zeros(8)
        c = C.c_int32()
        ok = lib().or_skin_appended(self.h, ptr(f64(x)), ptr(f64(node_live)), ptr(idx), ptr(w),
                                    C.byref(c))
        if not ok:
            return None
        return idx[:c.value], w[:c.value]

    def inverse_warp_strain(self, x, idx, w, node_live):
        s = np.zeros(9)
        ok = lib().or_inverse_warp_strain(self.h, ptr(f64(x)), ptr(i32(idx)), ptr(f64(w)),
                                          len(idx), ptr(f64(node_live)), ptr(s))
        return s.reshape(3, 3) if ok else None

    def check_compressive(self, x, idx, w, node_live):
        return bool(lib().or_check_compressive(self.h, ptr(f64(x)), ptr(i32(idx)), ptr(f64(w)),
                                               len(idx), ptr(f64(node_live))))

    def remove_surfels(self, index_map, factor, pose, t_now):
        mask = np.zeros(self.size(), np.uint8)
        lib().or_remove_surfels(self.h, ptr(i32(index_map)), factor, ptr(f64(pose)), t_now,
                                ptr(mask))
        return mask

    def apply_fusion(self, pose, t_now):
        out = OrFusionOutcome()
        st = lib().or_apply_fusion(self.h, ptr(f64(pose)), t_now, C.byref(out))
        assert st == 0, lib().or_last_error()
        return out

    def clean_and_reset(self, pose):
        r, s = C.c_int32(), C.c_int32()
        st = lib().or_clean_and_reset(self.h, ptr(f64(pose)), C.byref(r), C.byref(s))
        return st, r.value, s.value


class OraclePipeline:
    """Pipeline (pipeline.hpp:38-62) restated; mirror=True rounds surfel state to
    fp32 between stages like the device SoA storage."""

    def __init__(self, cfg: dict, mirror=False):
        self.cfg = dict(cfg)
        self._c = to_struct(cfg)
        self.h = lib().or_pipeline_new(C.byref(self._c), 1 if mirror else 0)

    def __del__(self):
        if getattr(self, "h", None):
            lib().or_pipeline_free(self.h)
            self.h = None

    def process_frame(self, depth, frame_index):
        d = np.ascontiguousarray(depth, dtype=np.uint16)
        h, w = d.shape
        st = OrFrameStats()
        code = lib().or_pipeline_process_frame(self.h, ptr(d), w, h, frame_index, C.byref(st))
        if code != 0:
            raise RuntimeError(f"oracle process_frame failed {code}: {lib().or_last_error()}")
        return st

    @property
    def state(self) -> OracleState:
        return OracleState.borrow(lib().or_pipeline_state(self.h), self.cfg)

    def pose(self):
        p = np.zeros(12)
        lib().or_pipeline_pose(self.h, ptr(p))
        return p


def voxel_knn(points, cell, q, k):
    pts = f64(points).reshape(-1, 3)
    out = np.zeros(max(k, 1), np.int32)
    n = lib().or_voxel_knn(ptr(pts), len(pts), cell, ptr(f64(q)), k, ptr(out))
    return [int(v) for v in out[:n]]


def compute_confidence(px, py, cfg):
    c = to_struct(cfg)
    return lib().or_compute_confidence(px, py, C.byref(c))


def compute_radius(d, f, nz):
    return lib().or_compute_radius(d, f, nz)


def backproject(depth, cfg):
    d = np.ascontiguousarray(depth, dtype=np.uint16)
    h, w = d.shape
    v = np.zeros((h, w, 3))
    vv = np.zeros((h, w), np.uint8)
    c = to_struct(cfg)
    st = lib().or_backproject(ptr(d), w, h, C.byref(c), ptr(v), ptr(vv))
    return st, v, vv


def estimate_normals(vert, vvalid):
    h, w = vvalid.shape
    n = np.zeros((h, w, 3))
    nv = np.zeros((h, w), np.uint8)
    lib().or_estimate_normals(ptr(f64(vert)), ptr(u8(vvalid)), w, h, ptr(n), ptr(nv))
    return n, nv


def bilateral_filter(depth, ss, sd):
    d = np.ascontiguousarray(depth, dtype=np.uint16)
    h, w = d.shape
    o = np.zeros_like(d)
    lib().or_bilateral_filter(ptr(d), w, h, ss, sd, ptr(o))
    return o


def ldlt_solve(a, b):
    a = f64(a)
    n = len(b)
    x = np.zeros(n)
    lib().or_ldlt_solve(n, ptr(a), ptr(f64(b)), ptr(x))
    return x


def sigma_max3(m):
    return lib().or_sigma_max3(ptr(f64(m).reshape(9)))


def should_reinitialize(mean_residuals, appended, t_now, t_last, cfg):
    mr = f64(mean_residuals)
    ap = i32(appended)
    c = to_struct(cfg)
    return bool(lib().or_should_reinitialize(len(mr), ptr(mr), ptr(ap), t_now, t_last,
                                             C.byref(c)))


def reg_terms(dq_j, dq_i, p_j):
    r = np.zeros(3)
    jj = np.zeros((3, 6))
    ji = np.zeros((3, 6))
    lib().or_reg_terms(ptr(f64(dq_j)), ptr(f64(dq_i)), ptr(f64(p_j)), ptr(r), ptr(jj), ptr(ji))
    return r, jj, ji


def assert_normal_equations(h):
    h = f64(h)
    return lib().or_assert_normal_equations(h.shape[0], ptr(h))
