"""Host mirror of the reference's per-frame API over the C ABI.

  Pipeline            dynsurf::Pipeline (pipeline.hpp:38-62): process_frame,
                      model(), nodes(), pose(), initialized(), last_reinit_frame()
  Context             stage entry points (warp_field.hpp, raster.hpp, solver.hpp,
                      fusion.hpp, depth_processing.hpp) on device-resident state,
                      used by the parity harness
  SyntheticSequence   synth.hpp:28-73 (host-side scene generator)

Arrays use the reference's host layouts in fp64 (see include/dynsurf_b200.h);
the device keeps fp32 SoA surfels and fp64 node transforms / frame maps.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import DsConfig, DsFrameStats, DsFusionOutcome, DsRigidResult, DsSolverReport, check

DEFAULTS = dict(
    node_sigma=0.025, knn_k=4, node_neighbor_k=8, lambda_=5.0, max_gn_iters=10,
    delta_distance=0.001, delta_normal=0.85, epsilon=0.2, delta_stable=10.0,
    t_low_confid=30, delta_recent=2, delta_nn=0.03, supersample_factor=4,
    compressive_check=1, depth_min=0.1, depth_max=5.0, bilateral_filter=0,
    bilateral_sigma_space=4.5, bilateral_sigma_depth=30.0, reinit_energy_threshold=0.005,
    reinit_append_threshold=3000, reinit_window=3, periodic_reinit_interval=0,
    delta_distance_reinit=0.010, fx=0.0, fy=0.0, cx=0.0, cy=0.0, width=0, height=0,
    pcg_max_iters=10, max_surfels=0, pcg_tol=0.0, max_nodes=0, profile=0,
)


def make_config(**kw) -> dict:
    """PipelineConfig{} defaults (config.hpp:11-50) + intrinsics + device knobs."""
    cfg = dict(DEFAULTS)
    if "lambda" in kw:
        kw["lambda_"] = kw.pop("lambda")
    for k, v in kw.items():
        if k not in cfg:
            raise KeyError(f"unknown config key: {k}")
        cfg[k] = v
    return cfg


def camera_config(width, height, focal, **kw) -> dict:
    """Synthetic-camera convention of synth.cpp:250-258: c = ((W-1)/2, (H-1)/2)."""
    return make_config(fx=focal, fy=focal, cx=(width - 1) / 2.0, cy=(height - 1) / 2.0,
                       width=width, height=height, **kw)


def to_struct(cfg: dict) -> DsConfig:
    s = DsConfig()
    for name, _ in DsConfig._fields_:
        if not name.startswith("_pad") and name in cfg:
            setattr(s, name, cfg[name])
    return s


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a if shape is None else a.reshape(shape)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _u8(a):
    return np.ascontiguousarray(a, dtype=np.uint8)


def stats_to_dict(st: DsFrameStats) -> dict:
    """FrameStats (pipeline.hpp:16-33) as the reference's metrics line fields."""
    return dict(
        frame=st.frame, skipped=bool(st.skipped), valid_pixels=st.valid_pixels,
        surfel_count=st.surfel_count, node_count=st.node_count,
        fused=st.fusion.fused, appended=st.fusion.appended, removed=st.fusion.removed,
        compressive_rejected=st.fusion.compressive_rejected,
        low_support_rejected=st.fusion.low_support_rejected, new_nodes=st.fusion.new_nodes,
        degenerate_warps=st.fusion.degenerate_warps, gn_iters=st.solver.iterations,
        correspondences=st.solver.correspondences, initial_energy=st.solver.initial_energy,
        final_energy=st.solver.final_energy, mean_residual=st.solver.mean_residual,
        rigid_pairs=st.rigid.correspondences, rigid_residual=st.rigid.mean_residual,
        rigid_low_confidence=bool(st.rigid.low_confidence), reinit=bool(st.reinit),
        reinit_removed=st.reinit_removed, pose=list(st.pose),
        depth_ms=st.depth_ms, rigid_ms=st.rigid_ms, solve_ms=st.solve_ms,
        fusion_ms=st.fusion_ms, reinit_ms=st.reinit_ms, total_ms=st.total_ms,
        lm_attempts=st.lm_attempts, pcg_iterations=st.pcg_iterations, gn_blocks=st.gn_blocks,
        kernel_launches=st.kernel_launches)


class Context:
    """One device-resident sequence state (ds_context); stage-level API."""

    def __init__(self, cfg: dict, device: int = 0, stream=None):
        self.cfg = dict(cfg)
        self._c = to_struct(cfg)
        self.L = _lib.load()
        h = C.c_void_p()
        check(self.L.ds_create(C.byref(self._c), device, stream, C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.L.ds_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def W(self):
        return self.cfg["width"]

    @property
    def H(self):
        return self.cfg["height"]

    # ---- state transfer
    def upload_model(self, m: dict):
        n = len(m["ref_pos"])
        radius = m.get("radius", m.get("live_radius"))
        conf = m.get("conf", m.get("live_conf"))
        t_init = m.get("t_init", m.get("live_t_init"))
        t_obs = m.get("t_obs", m.get("live_t_obs"))
        arrs = [_f64(m["ref_pos"]), _f64(m["ref_nrm"]), _f64(m["live_pos"]), _f64(m["live_nrm"]),
                _f64(radius), _f64(conf), _i32(t_init), _i32(t_obs), _i32(m["skin_idx"]),
                _f64(m["skin_w"]), _i32(m["skin_count"])]
        check(self.L.ds_upload_model(self.h, n, *[_p(a) for a in arrs]))

    def model_size(self) -> int:
        n = C.c_int32()
        check(self.L.ds_model_size(self.h, C.byref(n)))
        return n.value

    def download_model(self) -> dict:
        n = self.model_size()
        m = dict(ref_pos=np.zeros((n, 3)), ref_nrm=np.zeros((n, 3)), live_pos=np.zeros((n, 3)),
                 live_nrm=np.zeros((n, 3)), radius=np.zeros(n), conf=np.zeros(n),
                 t_init=np.zeros(n, np.int32), t_obs=np.zeros(n, np.int32),
                 skin_idx=np.zeros((n, 8), np.int32), skin_w=np.zeros((n, 8)),
                 skin_count=np.zeros(n, np.int32))
        check(self.L.ds_download_model(self.h, *[_p(m[k]) for k in (
            "ref_pos", "ref_nrm", "live_pos", "live_nrm", "radius", "conf", "t_init", "t_obs",
            "skin_idx", "skin_w", "skin_count")]))
        return m

    def upload_nodes(self, nd: dict):
        n = len(nd["pos"])
        check(self.L.ds_upload_nodes(self.h, n, _p(_f64(nd["pos"])), _p(_f64(nd["sigma"])),
                                     _p(_f64(nd["dq"])), _p(_i32(nd["nbr"])),
                                     _p(_i32(nd["nbr_count"]))))

    def num_nodes(self) -> int:
        n = C.c_int32()
        check(self.L.ds_num_nodes(self.h, C.byref(n)))
        return n.value

    def download_nodes(self) -> dict:
        n = self.num_nodes()
        nd = dict(pos=np.zeros((n, 3)), sigma=np.zeros(n), dq=np.zeros((n, 8)),
                  nbr=np.zeros((n, 8), np.int32), nbr_count=np.zeros(n, np.int32))
        check(self.L.ds_download_nodes(self.h, _p(nd["pos"]), _p(nd["sigma"]), _p(nd["dq"]),
                                       _p(nd["nbr"]), _p(nd["nbr_count"])))
        return nd

    def set_pose(self, pose):
        check(self.L.ds_set_pose(self.h, _p(_f64(pose))))

    def get_pose(self):
        p = np.zeros(12)
        check(self.L.ds_get_pose(self.h, _p(p)))
        return p

    # ---- stages
    def frame_maps(self, depth, frame_index=0) -> int:
        d = np.ascontiguousarray(depth, dtype=np.uint16)
        h, w = d.shape
        vc = C.c_int32()
        check(self.L.ds_frame_maps(self.h, _p(d), w, h, frame_index, C.byref(vc)))
        return vc.value

    def download_frame(self) -> dict:
        W, H = self.W, self.H
        f = dict(vert=np.zeros((H, W, 3)), nrm=np.zeros((H, W, 3)), conf=np.zeros((H, W)),
                 radius=np.zeros((H, W)), vertex_valid=np.zeros((H, W), np.uint8),
                 valid=np.zeros((H, W), np.uint8))
        check(self.L.ds_download_frame(self.h, _p(f["vert"]), _p(f["nrm"]), _p(f["conf"]),
                                       _p(f["radius"]), _p(f["vertex_valid"]), _p(f["valid"])))
        f["valid_count"] = int(f["valid"].sum())
        return f

    def upload_frame(self, f: dict, frame_index=0):
        H, W = f["valid"].shape
        check(self.L.ds_upload_frame(self.h, W, H, frame_index, _p(_f64(f["vert"])),
                                     _p(_f64(f["nrm"])), _p(_f64(f["conf"])),
                                     _p(_f64(f["radius"])), _p(_u8(f["vertex_valid"])),
                                     _p(_u8(f["valid"]))))

    def init_warp_field(self):
        check(self.L.ds_init_warp_field(self.h))

    def compute_node_edges(self):
        check(self.L.ds_compute_node_edges(self.h))

    def forward_warp(self) -> int:
        d = C.c_int32()
        check(self.L.ds_forward_warp(self.h, C.byref(d)))
        return d.value

    def render_index_map(self, pose, factor):
        idx = np.zeros((self.H * factor, self.W * factor), np.int32)
        check(self.L.ds_render_index_map(self.h, _p(_f64(pose)), factor, _p(idx)))
        return idx

    def render_model_maps(self, pose, t_now, t_last) -> dict:
        W, H = self.W, self.H
        mm = dict(idx=np.zeros((H, W), np.int32), vert=np.zeros((H, W, 3)),
                  nrm=np.zeros((H, W, 3)), depth=np.zeros((H, W)),
                  valid=np.zeros((H, W), np.uint8))
        check(self.L.ds_render_model_maps(self.h, _p(_f64(pose)), t_now, t_last, _p(mm["idx"]),
                                          _p(mm["vert"]), _p(mm["nrm"]), _p(mm["depth"]),
                                          _p(mm["valid"])))
        return mm

    def associate(self, pose) -> dict:
        cap = self.W * self.H
        out = dict(surfel=np.zeros(cap, np.int32), px=np.zeros(cap, np.int32),
                   py=np.zeros(cap, np.int32), v_model=np.zeros((cap, 3)),
                   v_depth=np.zeros((cap, 3)), n_depth=np.zeros((cap, 3)))
        n = C.c_int32()
        check(self.L.ds_associate(self.h, _p(_f64(pose)), cap, C.byref(n), _p(out["surfel"]),
                                  _p(out["px"]), _p(out["py"]), _p(out["v_model"]),
                                  _p(out["v_depth"]), _p(out["n_depth"])))
        return {k: v[:n.value] for k, v in out.items()}

    def build_normal_equations(self, pose, t_now, t_last) -> dict:
        nb, npairs, e = C.c_int32(), C.c_int32(), C.c_double()
        check(self.L.ds_build_normal_equations(self.h, _p(_f64(pose)), t_now, t_last,
                                               C.byref(nb), C.byref(npairs), C.byref(e)))
        N = self.num_nodes()
        B = nb.value
        out = dict(row_ptr=np.zeros(N + 1, np.int32), col=np.zeros(B, np.int32),
                   values=np.zeros((B, 6, 6)), touched=np.zeros(B, np.uint8), g=np.zeros(6 * N),
                   e_pre=e.value, n_pairs=npairs.value)
        check(self.L.ds_download_normal_equations(self.h, _p(out["row_ptr"]), _p(out["col"]),
                                                  _p(out["values"]), _p(out["touched"]),
                                                  _p(out["g"])))
        return out

    def check_normal_equations(self):
        """assert_normal_equations (solver.cpp:157-167); raises errors.Error."""
        check(self.L.ds_check_normal_equations(self.h))

    def set_normal_equation_values(self, values, g=None):
        v = np.ascontiguousarray(values, dtype=np.float64)
        check(self.L.ds_set_normal_equation_values(self.h, _p(v), _p(_f64(g)) if g is not None
                                                   else None))

    def pcg_solve(self, mu, max_iters, tol=0.0):
        N = self.num_nodes()
        delta = np.zeros(6 * N)
        it, rel = C.c_int32(), C.c_double()
        check(self.L.ds_pcg_solve(self.h, mu, max_iters, tol, _p(delta), C.byref(it),
                                  C.byref(rel)))
        return delta, it.value, rel.value

    def bsr_spmv(self, x, mu=0.0, reps=1):
        """y = (H + mu I) x with the standalone SpMV kernel; returns (y, mean ms)."""
        x = _f64(x)
        y = np.zeros_like(x)
        ms = C.c_double()
        check(self.L.ds_bsr_spmv(self.h, _p(x), _p(y), mu, reps, C.byref(ms)))
        return y, ms.value

    def solve_nonrigid(self, pose, t_now, t_last) -> DsSolverReport:
        rep = DsSolverReport()
        check(self.L.ds_solve_nonrigid(self.h, _p(_f64(pose)), t_now, t_last, C.byref(rep)))
        return rep

    def rigid_align(self, render_pose, init_pose, t_now, t_last) -> DsRigidResult:
        out = DsRigidResult()
        check(self.L.ds_rigid_align(self.h, _p(_f64(render_pose)), _p(_f64(init_pose)), t_now,
                                    t_last, C.byref(out)))
        return out

    def apply_fusion(self, pose, t_now) -> DsFusionOutcome:
        out = DsFusionOutcome()
        check(self.L.ds_apply_fusion(self.h, _p(_f64(pose)), t_now, C.byref(out)))
        return out

    def fuse_depth(self, pose, t_now):
        fused, nc = C.c_int32(), C.c_int32()
        check(self.L.ds_fuse_depth(self.h, _p(_f64(pose)), t_now, C.byref(fused), C.byref(nc)))
        n = nc.value
        cand = dict(pos=np.zeros((n, 3)), nrm=np.zeros((n, 3)), radius=np.zeros(n),
                    conf=np.zeros(n), px=np.zeros(n, np.int32), py=np.zeros(n, np.int32))
        check(self.L.ds_download_candidates(self.h, _p(cand["pos"]), _p(cand["nrm"]),
                                            _p(cand["radius"]), _p(cand["conf"]), _p(cand["px"]),
                                            _p(cand["py"])))
        return fused.value, cand

    def skin_appended(self, positions):
        pos = _f64(positions).reshape(-1, 3)
        n = len(pos)
        out = dict(idx=np.zeros((n, 8), np.int32), w=np.zeros((n, 8)),
                   count=np.zeros(n, np.int32), supported=np.zeros(n, np.uint8),
                   compressive_ok=np.zeros(n, np.uint8))
        check(self.L.ds_skin_appended(self.h, n, _p(pos), None, _p(out["idx"]), _p(out["w"]),
                                      _p(out["count"]), _p(out["supported"]),
                                      _p(out["compressive_ok"])))
        return out

    def remove_mask(self, pose, t_now):
        mask = np.zeros(self.model_size(), np.uint8)
        check(self.L.ds_remove_mask(self.h, _p(_f64(pose)), t_now, _p(mask)))
        return mask

    def extend_warp_field(self, positions) -> int:
        pos = _f64(positions).reshape(-1, 3)
        a = C.c_int32()
        check(self.L.ds_extend_warp_field(self.h, len(pos), _p(pos), C.byref(a)))
        return a.value

    def update_skinning_incremental(self, first_new):
        check(self.L.ds_update_skinning_incremental(self.h, first_new))

    def clean_and_reset(self, pose):
        r, s = C.c_int32(), C.c_int32()
        check(self.L.ds_clean_and_reset(self.h, _p(_f64(pose)), C.byref(r), C.byref(s)))
        return r.value, s.value

    # ---- frame loop
    def process_frame(self, depth, frame_index) -> DsFrameStats:
        d = np.ascontiguousarray(depth, dtype=np.uint16)
        h, w = d.shape
        st = DsFrameStats()
        check(self.L.ds_process_frame(self.h, _p(d), w, h, frame_index, C.byref(st)))
        return st

    def process_frame_device(self, depth_ptr: int, frame_index) -> DsFrameStats:
        st = DsFrameStats()
        check(self.L.ds_process_frame_device(self.h, C.c_void_p(depth_ptr), self.W, self.H,
                                             frame_index, C.byref(st)))
        return st

    def synchronize(self):
        check(self.L.ds_synchronize(self.h))

    def capacity(self) -> dict:
        """Device capacities; grown geometrically at frame boundaries."""
        a, b, g = C.c_int32(), C.c_int32(), C.c_int32()
        check(self.L.ds_capacity(self.h, C.byref(a), C.byref(b), C.byref(g)))
        return dict(surfels=a.value, nodes=b.value, growths=g.value)

    def join_deferred(self):
        """Context stream waits for the frame's deferred side-stream work (no host sync)."""
        check(self.L.ds_join_deferred(self.h))

    # ---- measurement
    def kernel_stats(self) -> dict:
        out = {}
        for k in range(self.L.ds_num_kernel_kinds()):
            n, ms, b = C.c_int64(), C.c_double(), C.c_double()
            check(self.L.ds_kernel_stats(self.h, k, C.byref(n), C.byref(ms), C.byref(b)))
            out[self.L.ds_kernel_name(k).decode()] = dict(launches=n.value, ms=ms.value,
                                                          bytes=b.value)
        return out

    def reset_kernel_stats(self):
        check(self.L.ds_reset_kernel_stats(self.h))

    def set_profiling(self, on: bool):
        check(self.L.ds_set_profiling(self.h, 1 if on else 0))

    def total_launches(self) -> int:
        n = C.c_int64()
        check(self.L.ds_total_launches(self.h, C.byref(n)))
        return n.value


class Pipeline:
    """dynsurf::Pipeline (pipeline.hpp:38-62) on the B200 path."""

    def __init__(self, cfg: dict, device: int = 0, stream=None):
        check(_lib.load().ds_validate_config(C.byref(to_struct(cfg))))
        self._ctx = Context(cfg, device, stream)

    @property
    def context(self) -> Context:
        return self._ctx

    def config(self) -> dict:
        return dict(self._ctx.cfg)

    def process_frame(self, depth, frame_index: int) -> dict:
        return stats_to_dict(self._ctx.process_frame(depth, frame_index))

    def model(self) -> dict:
        return self._ctx.download_model()

    def nodes(self) -> dict:
        return self._ctx.download_nodes()

    def pose(self):
        return self._ctx.get_pose()

    def initialized(self) -> bool:
        i, t = C.c_int32(), C.c_int32()
        check(self._ctx.L.ds_is_initialized(self._ctx.h, C.byref(i), C.byref(t)))
        return bool(i.value)

    def last_reinit_frame(self) -> int:
        i, t = C.c_int32(), C.c_int32()
        check(self._ctx.L.ds_is_initialized(self._ctx.h, C.byref(i), C.byref(t)))
        return t.value

    def close(self):
        self._ctx.close()


class SyntheticSequence:
    """SyntheticSequence (synth.hpp:28-73): analytic scenes ray-cast to mm depth."""

    def __init__(self, scenario: str, frames: int, cfg: dict, noise_sigma_mm=0.0,
                 seed=20240901):
        self.L = _lib.load_synth()
        self.kind = self.L.ds_synth_scenario(scenario.encode())
        if self.kind < 0:
            from .errors import UnknownScenario
            raise UnknownScenario(f"unknown scenario: {scenario}")
        self.frames = frames if frames > 0 else self.L.ds_synth_default_frames(self.kind)
        self.cfg = dict(cfg)
        self._c = to_struct(cfg)
        self.noise = float(noise_sigma_mm)
        self.seed = int(seed)

    def frame_count(self):
        return self.frames

    def render_depth(self, t: int) -> np.ndarray:
        d = np.zeros((self.cfg["height"], self.cfg["width"]), np.uint16)
        _lib.check_synth(self.L.ds_synth_render_depth(self.kind, self.frames, C.byref(self._c),
                                                      self.noise, self.seed, t, _p(d)))
        return d

    def camera_pose(self, t: int):
        p = np.zeros(12)
        _lib.check_synth(self.L.ds_synth_camera_pose(self.kind, self.frames, t, _p(p)))
        return p

    def surface_distance(self, p, t: int) -> float:
        return self.L.ds_synth_surface_distance(self.kind, self.frames, _p(_f64(p)), t)
