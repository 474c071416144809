"""Parity harness helpers: run the CUDA path and the CPU oracle on the same
(fp32-rounded) inputs. TEST INFRASTRUCTURE."""
from __future__ import annotations

import numpy as np

import oracle_py as O


def oracle_cfg(cfg: dict) -> dict:
    return O.make_config(**{k: v for k, v in cfg.items() if k in O.DEFAULTS})


def device_to_oracle_model(m: dict) -> dict:
    """Product host model (shared attributes) -> oracle model (ref/live attributes)."""
    n = len(m["ref_pos"])
    return dict(ref_pos=m["ref_pos"].copy(), ref_nrm=m["ref_nrm"].copy(),
                ref_radius=m["radius"].copy(), ref_conf=m["conf"].copy(),
                ref_t_init=m["t_init"].copy(), ref_t_obs=m["t_obs"].copy(),
                live_pos=m["live_pos"].copy(), live_nrm=m["live_nrm"].copy(),
                live_radius=m["radius"].copy(), live_conf=m["conf"].copy(),
                live_t_init=m["t_init"].copy(), live_t_obs=m["t_obs"].copy(),
                skin_idx=m["skin_idx"].copy().reshape(n, 8), skin_w=m["skin_w"].copy().reshape(n, 8),
                skin_count=m["skin_count"].copy())


def oracle_to_device_model(m: dict) -> dict:
    return dict(ref_pos=m["ref_pos"], ref_nrm=m["ref_nrm"], live_pos=m["live_pos"],
                live_nrm=m["live_nrm"], radius=m["live_radius"], conf=m["live_conf"],
                t_init=m["live_t_init"], t_obs=m["live_t_obs"], skin_idx=m["skin_idx"],
                skin_w=m["skin_w"], skin_count=m["skin_count"])


def surfels_from_frame(frame: dict, confidence=None, t_init=0, x_range=None):
    """Model surfels straight from frame pixels (test_solver.cpp:190-201)."""
    H, W = frame["valid"].shape
    out = []
    for y in range(H):
        for x in range(W):
            if not frame["valid"][y, x]:
                continue
            if x_range is not None and not (x_range[0] <= x < x_range[1]):
                continue
            out.append(O.make_surfel(frame["vert"][y, x], frame["nrm"][y, x],
                                     frame["radius"][y, x],
                                     frame["conf"][y, x] if confidence is None else confidence,
                                     t_init))
    return out


def round_trip(ctx, model: dict, nodes: dict | None = None):
    """Upload to the device and read back: the fp32-rounded shared input."""
    ctx.upload_model(oracle_to_device_model(model) if "live_radius" in model else model)
    if nodes is not None:
        ctx.upload_nodes(nodes)
    dm = ctx.download_model()
    dn = ctx.download_nodes() if nodes is not None else None
    return device_to_oracle_model(dm), dn


def bsr_to_dense(ne: dict, N: int):
    H = np.zeros((6 * N, 6 * N))
    T = np.zeros((N, N), np.uint8)
    rp, col = ne["row_ptr"], ne["col"]
    for r in range(N):
        for k in range(rp[r], rp[r + 1]):
            c = col[k]
            H[6 * r:6 * r + 6, 6 * c:6 * c + 6] = ne["values"][k]
            T[r, c] = ne["touched"][k]
    return H, T
