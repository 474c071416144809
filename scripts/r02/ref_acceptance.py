"""SPEC acceptance criteria 3-6 measured on the COMPILED REFERENCE (oracle/_ref,
the unmodified reference sources): the same scenes, sizes and measures as
tests/test_gpu_acceptance.py, to show where the thresholds are a property of
the algorithm as specified rather than of the B200 port. CPU only."""
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle_py as O  # noqa: E402
import ref_py as R  # noqa: E402
import paper_1904_13073_b200 as pkg  # noqa: E402

SMALL = dict(fx=140.0, fy=140.0, cx=79.5, cy=59.5, width=160, height=120)


def run(scene, frames=None, **kw):
    cfg = pkg.make_config(**{**SMALL, **kw})
    n = frames if frames is not None else pkg.SyntheticSequence(scene, 0, cfg).frames
    seq = pkg.SyntheticSequence(scene, n, cfg)
    rp = R.RefPipeline(O.make_config(**{k: v for k, v in cfg.items() if k in O.DEFAULTS}))
    return cfg, seq, rp, n


def surface_distance(rp, seq, t, delta_stable):
    m = rp.model()
    sel = m["confidence"] > delta_stable
    pts = m["live_pos"][sel] if sel.any() else m["live_pos"]
    d = np.array([seq.surface_distance(p, t) for p in pts])
    return float(d.mean()), float(d.max())


which = sys.argv[1:] or ["3", "4", "5", "6"]
if "3" in which:
    _, seq, rp, n = run("rigid_orbit", 50)
    wt, wr, first = 0.0, 0.0, None
    for t in range(n):
        st = rp.process_frame(seq.render_depth(t), t)
        gt = np.asarray(seq.camera_pose(t))
        Re, Rg = st["pose_R"], gt[:9].reshape(3, 3)
        ang = math.degrees(math.acos(max(-1.0, min(1.0, (np.trace(Re.T @ Rg) - 1.0) / 2.0))))
        et = float(np.linalg.norm(st["pose_t"] - gt[9:]))
        wt, wr = max(wt, et), max(wr, ang)
        if first is None and (et >= 1e-3 or ang >= 0.2):
            first = (t, et, ang)
    print(f"criterion 3 (rigid_orbit, {n} frames): worst translation {wt * 1e3:.3f} mm, "
          f"rotation {wr:.4f} deg; first frame past the bar {first}", flush=True)
if "4" in which:
    cfg, seq, rp, n = run("bending_sheet", 100)
    iters, wm, wx = [], 0.0, 0.0
    for t in range(n):
        st = rp.process_frame(seq.render_depth(t), t)
        if t > 0:
            iters.append(st["solver_iterations"])
        mean, mx = surface_distance(rp, seq, t, cfg["delta_stable"])
        wm, wx = max(wm, mean), max(wx, mx)
    print(f"criterion 4 (bending_sheet, {n} frames): worst mean {wm * 1e3:.3f} mm, worst max "
          f"{wx * 1e3:.3f} mm, GN median {np.median(iters)}, max {max(iters)}", flush=True)
if "5" in which:
    _, seq, rp, n = run("turntable")
    counts, ratio = [], 0.0
    for t in range(n):
        st = rp.process_frame(seq.render_depth(t), t)
        if t >= n // 2:
            counts.append(st["surfel_count"])
            ratio = max(ratio, st["appended"] / max(st["valid_pixels"], 1))
    print(f"criterion 5 (turntable, {n} frames): count ratio {max(counts) / min(counts):.4f}, "
          f"max appended fraction {ratio:.4f}", flush=True)
if "6" in which:
    tot = {}
    for on in (1, 0):
        _, seq, rp, n = run("open_to_close", compressive_check=on)
        tot[on] = sum(rp.process_frame(seq.render_depth(t), t)["compressive_rejected"]
                      for t in range(n))
    print(f"criterion 6 (open_to_close, {n} frames): compressive rejections on={tot[1]} "
          f"off={tot[0]}", flush=True)
