"""Free-running sequence drift: rigid_orbit, 160x120, 50
frames. Device pipeline vs the oracle pipeline in fp32 mirror mode, and the
oracle's own faithful (fp64) vs mirror runs: per-frame pose gap, and the first
frame each pair parts by more than 1e-4."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import harness as Hh  # noqa: E402
import oracle_py as O  # noqa: E402
import paper_1904_13073_b200 as pkg  # noqa: E402

SMALL = dict(fx=140.0, fy=140.0, cx=79.5, cy=59.5, width=160, height=120)
frames = int(sys.argv[1]) if len(sys.argv) > 1 else 50
cfg = pkg.make_config(**SMALL, pcg_tol=1e-12, pcg_max_iters=2000)
seq = pkg.SyntheticSequence("rigid_orbit", frames, cfg)
pipe = pkg.Pipeline(cfg)
mir = O.OraclePipeline(Hh.oracle_cfg(cfg), mirror=True)
fai = O.OraclePipeline(Hh.oracle_cfg(cfg), mirror=False)
first = {}
for t in range(frames):
    d = seq.render_depth(t)
    g = pipe.process_frame(d, t)
    m = mir.process_frame(d, t)
    f = fai.process_frame(d, t)
    gp, mp, fp = np.array(g["pose"]), np.array(m.pose), np.array(f.pose)
    gt = np.asarray(seq.camera_pose(t))
    gaps = {"device-mirror": np.abs(gp - mp).max(), "faithful-mirror": np.abs(fp - mp).max()}
    for k, v in gaps.items():
        if v > 1e-4 and k not in first:
            first[k] = t
    print(t, " ".join(f"{k} {v:.2e}" for k, v in gaps.items()),
          f"| truth err dev {np.linalg.norm(gp[9:] - gt[9:]) * 1e3:.2f} mm "
          f"mirror {np.linalg.norm(mp[9:] - gt[9:]) * 1e3:.2f} mm "
          f"faithful {np.linalg.norm(fp[9:] - gt[9:]) * 1e3:.2f} mm | surfels {g['surfel_count']} "
          f"{m.surfel_count} {f.surfel_count}", flush=True)
print("first frame with pose gap > 1e-4:", first)
