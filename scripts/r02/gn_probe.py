"""GN / PCG convergence probe: per-frame GN
iterations, LM attempts, PCG iterations and solve time of the device pipeline
under several PCG budgets, on a BASELINE config's sequence."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1904_13073_b200 as pkg  # noqa: E402

VARIANTS = {
    "pcg10": dict(pcg_max_iters=10, pcg_tol=0.0),
    "pcg20": dict(pcg_max_iters=20, pcg_tol=0.0),
    "pcg40": dict(pcg_max_iters=40, pcg_tol=0.0),
    "tol1e-4": dict(pcg_max_iters=200, pcg_tol=1e-4),
    "tol1e-6": dict(pcg_max_iters=500, pcg_tol=1e-6),
    "tol1e-10": dict(pcg_max_iters=2000, pcg_tol=1e-10),
}


def main(config="cfg2", frames=26, names=None):
    spec = bench.CONFIGS[config]
    gn = 3 if config == "cfg1" else 10
    frames = min(frames, spec["seq_frames"])
    base = pkg.camera_config(spec["width"], spec["height"], spec["focal"], max_gn_iters=gn)
    seq = pkg.SyntheticSequence(spec["scene"], spec["seq_frames"], base)
    depth = [seq.render_depth(t) for t in range(frames)]
    for name, kw in VARIANTS.items():
        if names and name not in names:
            continue
        cfg = pkg.camera_config(spec["width"], spec["height"], spec["focal"], max_gn_iters=gn, **kw)
        p = pkg.Pipeline(cfg)
        rows = []
        for t in range(frames):
            s = p.process_frame(depth[t], t)
            if t >= 1:
                rows.append(s)
            if t in (1, 5, 10, 25):
                print(f"  {config} {name} f{t}: gn {s['gn_iters']} lm {s['lm_attempts']} pcg "
                      f"{s['pcg_iterations']} solve {s['solve_ms']:.3f} ms e0 {s['initial_energy']:.4e} "
                      f"e1 {s['final_energy']:.4e} mr {s['mean_residual']:.3e} S {s['surfel_count']} "
                      f"N {s['node_count']} corr {s['correspondences']} app {s['appended']}", flush=True)
        p.close()
        f = lambda k: float(np.mean([r[k] for r in rows]))  # noqa: E731
        print(f"{config} {name}: gn {f('gn_iters'):.2f} lm {f('lm_attempts'):.2f} pcg "
              f"{f('pcg_iterations'):.1f} solve {f('solve_ms'):.3f} ms total {f('total_ms'):.3f} ms "
              f"e1/e0 {np.mean([r['final_energy'] / max(r['initial_energy'], 1e-30) for r in rows]):.4f} "
              f"mr {f('mean_residual'):.3e} S_end {rows[-1]['surfel_count']}", flush=True)


if __name__ == "__main__":
    cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 26
    main(cfg, n, sys.argv[3].split(",") if len(sys.argv) > 3 else None)
