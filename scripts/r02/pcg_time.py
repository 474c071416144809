"""PCG launch time at config 2: cluster kernel vs cooperative grid kernel, on
the system of frame `skip` (after running the sequence up to it)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def run(mode, skip, reps=50):
    os.environ["DS_PCG_CLUSTER"] = mode
    import paper_1904_13073_b200 as pkg
    spec = bench.CONFIGS["cfg2"]
    cfg = bench.make_cfg(spec)
    frames = bench.render_frames(spec, cfg, skip + 1, 0)
    pipe = pkg.Pipeline(cfg)
    for t in range(skip):
        pipe.process_frame(frames[t], t)
    ctx = pipe.context
    ctx.frame_maps(frames[skip], skip)
    ne = ctx.build_normal_equations(pipe.pose(), skip, 0)
    N = ctx.num_nodes()
    out = []
    for iters in (0, 1, 10, 20):
        ctx.pcg_solve(1e-3, iters, 0.0)
        ctx.reset_kernel_stats()
        ctx.set_profiling(True)
        for _ in range(reps):
            ctx.pcg_solve(1e-3, iters, 0.0)
        k = ctx.kernel_stats()["pcg"]
        ctx.set_profiling(False)
        out.append((iters, round(1e3 * k["ms"] / max(k["launches"], 1), 2)))
    x, it, rel = ctx.pcg_solve(1e-3, 10, 0.0)
    print(f"mode {mode} frame {skip} nodes {N} blocks {len(ne['col'])} us by iters {out} "
          f"rel_res10 {rel:.3e} |x| {np.abs(x).max():.6e}", flush=True)
    pipe.close()


if __name__ == "__main__":
    run(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 20)
