"""PCG launch time vs iteration count on a cfg4 system (per-iteration cost)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench_solver as bs


def main():
    import paper_1904_13073_b200 as pkg
    for nodes in (1024, 4096):
        W, H = bs.dims_for(nodes)
        cfg = pkg.camera_config(W, H, 560.0, max_nodes=8192, max_surfels=2 * W * H, pcg_max_iters=10)
        seq = pkg.SyntheticSequence("sine_sheet", 10, cfg)
        ctx = pkg.Context(cfg)
        ctx.process_frame(seq.render_depth(0), 0)
        ctx.frame_maps(seq.render_depth(1), 1)
        I = np.eye(3).reshape(9).tolist() + [0.0, 0.0, 0.0]
        ctx.build_normal_equations(I, 1, 0)
        out = []
        for iters in (0, 1, 2, 5, 10, 20):
            ctx.reset_kernel_stats()
            ctx.set_profiling(True)
            for _ in range(20):
                ctx.pcg_solve(1e-3, iters, 0.0)
            k = ctx.kernel_stats()["pcg"]
            ctx.set_profiling(False)
            out.append((iters, round(1e3 * k["ms"] / max(k["launches"], 1), 2)))
        print("nodes", ctx.num_nodes(), "pcg us by iters", out, flush=True)
        ctx.close()


if __name__ == "__main__":
    main()
