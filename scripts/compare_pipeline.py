"""Per-frame stats of the B200 pipeline vs the oracle pipeline (fp32 mirror)."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import paper_1904_13073_b200 as pkg
import oracle_py as O
import harness as Hh

scene = sys.argv[1] if len(sys.argv) > 1 else "articulated_two_part"
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 6
tol = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-12
W, H, F = (160, 120, 140.0) if len(sys.argv) <= 4 else (int(sys.argv[4]), int(sys.argv[5]), float(sys.argv[6]))
cfg = pkg.make_config(fx=F, fy=F, cx=(W - 1) / 2, cy=(H - 1) / 2, width=W, height=H,
                      pcg_tol=tol, pcg_max_iters=2000 if tol > 0 else 10)
seq = pkg.SyntheticSequence(scene, 30, cfg)
pipe = pkg.Pipeline(cfg)
ore = O.OraclePipeline(Hh.oracle_cfg(cfg), mirror=True)
keys = ["valid_pixels", "surfel_count", "node_count", "correspondences", "gn_iters", "fused",
        "appended", "removed", "low_support_rejected", "compressive_rejected", "new_nodes"]
for t in range(frames):
    d = seq.render_depth(t)
    g = pipe.process_frame(d, t)
    o = ore.process_frame(d, t)
    ov = dict(valid_pixels=o.valid_pixels, surfel_count=o.surfel_count, node_count=o.node_count,
              correspondences=o.solver.correspondences, gn_iters=o.solver.iterations,
              fused=o.fusion.fused, appended=o.fusion.appended, removed=o.fusion.removed,
              low_support_rejected=o.fusion.low_support_rejected,
              compressive_rejected=o.fusion.compressive_rejected, new_nodes=o.fusion.new_nodes)
    print(f"t={t}", " ".join(f"{k}={g[k]}/{ov[k]}" for k in keys))
    print("   E0 %.3e/%.3e E1 %.3e/%.3e mr %.3e/%.3e pose %.2e ms %.2f" % (
        g["initial_energy"], o.solver.initial_energy, g["final_energy"], o.solver.final_energy,
        g["mean_residual"], o.solver.mean_residual,
        np.abs(np.array(g["pose"]) - np.array(o.pose)).max(), g["total_ms"]))
