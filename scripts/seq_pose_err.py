"""Per-frame pose / residual gap between the device pipeline and the oracle
pipeline (fp32 mirror mode) on a small synthetic sequence."""
import os
import sys

import numpy as np

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, root)
sys.path.insert(0, os.path.join(root, "tests"))
import harness as Hh  # noqa: E402
import oracle_py as O  # noqa: E402
import paper_1904_13073_b200 as pkg  # noqa: E402
from test_gpu_solve_fusion import SMALL, CONVERGED  # noqa: E402


def main(scene="rigid_orbit", frames=8):
    cfg = pkg.make_config(**{**SMALL, **CONVERGED})
    seq = pkg.SyntheticSequence(scene, 30, cfg)
    pipe = pkg.Pipeline(cfg)
    ore = O.OraclePipeline(Hh.oracle_cfg(cfg), mirror=True)
    for t in range(frames):
        d = seq.render_depth(t)
        g = pipe.process_frame(d, t)
        o = ore.process_frame(d, t)
        print(t, "pose %.3e" % np.abs(np.array(g["pose"]) - np.array(o.pose)).max(),
              "res %.3e" % abs(g["mean_residual"] - o.solver.mean_residual),
              "it", g["gn_iters"], o.solver.iterations, "corr", g["correspondences"], o.solver.correspondences)


if __name__ == "__main__":
    main(*sys.argv[1:2], *(int(a) for a in sys.argv[2:3]))
