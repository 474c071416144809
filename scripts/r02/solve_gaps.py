"""Measured gaps of tests/test_gpu_solve_fusion.py::test_solve_nonrigid_matches_oracle
(converged PCG vs the oracle's LDLT), to set the tolerances written in the test."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle_py as O  # noqa: E402
from test_gpu_solve_fusion import dq_close, setup  # noqa: E402

for scene, t in (("rigid_orbit", 2), ("articulated_two_part", 10), ("bending_sheet", 40)):
    cfg, seq, ctx, st = setup(scene, frames=60, t_frame=t)
    pose = O.pose_identity()
    g = ctx.solve_nonrigid(pose, t, 0)
    o = st.solve_nonrigid(pose, t, 0)
    gn, on = ctx.download_nodes(), st.get_nodes()
    ctx.forward_warp()
    st.forward_warp()
    gm, om = ctx.download_model(), st.get_model()
    print(scene, "iters", g.iterations, o.iterations, "corr", g.correspondences, o.correspondences,
          "e0 rel %.2e" % (abs(g.initial_energy - o.initial_energy) / o.initial_energy),
          "e1 gap/e0 %.2e" % (abs(g.final_energy - o.final_energy) / o.initial_energy),
          "dq %.2e" % dq_close(gn["dq"], on["dq"]),
          "warp %.2e m" % np.abs(gm["live_pos"] - om["live_pos"]).max(),
          "mr %.2e" % abs(g.mean_residual - o.mean_residual), flush=True)
