"""JtJ / g accuracy of the device assembly against the oracle's fp64 assembly
(the test_normal_equations_pattern_and_values setup), as error statistics."""
import os
import sys

import numpy as np

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, root)
sys.path.insert(0, os.path.join(root, "tests"))
import harness as Hh  # noqa: E402
import oracle_py as O  # noqa: E402
import test_gpu_stages as T  # noqa: E402

for seed in (7, 8, 9):
    cfg, seq = T.scene()
    d0 = seq.render_depth(0)
    model, _ = T.frame_model(cfg, d0)
    ctx, st = T._init_both(cfg, model)
    T._random_field(ctx, st, np.random.default_rng(seed), angle=0.02, shift=0.003)
    st.set_model(Hh.device_to_oracle_model(ctx.download_model()))
    ctx.frame_maps(d0, 1)
    st.build_frame(d0, 1)
    pose = O.pose_identity()
    g = ctx.build_normal_equations(pose, 1, 0)
    o = st.normal_equations(pose, 1, 0)
    Hg, _ = Hh.bsr_to_dense(g, ctx.num_nodes())
    dh = Hg - o["h"]
    print(seed, "H maxrel %.3e frob %.3e" % (np.abs(dh).max() / np.abs(o["h"]).max(),
                                           np.linalg.norm(dh) / np.linalg.norm(o["h"])),
          "g maxrel %.3e" % (np.abs(g["g"] - o["g"]).max() / np.abs(o["g"]).max()))
    ctx.close()
