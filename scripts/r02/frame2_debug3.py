"""Where do the frame-2 pairs of the GN linearisation part from the oracle's?"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import harness as Hh  # noqa: E402
import lockstep as L  # noqa: E402
import oracle_py as O  # noqa: E402
import paper_1904_13073_b200 as pkg  # noqa: E402

cfg = pkg.camera_config(640, 480, 560.0, max_gn_iters=10, pcg_tol=1e-12, pcg_max_iters=2000)
seq = pkg.SyntheticSequence("articulated_body", 100, cfg)
depth = [seq.render_depth(t) for t in range(3)]
ctx, rec0 = L.init_both(pkg, cfg, depth[0])
st = O.OracleState(Hh.oracle_cfg(cfg))
st.set_mirror(True)
pose = ctx.get_pose()
t = 1
ctx.frame_maps(depth[t], t)
st.build_frame(depth[t], t)
L.sync_oracle(st, ctx)
g = ctx.rigid_align(pose, pose, t, 0)
pose = list(g.pose)
ctx.set_pose(pose)
ctx.solve_nonrigid(pose, t, 0)
ctx.forward_warp()
L.sync_oracle(st, ctx)
ctx.apply_fusion(pose, t)
t = 2
ctx.frame_maps(depth[t], t)
st.build_frame(depth[t], t)
L.sync_oracle(st, ctx)
f32 = lambda a: np.asarray(a).astype(np.float32).astype(np.float64)  # noqa: E731
# (1) forward warp from the same state
ctx.forward_warp()
st.forward_warp()
gm, om = ctx.download_model(), st.get_model()
mp = (gm["live_pos"] != f32(om["live_pos"])).any(1)
mn = (gm["live_nrm"] != f32(om["live_nrm"])).any(1)
print("forward warp mismatches: pos", int(mp.sum()), "nrm", int(mn.sum()), "of", len(mp),
      "max pos diff", float(np.abs(gm["live_pos"] - om["live_pos"]).max()))
idx = np.nonzero(mp | mn)[0][:5]
for i in idx:
    print("  surfel", i, "dev", gm["live_pos"][i], "or", om["live_pos"][i], "ordiff",
          gm["live_pos"][i] - om["live_pos"][i])
# (2) model maps + association on each side's own warp
st.set_model(dict(Hh.device_to_oracle_model(gm), live_pos=f32(om["live_pos"]),
                  live_nrm=f32(om["live_nrm"])))
mg = ctx.render_model_maps(pose, t, 0)
mo = st.render_model_maps(pose, t, 0)
print("model maps: valid diff", int((mg["valid"] != mo["valid"]).sum()), "idx diff",
      int((mg["idx"] != mo["idx"]).sum()))
pg = ctx.associate(pose)
po = st.find_correspondences(mo, pose)
print("pairs", len(pg["surfel"]), len(po["surfel"]))
# (3) the linearisation's association, pair count only
ne = ctx.build_normal_equations(pose, t, 0)
o = st.normal_equations(pose, t, 0)
print("normal eq pairs", ne["n_pairs"], o["n_pairs"], "e_pre rel %.3e" % (abs(ne["e_pre"] - o["e_pre"]) / o["e_pre"]))
