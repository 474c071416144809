"""cfg2 frame-2 normal-equation mismatch: compare the full device state with the
oracle's after frame 1 (each ran its own fusion on the shared post-solve state),
then locate the differing JtJ blocks at frame 2."""
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
gfu = ctx.apply_fusion(pose, t)
ofu = st.apply_fusion(pose, t)
print("fusion new nodes", gfu.new_nodes, ofu.new_nodes, "appended", gfu.appended, ofu.appended)
gm, om = Hh.device_to_oracle_model(ctx.download_model()), st.get_model()
gn, on = ctx.download_nodes(), st.get_nodes()
for k in gn:
    a, b = np.asarray(gn[k]), np.asarray(on[k])
    print("node", k, a.shape, b.shape, "equal" if a.shape == b.shape and np.array_equal(a, b) else
          ("maxdiff %.3e" % np.abs(a - b).max() if a.shape == b.shape else "shape"))
    if k == "nbr" and a.shape == b.shape:
        bad = np.nonzero((a != b).any(1))[0]
        print("   nodes with different nbr:", bad[:20], len(bad))
        for j in bad[:5]:
            print("   ", j, a[j], b[j])
for k in om:
    a, b = np.asarray(gm[k]), np.asarray(om[k])
    if a.shape != b.shape:
        print("model", k, "shape", a.shape, b.shape)
        continue
    if np.array_equal(a, b):
        continue
    d = np.abs(a.astype(np.float64) - b.astype(np.float64))
    print("model", k, "maxdiff %.3e" % d.max(), "rows", np.count_nonzero(d.reshape(len(d), -1).max(1)))
# oracle from-scratch edges vs the device's
st2 = O.OracleState(Hh.oracle_cfg(cfg))
st2.set_nodes(gn)
st2.compute_node_edges(8)
print("device nbr == oracle recomputed edges:", np.array_equal(st2.get_nodes()["nbr"], gn["nbr"]))
# frame 2
t = 2
ctx.frame_maps(depth[t], t)
st.build_frame(depth[t], t)
L.sync_oracle(st, ctx)
ctx.forward_warp()
L.sync_oracle(st, ctx)
ne = ctx.build_normal_equations(pose, t, 0)
o = st.normal_equations(pose, t, 0)
N = ctx.num_nodes()
Hg, Tg = Hh.bsr_to_dense(ne, N)
To = o["touched"]
diff = np.argwhere(Tg != To)
print("touched diffs", len(diff), diff[:20].tolist(), "dev", Tg[tuple(diff[:5].T)] if len(diff) else "", "or",
      To[tuple(diff[:5].T)] if len(diff) else "")
Hd = np.abs(Hg - o["h"]).reshape(N, 6, N, 6).max(axis=(1, 3))
bad = np.argwhere(Hd > 1e-6 * np.abs(o["h"]).max())
print("H blocks differing", len(bad), bad[:20].tolist())
print("e_pre", ne["e_pre"], o["e_pre"], "pairs", ne["n_pairs"], o["n_pairs"])
gd = np.abs(ne["g"] - o["g"]).reshape(N, 6).max(1)
print("g nodes differing", np.argwhere(gd > 1e-6 * np.abs(o["g"]).max()).ravel()[:30])
