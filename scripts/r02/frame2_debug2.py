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

t = 2
ctx.frame_maps(depth[t], t)
st.build_frame(depth[t], t)
full = ctx.download_model()
nodes = ctx.download_nodes()
N = ctx.num_nodes()


def subset(m, keep):
    out = {}
    for k, v in m.items():
        out[k] = np.ascontiguousarray(np.asarray(v)[keep])
    return out


def compare(label, keep):
    m = subset(full, keep)
    ctx.upload_model(m)
    ctx.upload_nodes(nodes)
    ctx.forward_warp()
    L.sync_oracle(st, ctx)
    ne = ctx.build_normal_equations(pose, t, 0)
    o = st.normal_equations(pose, t, 0)
    Hg, Tg = Hh.bsr_to_dense(ne, N)
    Hd = np.abs(Hg - o["h"]).reshape(N, 6, N, 6).max(axis=(1, 3))
    bad = np.argwhere(Hd > 1e-6 * np.abs(o["h"]).max())
    print(label, "surfels", int(keep.sum()), "pairs", ne["n_pairs"], o["n_pairs"], "touched diff",
          int((Tg != o["touched"]).sum()), "H blocks differing", len(bad), bad[:8].tolist(),
          "e_pre rel %.3e" % (abs(ne["e_pre"] - o["e_pre"]) / o["e_pre"]), flush=True)
    return bad


tin = np.asarray(full["t_init"])
cnt = np.asarray(full["skin_count"])
print("t_init values", np.unique(tin, return_counts=True), "skin counts", np.unique(cnt, return_counts=True))
bad = compare("all", np.ones(len(tin), bool))
compare("t_init==0", tin == 0)
compare("t_init==1", tin == 1)
compare("count==4", cnt == 4)
compare("count<4", cnt < 4)
if len(bad):
    j = bad[0][0]
    idx = np.asarray(full["skin_idx"]).reshape(len(tin), 8)
    hit = np.nonzero((idx == j).any(1))[0]
    print("surfels skinned to node", j, len(hit), "t_init", np.unique(tin[hit], return_counts=True),
          "counts", np.unique(cnt[hit], return_counts=True))
    print("node", j, "pos", nodes["pos"][j], "nbr", nodes["nbr"][j], "dq", nodes["dq"][j])
