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


sub = np.array([15204, 15205, 15206, 15207, 15208, 15209, 15210, 15211, 15212, 15472, 15473, 15474, 15475, 15476, 15477, 15478, 15479, 15480, 15481, 15482, 15483, 15484, 15485, 15486, 15487, 15488, 15489, 15490, 15758, 15759, 15760, 15761, 15762, 15763, 15764, 15765])
keep = np.zeros(len(full["t_init"]), bool)
keep[sub] = True
m = subset(full, keep)
ctx.upload_model(m)
ctx.upload_nodes(nodes)
ctx.forward_warp()
L.sync_oracle(st, ctx)
mg = ctx.render_model_maps(pose, t, 0)
mo = st.render_model_maps(pose, t, 0)
d = np.argwhere(mg["idx"] != mo["idx"])
print("stage model maps idx diffs", len(d), [(int(y), int(x), int(mg["idx"][y, x]), int(mo["idx"][y, x])) for y, x in d[:10]])
pg = ctx.associate(pose)
po = st.find_correspondences(mo, pose)
print("stage pairs", len(pg["surfel"]), len(po["surfel"]), "equal", len(pg["surfel"]) == len(po["surfel"]) and all(np.array_equal(pg[k], po[k]) for k in ("surfel", "px", "py")))
ne = ctx.build_normal_equations(pose, t, 0)
o = st.normal_equations(pose, t, 0)
print("normal eq pairs", ne["n_pairs"], o["n_pairs"], "e_pre", ne["e_pre"], o["e_pre"])
pl = ctx.associate(pose)  # winners of the linearisation's own model maps
print("linearise pairs", len(pl["surfel"]))
a = {(int(x), int(y)): int(s) for s, x, y in zip(pl["surfel"], pl["px"], pl["py"])}
b = {(int(x), int(y)): int(s) for s, x, y in zip(po["surfel"], po["px"], po["py"])}
diff = sorted(set(a.items()) ^ set(b.items()))
print("pair diffs (dev ^ oracle)", len(diff), diff[:20])
for (x, y), s in diff[:6]:
    print("  px", x, y, "dev", a.get((x, y)), "or", b.get((x, y)), "oracle map idx", int(mo["idx"][y, x]), "depth", float(mo["depth"][y, x]))
gmm = ctx.download_model()
for sidx in sorted(set(s for _, s in diff))[:6]:
    print("  surfel", sidx, "dev live", gmm["live_pos"][sidx].tolist(), "conf", float(gmm["conf"][sidx]))
# pixel-level: per-pair residuals from the oracle on the stage pairs
for k in range(min(5, len(po["surfel"]))):
    print(" pair", int(po["surfel"][k]), int(po["px"][k]), int(po["py"][k]))
# the same after a fresh context (no z-buffer history)
ctx2 = pkg.Context(cfg)
ctx2.upload_model(m)
ctx2.upload_nodes(nodes)
ctx2.frame_maps(depth[t], t)
ctx2.forward_warp()
ne2 = ctx2.build_normal_equations(pose, t, 0)
print("fresh ctx normal eq pairs", ne2["n_pairs"], "e_pre", ne2["e_pre"])
ne3 = ctx2.build_normal_equations(pose, t, 0)
print("fresh ctx again", ne3["n_pairs"], "e_pre", ne3["e_pre"])
