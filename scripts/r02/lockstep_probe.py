"""Measure the lock-step parity gaps on BASELINE configs (inputs for the
tolerances written into tests/test_gpu_baseline_parity.py)."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import harness as Hh  # noqa: E402
import lockstep as L  # noqa: E402
import oracle_py as O  # noqa: E402
import paper_1904_13073_b200 as pkg  # noqa: E402

CONVERGED = dict(pcg_tol=1e-12, pcg_max_iters=2000)


def log(t, r):
    print(t, json.dumps(r, default=lambda x: str(x)), flush=True)


def cfg1():
    base = dict(max_gn_iters=3)
    cfg = pkg.camera_config(320, 240, 280.0, **base, **CONVERGED)
    variants = {"pcg10": pkg.camera_config(320, 240, 280.0, max_gn_iters=3, pcg_max_iters=10),
                "tol1e-6": pkg.camera_config(320, 240, 280.0, max_gn_iters=3, pcg_max_iters=500,
                                             pcg_tol=1e-6)}
    t0 = time.time()
    rec0, recs, pst = L.run(pkg, cfg, "deforming_sphere", 10, solve_variants=variants, log=log)
    print("cfg1 lockstep done in", round(time.time() - t0, 1), "s")
    # production pipeline vs the stage chain
    for r, d in zip(recs, pst[1:]):
        print("pipe-vs-chain f%d surfels %s/%s nodes %s/%s fused %s/%s pose %.3e corr %s/%s" % (
            r["frame"], d["surfel_count"], r["surfels"][0], d["node_count"], r["nodes"][0],
            d["fused"], r["fusion"]["fused"][0],
            float(np.abs(np.array(d["pose"]) - np.array(r["pose"])).max()),
            d["correspondences"], r["solve"]["correspondences"][0]), flush=True)


def cfg2(frames=3):
    cfg = pkg.camera_config(640, 480, 560.0, max_gn_iters=10, **CONVERGED)
    seq = pkg.SyntheticSequence("articulated_body", 100, cfg)
    depth = [seq.render_depth(t) for t in range(frames)]
    t0 = time.time()
    ctx, rec0 = L.init_both(pkg, cfg, depth[0])
    log(0, rec0)
    print("cfg2 init", round(time.time() - t0, 1), "s", flush=True)
    st = O.OracleState(Hh.oracle_cfg(cfg))
    st.set_mirror(True)
    pose = ctx.get_pose()
    for t in range(1, frames):
        rec = dict(frame=t)
        vc = ctx.frame_maps(depth[t], t)
        st.build_frame(depth[t], t)
        gf, of = ctx.download_frame(), st.get_frame()
        rec["frame_maps_equal"] = bool(np.array_equal(gf["valid"], of["valid"]) and
                                       np.array_equal(gf["vert"], of["vert"]))
        L.sync_oracle(st, ctx)
        t1 = time.time()
        g = ctx.rigid_align(pose, pose, t, 0)
        o = st.rigid_align(pose, pose, t, 0)
        rec["rigid_pose_gap"] = float(np.abs(np.array(g.pose) - np.array(o.pose)).max())
        rec["rigid_pairs"] = (g.correspondences, o.correspondences)
        pose = list(g.pose)
        ctx.set_pose(pose)
        rec["t_rigid"] = round(time.time() - t1, 2)
        # warp + model maps + association, shared live state
        ctx.forward_warp()
        L.sync_oracle(st, ctx)
        mg = ctx.render_model_maps(pose, t, 0)
        mo = st.render_model_maps(pose, t, 0)
        rec["model_maps_equal"] = bool(np.array_equal(mg["valid"], mo["valid"]) and
                                       np.array_equal(mg["idx"], mo["idx"]))
        pg = ctx.associate(pose)
        po = st.find_correspondences(mo, pose)
        rec["pairs"] = (len(pg["surfel"]), len(po["surfel"]))
        rec["pairs_equal"] = bool(all(np.array_equal(pg[k], po[k]) for k in ("surfel", "px", "py")))
        t1 = time.time()
        ne = ctx.build_normal_equations(pose, t, 0)
        on = st.normal_equations(pose, t, 0)
        N = ctx.num_nodes()
        Hg, Tg = Hh.bsr_to_dense(ne, N)
        rec["t_normal_eq"] = round(time.time() - t1, 2)
        rec["touched_equal"] = bool(np.array_equal(Tg, on["touched"]))
        rec["touched_blocks"] = int(on["touched"].sum())
        scale = np.abs(on["h"]).max()
        rec["H_gap_rel"] = float(np.abs(Hg - on["h"]).max() / scale)
        rec["g_gap_rel"] = float(np.abs(ne["g"] - on["g"]).max() / np.abs(on["g"]).max())
        rec["e_pre_rel"] = float(abs(ne["e_pre"] - on["e_pre"]) / on["e_pre"])
        # one damped GN step: device PCG (converged) on the device system vs a
        # dense solve of the oracle's system
        mu = 1e-6 * np.trace(on["h"]) / (6 * N)
        t1 = time.time()
        delta, it, rel = ctx.pcg_solve(mu, 2000, 1e-12)
        ref = np.linalg.solve(on["h"] + mu * np.eye(6 * N), -on["g"])
        rec["step_gap_rel"] = float(np.abs(delta - ref).max() / np.abs(ref).max())
        for iters in (10, 20, 40):
            d10, _, r10 = ctx.pcg_solve(mu, iters, 0.0)
            rec[f"step_gap_rel_pcg{iters}"] = float(np.abs(d10 - ref).max() / np.abs(ref).max())
            rec[f"rel_res_pcg{iters}"] = float(r10)
        rec["t_solve"] = round(time.time() - t1, 2)
        # restore the pre-solve live state, device solve, then shared fusion
        ctx.forward_warp()
        gs = ctx.solve_nonrigid(pose, t, 0)
        rec["solve_iters"] = gs.iterations
        ctx.forward_warp()
        L.sync_oracle(st, ctx)
        t1 = time.time()
        gfu = ctx.apply_fusion(pose, t)
        ofu = st.apply_fusion(pose, t)
        rec["t_fusion"] = round(time.time() - t1, 2)
        keys = ("fused", "appended", "removed", "compressive_rejected", "low_support_rejected",
                "new_nodes", "degenerate_warps")
        rec["fusion"] = {k: (getattr(gfu, k), getattr(ofu, k)) for k in keys}
        gm, om = ctx.download_model(), st.get_model()
        gn, onn = ctx.download_nodes(), st.get_nodes()
        same = len(gm["ref_pos"]) == len(om["ref_pos"])
        rec["surfels"] = (len(gm["ref_pos"]), len(om["ref_pos"]))
        rec["skin_idx_equal"] = bool(same and np.array_equal(gm["skin_idx"], om["skin_idx"]))
        rec["node_pos_equal"] = bool(len(gn["pos"]) == len(onn["pos"]) and
                                     np.array_equal(gn["pos"], onn["pos"]))
        rec["live_gap"] = L.model_gap(gm, om) if same else None
        log(t, rec)
    ctx.close()


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
    if which == "cfg1":
        cfg1()
    else:
        cfg2(int(sys.argv[2]) if len(sys.argv) > 2 else 3)
