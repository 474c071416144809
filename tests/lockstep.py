"""Lock-step parity harness on BASELINE sequences. TEST INFRASTRUCTURE.

The reference's per-frame chain (pipeline.cpp:74-142: build_frame_maps ->
render_model_maps + rigid_align -> solve_nonrigid -> forward_warp ->
apply_fusion) is driven stage by stage on the device (ds_* stage entry points
of one context) and on the CPU oracle. Before every stage the oracle is handed
the device's fp32 state, so each stage is compared on identical inputs:

  frame maps, fusion counts / order, node sets, skinning  -> bit-exact
  rigid pose, solve (node SE(3), warped surfels, energies) -> measured gaps

A free-running comparison of two whole sequences is chaotic (the oracle's own
fp64 and fp32-mirror runs part ways by frame 2 on config 1: one marginal
fusion decision moves thousands of appends a few frames later), so
sequence-level parity is stated per frame on shared state.

A second device object, the production `Pipeline` (ds_process_frame: fused
warp / index map, side-stream pattern build, deferred node updates), runs the
same frames; its per-frame stats are compared with the stage chain's.
"""
from __future__ import annotations

import numpy as np

import harness as Hh
import oracle_py as O


def dq_gap(a, b):
    s = np.where((a[:, :4] * b[:, :4]).sum(1) < 0, -1.0, 1.0)[:, None]
    return float(np.abs(s * a - b).max()) if len(a) else 0.0


def model_gap(gm, om, key_g="live_pos", key_o="live_pos"):
    return float(np.abs(np.asarray(gm[key_g]) - np.asarray(om[key_o])).max()) if len(gm[key_g]) else 0.0


def sync_oracle(st, ctx):
    st.set_model(Hh.device_to_oracle_model(ctx.download_model()))
    st.set_nodes(ctx.download_nodes())


def init_both(pkg, cfg, depth0):
    """Frame 0: device initialize_from_frame vs the oracle pipeline's (mirror)."""
    ctx = pkg.Context(cfg)
    s0 = ctx.process_frame(depth0, 0)
    ore = O.OraclePipeline(Hh.oracle_cfg(cfg), mirror=True)
    o0 = ore.process_frame(depth0, 0)
    gm, om = ctx.download_model(), ore.state.get_model()
    gn, on = ctx.download_nodes(), ore.state.get_nodes()
    rec = dict(valid=(s0.valid_pixels, o0.valid_pixels),
               surfels=(s0.surfel_count, o0.surfel_count),
               nodes=(s0.node_count, o0.node_count),
               node_pos_equal=bool(np.array_equal(gn["pos"], on["pos"])),
               node_nbr_equal=bool(np.array_equal(gn["nbr"], on["nbr"])),
               skin_idx_equal=bool(np.array_equal(gm["skin_idx"], om["skin_idx"])),
               skin_count_equal=bool(np.array_equal(gm["skin_count"], om["skin_count"])),
               ref_pos_gap=model_gap(gm, om, "ref_pos", "ref_pos"),
               skin_w_rel_gap=float(np.max(np.abs(gm["skin_w"] - om["skin_w"]) /
                                           np.maximum(np.abs(om["skin_w"]), 1e-30))))
    return ctx, rec


def frame_step(pkg, ctx, st, depth, t, t_last, solve_variants=()):
    """One lock-step frame. Returns the record of per-stage comparisons."""
    rec = dict(frame=t)
    pose = ctx.get_pose()
    # (1) build_frame_maps (depth_processing.cpp:103-138)
    vc = ctx.frame_maps(depth, t)
    st.build_frame(depth, t)
    gf, of = ctx.download_frame(), st.get_frame()
    rec["valid"] = (vc, of["valid_count"])
    rec["frame_maps_equal"] = bool(np.array_equal(gf["valid"], of["valid"]) and
                                   np.array_equal(gf["vert"], of["vert"]) and
                                   np.array_equal(gf["nrm"], of["nrm"]))
    # (2) rigid_align (solver.cpp:171-242) on the shared model
    sync_oracle(st, ctx)
    g = ctx.rigid_align(pose, pose, t, t_last)
    o = st.rigid_align(pose, pose, t, t_last)
    rec["rigid_pose_gap"] = float(np.abs(np.array(g.pose) - np.array(o.pose)).max())
    rec["rigid_pairs"] = (g.correspondences, o.correspondences)
    pose = list(g.pose)
    ctx.set_pose(pose)
    # (3) solve_nonrigid (solver.cpp:296-420) on the shared model and nodes
    for name, vctx in solve_variants:  # other device PCG settings, same state
        vctx.upload_model(ctx.download_model())
        vctx.upload_nodes(ctx.download_nodes())
        vctx.frame_maps(depth, t)
    gs = ctx.solve_nonrigid(pose, t, t_last)
    os_ = st.solve_nonrigid(pose, t, t_last)
    ctx.forward_warp()
    st.forward_warp()
    gm, om = ctx.download_model(), st.get_model()
    gn, on = ctx.download_nodes(), st.get_nodes()
    rec["solve"] = _solve_rec(gs, os_, gm, om, gn, on)
    for name, vctx in solve_variants:
        vs = vctx.solve_nonrigid(pose, t, t_last)
        vctx.forward_warp()
        rec["solve_" + name] = _solve_rec(vs, os_, vctx.download_model(), om,
                                          vctx.download_nodes(), on)
    # (4) apply_fusion (fusion.cpp:220-307) on the shared post-solve state
    sync_oracle(st, ctx)
    gfu = ctx.apply_fusion(pose, t)
    ofu = st.apply_fusion(pose, t)
    keys = ("fused", "appended", "removed", "compressive_rejected", "low_support_rejected",
            "new_nodes", "degenerate_warps")
    rec["fusion"] = {k: (getattr(gfu, k), getattr(ofu, k)) for k in keys}
    gm, om = ctx.download_model(), st.get_model()
    gn, on = ctx.download_nodes(), st.get_nodes()
    rec["surfels"] = (len(gm["ref_pos"]), len(om["ref_pos"]))
    rec["nodes"] = (len(gn["pos"]), len(on["pos"]))
    same_n = len(gm["ref_pos"]) == len(om["ref_pos"])
    rec["fusion_skin_idx_equal"] = bool(same_n and np.array_equal(gm["skin_idx"], om["skin_idx"]))
    rec["fusion_t_obs_equal"] = bool(same_n and np.array_equal(gm["t_obs"], om["live_t_obs"]))
    rec["fusion_live_gap"] = model_gap(gm, om) if same_n else None
    rec["fusion_ref_gap"] = model_gap(gm, om, "ref_pos", "ref_pos") if same_n else None
    rec["fusion_conf_gap"] = (float(np.abs(gm["conf"] - om["live_conf"]).max())
                              if same_n and len(gm["conf"]) else None)
    rec["node_pos_equal"] = bool(len(gn["pos"]) == len(on["pos"]) and
                                 np.array_equal(gn["pos"], on["pos"]))
    rec["node_nbr_equal"] = bool(len(gn["pos"]) == len(on["pos"]) and
                                 np.array_equal(gn["nbr"], on["nbr"]))
    rec["pose"] = pose
    return rec


def _solve_rec(g, o, gm, om, gn, on):
    scale = max(float(np.abs(om["live_pos"]).max()), 1e-30) if len(om["live_pos"]) else 1.0
    warp_gap = model_gap(gm, om)
    return dict(iterations=(g.iterations, o.iterations),
                correspondences=(g.correspondences, o.correspondences),
                e0_rel=abs(g.initial_energy - o.initial_energy) / max(o.initial_energy, 1e-30),
                e1=(g.final_energy, o.final_energy),
                e1_rel_e0=abs(g.final_energy - o.final_energy) / max(o.initial_energy, 1e-30),
                mean_residual=(g.mean_residual, o.mean_residual),
                node_dq_gap=dq_gap(gn["dq"], on["dq"]),
                warp_pos_gap_m=warp_gap, warp_pos_gap_rel=warp_gap / scale,
                warp_nrm_gap=model_gap(gm, om, "live_nrm", "live_nrm"))


def run(pkg, cfg, scene, frames, seq_frames=None, solve_variants=None, pipeline=True, log=None):
    """Lock-step run over `frames` frames; returns (init record, frame records,
    production-pipeline stats per frame or None)."""
    seq = pkg.SyntheticSequence(scene, seq_frames or frames, cfg)
    depth = [seq.render_depth(t) for t in range(frames)]
    ctx, rec0 = init_both(pkg, cfg, depth[0])
    if log:
        log(0, rec0)
    st = O.OracleState(Hh.oracle_cfg(cfg))
    st.set_mirror(True)
    variants = [(n, pkg.Context(c)) for n, c in (solve_variants or {}).items()]
    recs = []
    for t in range(1, frames):
        r = frame_step(pkg, ctx, st, depth[t], t, 0, variants)
        recs.append(r)
        if log:
            log(t, r)
    pstats = None
    if pipeline:
        p = pkg.Pipeline(cfg)
        pstats = [p.process_frame(d, t) for t, d in enumerate(depth)]
        p.close()
    for _, v in variants:
        v.close()
    ctx.close()
    return rec0, recs, pstats
