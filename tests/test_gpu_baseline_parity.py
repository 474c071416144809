"""Parity on BASELINE configurations.

config 1  deforming sphere, 320x240, ~30k surfels, ~300 nodes, 10 frames,
          3 GN iterations: the whole sequence in lock-step (tests/lockstep.py)
          -- every frame's stages on the device and on the oracle from the
          same fp32 state. Bit-exact: frame maps, node sets / edges /
          skinning, fusion counts and the fused model. Solve: warped surfels
          after the full GN solve within 5e-5 relative with the PCG run to
          convergence (measured 5e-6); with the benchmarked 10-PCG budget the
          measured gap (1.0e-3) sets the stated tolerance (2e-3 relative,
          DESIGN.md §5).
          The production Pipeline (ds_process_frame: fused passes, side
          stream, deferred updates) is bit-identical to the stage chain.
config 2  articulated body, 640x480, ~185k surfels, ~1.5k nodes: frame 0
          initialisation and the frame 1 -> 2 stage chain: frame maps, node
          set, skinning, model-map winners, correspondence pairs (set and
          order), JtJ block pattern bit-exact; H within 2e-6 max|H|, g within
          1e-5; one converged GN step solves the oracle's system to a relative
          residual of 1e-5; fusion outcome counts exact.
Reference: pipeline.cpp:74-142, solver.cpp:296-420, fusion.cpp:220-307.
"""
import numpy as np
import pytest

import harness as Hh
import lockstep as L
import oracle_py as O

pytestmark = pytest.mark.gpu
pkg = pytest.importorskip("paper_1904_13073_b200")

CONVERGED = dict(pcg_tol=1e-12, pcg_max_iters=2000)
FUSION_KEYS = ("fused", "appended", "removed", "compressive_rejected", "low_support_rejected",
               "new_nodes", "degenerate_warps")


@pytest.fixture(scope="module")
def cfg1_run():
    cfg = pkg.camera_config(320, 240, 280.0, max_gn_iters=3, **CONVERGED)
    bench_cfg = pkg.camera_config(320, 240, 280.0, max_gn_iters=3, pcg_max_iters=10)
    return L.run(pkg, cfg, "deforming_sphere", 10, solve_variants={"pcg10": bench_cfg})


def test_cfg1_initialisation_bit_exact(cfg1_run):
    rec0, _, _ = cfg1_run
    assert rec0["valid"][0] == rec0["valid"][1] > 25000
    assert rec0["surfels"][0] == rec0["surfels"][1]
    assert rec0["nodes"][0] == rec0["nodes"][1] > 250
    for k in ("node_pos_equal", "node_nbr_equal", "skin_idx_equal", "skin_count_equal"):
        assert rec0[k], k
    assert rec0["ref_pos_gap"] == 0.0
    assert rec0["skin_w_rel_gap"] <= 1.2e-7  # fp32 weight storage


def test_cfg1_frame_maps_and_rigid(cfg1_run):
    _, recs, _ = cfg1_run
    for r in recs:
        assert r["valid"][0] == r["valid"][1], r["frame"]
        assert r["frame_maps_equal"], r["frame"]
        assert r["rigid_pairs"][0] == r["rigid_pairs"][1], r["frame"]
        assert r["rigid_pose_gap"] < 1e-9, (r["frame"], r["rigid_pose_gap"])


def test_cfg1_solve_converged_pcg(cfg1_run):
    _, recs, _ = cfg1_run
    for r in recs:
        s = r["solve"]
        assert s["iterations"][0] == s["iterations"][1], r["frame"]
        assert s["correspondences"][0] == s["correspondences"][1], r["frame"]
        assert s["e0_rel"] < 1e-12, (r["frame"], s["e0_rel"])
        assert s["e1_rel_e0"] < 1e-4, (r["frame"], s["e1_rel_e0"])
        # the north star's bar: warped surfels after the full GN solve
        # (measured: <= 5.2e-6 relative / 3.2e-6 m, node DQs <= 6.5e-5)
        assert s["warp_pos_gap_rel"] < 5e-5, (r["frame"], s["warp_pos_gap_rel"])
        assert s["warp_nrm_gap"] < 5e-4, (r["frame"], s["warp_nrm_gap"])
        assert s["node_dq_gap"] < 5e-4, (r["frame"], s["node_dq_gap"])


def test_cfg1_solve_benchmark_budget(cfg1_run):
    """10 PCG iterations per LM attempt (the benchmarked setting): the GN
    result differs from the LDLT path by the truncated inner solve; measured
    on this sequence up to 1.0e-3 relative (0.63 mm) on warped surfels -- the
    stated tolerance for this setting is 2e-3."""
    _, recs, _ = cfg1_run
    for r in recs:
        s = r["solve_pcg10"]
        assert s["correspondences"][0] == s["correspondences"][1], r["frame"]
        assert s["warp_pos_gap_rel"] < 2e-3, (r["frame"], s["warp_pos_gap_rel"])
        # final energy within 1 % of the initial one (measured <= 0.35 %)
        assert s["e1_rel_e0"] < 1e-2, (r["frame"], s["e1_rel_e0"])


def test_cfg1_fusion_bit_exact(cfg1_run):
    _, recs, _ = cfg1_run
    for r in recs:
        for k in FUSION_KEYS:
            assert r["fusion"][k][0] == r["fusion"][k][1], (r["frame"], k, r["fusion"][k])
        assert r["surfels"][0] == r["surfels"][1] and r["nodes"][0] == r["nodes"][1]
        for k in ("fusion_skin_idx_equal", "fusion_t_obs_equal", "node_pos_equal",
                  "node_nbr_equal"):
            assert r[k], (r["frame"], k)
        assert r["fusion_live_gap"] == 0.0 and r["fusion_ref_gap"] == 0.0
        assert r["fusion_conf_gap"] == 0.0


def test_cfg1_pipeline_equals_stage_chain(cfg1_run):
    """ds_process_frame (fused warp + index map, side-stream pattern build,
    deferred node updates) gives the same frames as the stage entry points."""
    _, recs, pst = cfg1_run
    for r, d in zip(recs, pst[1:]):
        assert d["surfel_count"] == r["surfels"][0], r["frame"]
        assert d["node_count"] == r["nodes"][0], r["frame"]
        assert d["correspondences"] == r["solve"]["correspondences"][0], r["frame"]
        for k in FUSION_KEYS:
            assert d[k] == r["fusion"][k][0], (r["frame"], k)
        assert d["pose"] == list(r["pose"]), r["frame"]


def test_cfg2_stage_chain():
    cfg = pkg.camera_config(640, 480, 560.0, max_gn_iters=10, **CONVERGED)
    seq = pkg.SyntheticSequence("articulated_body", 100, cfg)
    depth = [seq.render_depth(t) for t in range(3)]
    ctx, rec0 = L.init_both(pkg, cfg, depth[0])
    assert rec0["surfels"][0] == rec0["surfels"][1] > 150000
    assert rec0["nodes"][0] == rec0["nodes"][1] > 1200
    for k in ("node_pos_equal", "node_nbr_equal", "skin_idx_equal", "skin_count_equal"):
        assert rec0[k], k
    st = O.OracleState(Hh.oracle_cfg(cfg))
    st.set_mirror(True)
    pose = ctx.get_pose()
    for t in (1, 2):
        ctx.frame_maps(depth[t], t)
        st.build_frame(depth[t], t)
        gf, of = ctx.download_frame(), st.get_frame()
        assert np.array_equal(gf["valid"], of["valid"]) and np.array_equal(gf["vert"], of["vert"])
        L.sync_oracle(st, ctx)
        g = ctx.rigid_align(pose, pose, t, 0)
        o = st.rigid_align(pose, pose, t, 0)
        assert g.correspondences == o.correspondences
        assert np.abs(np.array(g.pose) - np.array(o.pose)).max() < 1e-9
        pose = list(g.pose)
        ctx.set_pose(pose)
        # warp, model maps, association on the shared live state
        ctx.forward_warp()
        gl = ctx.download_model()
        st.forward_warp()
        ol = st.get_model()
        f32 = lambda a: np.asarray(a).astype(np.float32).astype(np.float64)  # noqa: E731
        assert np.array_equal(gl["live_pos"], f32(ol["live_pos"]))
        assert np.array_equal(gl["live_nrm"], f32(ol["live_nrm"]))
        L.sync_oracle(st, ctx)
        mg = ctx.render_model_maps(pose, t, 0)
        mo = st.render_model_maps(pose, t, 0)
        assert np.array_equal(mg["valid"], mo["valid"]) and np.array_equal(mg["idx"], mo["idx"])
        pg = ctx.associate(pose)
        po = st.find_correspondences(mo, pose)
        assert len(pg["surfel"]) == len(po["surfel"]) > 150000
        for k in ("surfel", "px", "py"):
            assert np.array_equal(pg[k], po[k]), k
        # the GN linearisation (its own warp + model maps + association)
        ne = ctx.build_normal_equations(pose, t, 0)
        on = st.normal_equations(pose, t, 0)
        pl = ctx.associate(pose)  # the linearisation's winners
        for k in ("surfel", "px", "py"):
            assert np.array_equal(pl[k], po[k]), k
        N = ctx.num_nodes()
        Hg, Tg = Hh.bsr_to_dense(ne, N)
        assert ne["n_pairs"] == on["n_pairs"]
        assert np.array_equal(Tg, on["touched"])  # JtJ sparsity pattern
        assert np.abs(Hg - on["h"]).max() <= 2e-6 * np.abs(on["h"]).max()
        assert np.abs(ne["g"] - on["g"]).max() <= 1e-5 * np.abs(on["g"]).max()
        assert abs(ne["e_pre"] - on["e_pre"]) <= 1e-9 * on["e_pre"]
        # one damped step: the converged device PCG step solves the ORACLE's
        # system (H fp64, g) to a relative residual of 1e-5 (backward error;
        # the forward gap to a dense solve, measured 2.4e-3 relative, is the
        # fp32 block storage amplified by the system's conditioning -- weakly
        # observed nodes, solver.cpp:375-377)
        mu = 1e-6 * np.trace(on["h"]) / (6 * N)
        delta, it, rel = ctx.pcg_solve(mu, 2000, 1e-12)
        A = on["h"] + mu * np.eye(6 * N)
        res = np.linalg.norm(A @ delta + on["g"]) / np.linalg.norm(on["g"])
        assert res < 1e-5, res
        ref = np.linalg.solve(A, -on["g"])
        assert np.abs(delta - ref).max() <= 1e-2 * np.abs(ref).max()
        del A
        del Hg, on
        # device solve, then fusion on the shared post-solve state
        ctx.forward_warp()
        ctx.solve_nonrigid(pose, t, 0)
        ctx.forward_warp()
        L.sync_oracle(st, ctx)
        gfu = ctx.apply_fusion(pose, t)
        ofu = st.apply_fusion(pose, t)
        for k in FUSION_KEYS:
            assert getattr(gfu, k) == getattr(ofu, k), (t, k)
        gm, om = ctx.download_model(), st.get_model()
        assert len(gm["ref_pos"]) == len(om["ref_pos"])
        assert np.array_equal(gm["skin_idx"], om["skin_idx"])
        assert np.array_equal(gm["t_obs"], om["live_t_obs"])
        gn, onn = ctx.download_nodes(), st.get_nodes()
        assert np.array_equal(gn["pos"], onn["pos"]) and np.array_equal(gn["nbr"], onn["nbr"])
    ctx.close()


# ------------------------------------------------- directly against the reference
def _ref_or_skip():
    import ref_py as R

    if not R.available():
        pytest.skip("oracle/_ref (the compiled reference) not built")
    return R


def _as_sets_agree(a, b):
    return np.mean([set(x) == set(y) for x, y in zip(np.asarray(a), np.asarray(b))])


@pytest.mark.parametrize("name,scene,W,H,f", [("cfg1", "deforming_sphere", 320, 240, 280.0),
                                              ("cfg2", "articulated_body", 640, 480, 560.0)])
def test_initialisation_against_compiled_reference(name, scene, W, H, f):
    """Frame 0 on the device vs the UNMODIFIED reference (oracle/_ref,
    pipeline.cpp:42-72): the device stores surfels in fp32, the reference in
    fp64, so positions agree to fp32 rounding and the (d2, index) K-NN ties that
    rounding decides may order or pick differently; everything else exact.
    Measured (oracle fp32-mirror vs reference, which the device equals
    bit-exactly): cfg2 neighbour sets differ on 0.13 % of nodes, skinning sets
    on 0.02 % of surfels."""
    R = _ref_or_skip()
    cfg = pkg.camera_config(W, H, f, max_gn_iters=3)
    d0 = pkg.SyntheticSequence(scene, 2, cfg).render_depth(0)
    pipe = pkg.Pipeline(cfg)
    a = pipe.process_frame(d0, 0)
    rp = R.RefPipeline(O.make_config(**{k: v for k, v in cfg.items() if k in O.DEFAULTS}))
    b = rp.process_frame(d0, 0)
    for k in ("valid_pixels", "surfel_count", "node_count"):
        assert a[k] == b[k], k
    gn, rn = pipe.nodes(), rp.nodes()
    assert np.abs(np.asarray(gn["pos"]) - rn["pos"]).max() <= 1e-7  # fp32 surfel storage
    assert _as_sets_agree(gn["nbr"], rn["nbr"]) >= 0.995
    gm, rm = pipe.model(), rp.model()
    assert np.abs(np.asarray(gm["ref_pos"]) - rm["ref_pos"]).max() <= 1e-7
    assert np.array_equal(gm["skin_count"], rm["skin_count"])
    assert _as_sets_agree(np.asarray(gm["skin_idx"])[:, :4], rm["skin_idx"]) >= 0.999
    pipe.close()
    rp.close()


def test_cfg1_frames_against_compiled_reference():
    """BASELINE config 1, frames 0-3 through ds_process_frame (PCG run to
    convergence) and through the reference's own Pipeline::process_frame
    (dense LDLT), free-running: frame 0 exact; afterwards the fp32 device state
    and the fp64 reference may take a marginal append decision differently
    (measured: 1 surfel of 48k at frame 2, 3 of 2.8k appends at frame 3), so
    surfel / node counts within 0.1 %, appends within 0.5 %, poses within 1e-4
    (rotation entries) / 10 um, GN correspondences within 0.5 %."""
    R = _ref_or_skip()
    cfg = pkg.camera_config(320, 240, 280.0, max_gn_iters=3, **CONVERGED)
    seq = pkg.SyntheticSequence("deforming_sphere", 10, cfg)
    pipe = pkg.Pipeline(cfg)
    rp = R.RefPipeline(O.make_config(**{k: v for k, v in cfg.items() if k in O.DEFAULTS}))
    for t in range(4):
        d = seq.render_depth(t)
        a = pipe.process_frame(d, t)
        b = rp.process_frame(d, t)
        assert a["valid_pixels"] == b["valid_pixels"], t
        for k in ("surfel_count", "node_count", "appended"):
            if t == 0:
                assert a[k] == b[k], (t, k, a[k], b[k])
            else:
                tol = max(5, 5e-3 * b[k]) if k == "appended" else max(2, 1e-3 * b[k])
                assert abs(a[k] - b[k]) <= tol, (t, k, a[k], b[k])
        pr = np.concatenate([b["pose_R"].ravel(), b["pose_t"]])
        gap = np.abs(np.array(a["pose"]) - pr)
        # measured: frame 1 <= 1e-9; frame 2 2.5e-5 (rotation) / 0.6 um
        assert gap[:9].max() <= 1e-4 and gap[9:].max() <= 1e-5, (t, gap)
        if t > 0:
            assert abs(a["correspondences"] - b["solver_correspondences"]) <= 5e-3 * b["solver_correspondences"], t
            assert a["gn_iters"] == b["solver_iterations"], t
    pipe.close()
    rp.close()
