"""Oracle pinned against proj/tests/test_solver.cpp, test_fusion.cpp, test_reinit.cpp."""
import math

import numpy as np
import pytest

import harness as Hh
import oracle_py as O

pkg = __import__("paper_1904_13073_b200")


def synth(name, frames, cfg):
    k = {key: cfg[key] for key in ("fx", "fy", "cx", "cy", "width", "height")}
    return pkg.SyntheticSequence(name, frames, pkg.make_config(**k))


# ------------------------------------------------------------------ solver
def random_rig(rng, n_nodes, n_surf):  # test_solver.cpp:29-62
    P = np.array([O.random_point(rng, 0.2) for _ in range(n_nodes)])
    dq = [O.dq_from_se3(O.random_se3(rng, 0.5, 0.1)) for _ in range(n_nodes)]
    nodes = O.make_nodes(P, dq=dq, sigma=0.05)
    st = O.OracleState(O.test_config())
    st.set_nodes(nodes)
    st.compute_node_edges(min(4, n_nodes - 1))
    idx = np.full((n_surf, 8), -1, np.int32)
    w = np.zeros((n_surf, 8))
    cnt = np.zeros(n_surf, np.int32)
    surf = []
    for i in range(n_surf):
        surf.append(O.make_surfel(O.random_point(rng, 0.25)))
        k = 1 + int(rng.integers(min(4, n_nodes)))
        ch = rng.choice(n_nodes, size=k, replace=False)
        idx[i, :k] = ch
        w[i, :k] = rng.uniform(0.05, 1.0, k)
        cnt[i] = k
    st.set_model(O.model_from_surfels(surf, idx, w, cnt))
    return st


def perturb(st, j, xi):
    nd = st.get_nodes()
    nd["dq"][j] = O.dq_mul(O.dq_increment(xi[:3], xi[3:]), nd["dq"][j])
    st.set_nodes(nd)


def test_blend_jacobian_scale_orthogonal():  # test_solver.cpp:70-84
    rng = np.random.default_rng(3)
    for _ in range(20):
        st = random_rig(rng, 6, 3)
        y, dydb, _ = st.blend_jacobian(0)
        m = st.get_model()
        nd = st.get_nodes()
        e = m["skin_idx"][0, :m["skin_count"][0]]
        w = m["skin_w"][0, :len(e)]
        piv = nd["dq"][e[0], :4]
        b = np.zeros(8)
        for j, ww in zip(e, w):
            s = -1.0 if piv @ nd["dq"][j, :4] < 0 else 1.0
            b += s * ww * nd["dq"][j]
        assert np.linalg.norm(dydb @ b) < 1e-9


def test_data_jacobian_vs_finite_differences():  # :86-120
    rng = np.random.default_rng(17)
    h = 1e-6
    for _ in range(10):
        st = random_rig(rng, 8, 10)
        m = st.get_model()
        for si in range(10):
            y, dydb, nj = st.blend_jacobian(si)
            for slot in range(m["skin_count"][si]):
                j = m["skin_idx"][si, slot]
                fd = np.zeros((3, 6))
                for col in range(6):
                    xi = np.zeros(6)
                    xi[col] = h
                    base = st.get_nodes()
                    perturb(st, j, xi)
                    yp = st.blend_jacobian(si)[0]
                    st.set_nodes(base)
                    xi[col] = -h
                    perturb(st, j, xi)
                    ym = st.blend_jacobian(si)[0]
                    st.set_nodes(base)
                    fd[:, col] = (yp - ym) / (2 * h)
                scale = max(1.0, np.abs(fd).max())
                assert np.abs(nj[slot] - fd).max() / scale < 1e-4


def test_reg_jacobian_vs_finite_differences():  # :122-160
    rng = np.random.default_rng(23)
    h = 1e-6
    for _ in range(10):
        dqj = O.dq_from_se3(O.random_se3(rng, 0.5, 0.1))
        dqi = O.dq_from_se3(O.random_se3(rng, 0.5, 0.1))
        pj = O.random_point(rng, 0.2)
        _, Jj, Ji = O.reg_terms(dqj, dqi, pj)
        for col in range(6):
            xi = np.zeros(6)
            xi[col] = h
            p = O.dq_mul(O.dq_increment(xi[:3], xi[3:]), dqj)
            m_ = O.dq_mul(O.dq_increment(-xi[:3], -xi[3:]), dqj)
            fd = (O.reg_terms(p, dqi, pj)[0] - O.reg_terms(m_, dqi, pj)[0]) / (2 * h)
            assert np.linalg.norm(Jj[:, col] - fd) / max(1, np.linalg.norm(fd)) < 1e-4
            p = O.dq_mul(O.dq_increment(xi[:3], xi[3:]), dqi)
            m_ = O.dq_mul(O.dq_increment(-xi[:3], -xi[3:]), dqi)
            fd = (O.reg_terms(dqj, p, pj)[0] - O.reg_terms(dqj, m_, pj)[0]) / (2 * h)
            assert np.linalg.norm(Ji[:, col] - fd) / max(1, np.linalg.norm(fd)) < 1e-4


def test_reg_energy_zero_iff_rigid():  # :162-176
    rng = np.random.default_rng(31)
    rig = O.random_se3(rng, 0.7, 0.2)
    st = O.OracleState(O.test_config())
    st.set_nodes(O.make_nodes([[0, 0, 0], [0.05, 0, 0]], dq=[O.dq_from_se3(rig)] * 2,
                              nbr=[[1], [0]]))
    assert abs(st.reg_energy()) < 1e-18
    st.set_nodes(O.make_nodes([[0, 0, 0], [0.05, 0, 0]],
                              dq=[O.dq_from_se3(rig),
                                  O.dq_from_se3(O.se3_mul(O.make_se3([0, 0, 0], [0.001, 0, 0]), rig))],
                              nbr=[[1], [0]]))
    assert st.reg_energy() > 1e-10


def test_normal_equations_check_rejects_asymmetry():  # :178-182
    h = np.eye(6)
    h[0, 1] = 0.5
    assert O.assert_normal_equations(h) == 3
    assert O.assert_normal_equations(np.eye(12)) == 0


@pytest.fixture(scope="module")
def orbit_scene():  # SolverSceneTest, test_solver.cpp:184-211
    cfg = O.test_config()
    seq = synth("rigid_orbit", 5, cfg)
    st = O.OracleState(cfg)
    st.build_frame(seq.render_depth(0), 0)
    fr = st.get_frame()
    st.set_model(O.model_from_surfels(Hh.surfels_from_frame(fr, 20.0)))
    st.init_warp_field()
    return cfg, seq, st, fr


def fresh(orbit_scene):
    cfg, seq, st0, fr = orbit_scene
    st = O.OracleState(cfg)
    st.set_model(st0.get_model())
    st.set_nodes(st0.get_nodes())
    st.set_frame(fr)
    return st, fr


def test_rigid_align_fixed_point(orbit_scene):  # :213-222
    st, _ = fresh(orbit_scene)
    I = O.pose_identity()
    r = st.rigid_align(I, I, 1, 0)
    assert not r.low_confidence and r.correspondences >= 100
    p = np.array(r.pose)
    assert np.abs(p[:9].reshape(3, 3) - np.eye(3)).max() < 1e-6 and np.linalg.norm(p[9:]) < 1e-6


def test_rigid_align_recovers_translation(orbit_scene):  # :224-238
    st, _ = fresh(orbit_scene)
    m = st.get_model()
    m["live_pos"] = m["live_pos"] + [0.005, 0, 0]
    st.set_model(m)
    I = O.pose_identity()
    r = st.rigid_align(I, I, 1, 0)
    p = np.array(r.pose)
    assert not r.low_confidence and np.linalg.norm(p[9:] - [0.005, 0, 0]) < 0.5e-3
    ang = math.acos(max(-1, min(1, (np.trace(p[:9].reshape(3, 3)) - 1) / 2)))
    assert ang < 0.2 * math.pi / 180


def test_rigid_align_insufficient(orbit_scene):  # :240-249
    st, _ = fresh(orbit_scene)
    st.build_frame(np.zeros((120, 160), np.uint16), 1)
    init = O.make_se3([0, 0.01, 0], [0.002, 0, 0])
    r = st.rigid_align(O.pose_identity(), init, 1, 0)
    assert r.low_confidence and np.abs(np.array(r.pose) - init).max() < 1e-15


def test_correspondences_cover_mutual_pixels(orbit_scene):  # :251-261
    st, fr = fresh(orbit_scene)
    mm = st.render_model_maps(O.pose_identity(), 1, 0)
    mutual = int(((fr["valid"] > 0) & (mm["valid"] > 0)).sum())
    pairs = st.find_correspondences(mm, O.pose_identity())
    assert len(pairs["surfel"]) == mutual > 500


def test_displaced_plane_no_pairs():  # :263-282
    cfg = O.test_config()
    seq = synth("static_plane", 2, cfg)
    st = O.OracleState(cfg)
    st.build_frame(seq.render_depth(0), 0)
    fr = st.get_frame()
    surf = Hh.surfels_from_frame(fr, 20.0)
    for s in surf:
        s["pos"] = s["pos"] + [0, 0, 0.10]
    st.set_model(O.model_from_surfels(surf))
    mm = st.render_model_maps(O.pose_identity(), 1, 0)
    assert len(st.find_correspondences(mm, O.pose_identity())["surfel"]) == 0


def test_normal_gate_splits_flipped_side(orbit_scene):  # :284-300
    st, fr = fresh(orbit_scene)
    mm = dict(idx=np.zeros((120, 160), np.int32), vert=fr["vert"], nrm=fr["nrm"].copy(),
              valid=fr["valid"])
    mm["nrm"][:, 80:] *= -1
    pairs = st.find_correspondences(mm, O.pose_identity())
    assert len(pairs["px"]) > 0 and (pairs["px"] < 80).all()
    bad = dict(mm)
    bad["valid"] = np.zeros((120, 161), np.uint8)
    bad["idx"] = np.zeros((120, 161), np.int32)
    bad["vert"] = np.zeros((120, 161, 3))
    bad["nrm"] = np.zeros((120, 161, 3))
    assert st.find_correspondences(bad, O.pose_identity()) == 1  # DimensionMismatch


def test_nonrigid_fixed_point(orbit_scene):  # :302-313
    st, _ = fresh(orbit_scene)
    before = st.get_nodes()["dq"]
    rep = st.solve_nonrigid(O.pose_identity(), 1, 0)
    assert rep.correspondences > 500 and abs(rep.initial_energy) < 1e-18
    assert rep.final_energy <= rep.initial_energy + 1e-18
    assert np.abs(st.get_nodes()["dq"] - before).max() < 1e-6


@pytest.mark.slow
def test_rigidity_limit_huge_lambda():  # :315-359
    cfg = O.test_config()
    seq = synth("static_plane", 2, cfg)
    st = O.OracleState(cfg)
    st.build_frame(seq.render_depth(0), 0)
    fr = st.get_frame()
    tilt = O.make_se3([0.8 * math.pi / 180, 0, 0], [0, 0, 0.003])
    surf = []
    for y in range(30, 90):
        for x in range(40, 120):
            if fr["valid"][y, x]:
                surf.append(O.make_surfel(O.se3_apply(tilt, fr["vert"][y, x]),
                                          O.pose_R(tilt) @ fr["nrm"][y, x], fr["radius"][y, x], 20.0))
    st.set_model(O.model_from_surfels(surf))
    st.init_warp_field()
    st.set_config(O.test_config(lambda_=1e6))
    rep = st.solve_nonrigid(O.pose_identity(), 1, 0)
    assert rep.iterations >= 1 and rep.final_energy <= rep.initial_energy
    dq = st.get_nodes()["dq"]
    worst = 0
    for a in range(len(dq)):
        d = np.abs(dq - dq[a]).sum(1)
        f = np.abs(dq + dq[a]).sum(1)
        worst = max(worst, np.minimum(d, f).max())
    assert worst < 1e-3


def test_tracks_small_deformation(orbit_scene):  # :361-374
    st, fr = fresh(orbit_scene)
    sh = dict(fr)
    sh["vert"] = fr["vert"].copy()
    sh["vert"][fr["valid"] > 0, 2] += 0.002
    st.set_frame(sh, 1)
    rep = st.solve_nonrigid(O.pose_identity(), 1, 0)
    assert 1 <= rep.iterations <= 10 and rep.final_energy < rep.initial_energy
    assert rep.mean_residual < 1e-3


# ------------------------------------------------------------------ fusion
CENT = dict(fx=140.0, fy=140.0, width=64, height=48, cx=32.0, cy=24.0)


def const_frame(st, mm, fi=0):
    st.build_frame(np.full((48, 64), mm, np.uint16), fi)
    return st.get_frame()


def test_fuse_hand_case():  # test_fusion.cpp:34-62
    st = O.OracleState(O.make_config(**CENT, delta_distance=0.02))
    fr = const_frame(st, 1011, 3)
    assert fr["valid"][24, 32] and abs(fr["conf"][24, 32] - 1.0) < 1e-12
    st.set_model(O.model_from_surfels([O.make_surfel((0, 0, 1.0), (0, 0, -1), 0.004, 10.0)]))
    idx, _ = st.render_index_map(O.pose_identity(), 4)
    fused, cands = st.fuse_depth(idx, 4, O.pose_identity(), 3)
    m = st.get_model()
    assert fused == 1 and abs(m["live_conf"][0] - 11.0) < 1e-12
    assert abs(m["live_pos"][0, 2] - 1.001) < 1e-9 and abs(m["live_pos"][0, 0]) < 1e-12
    assert m["live_t_obs"][0] == 3 and len(cands["px"]) == fr["valid_count"] - 1


def test_fuse_distance_gate_candidate():  # :64-85
    st = O.OracleState(O.make_config(**CENT))
    const_frame(st, 1000, 1)
    st.set_model(O.model_from_surfels([O.make_surfel((0, 0, 1.002), (0, 0, -1), 0.004, 5.0)]))
    idx, _ = st.render_index_map(O.pose_identity(), 4)
    fused, c = st.fuse_depth(idx, 4, O.pose_identity(), 1)
    assert fused == 0 and st.get_model()["live_conf"][0] == 5.0
    assert any(x == 32 and y == 24 for x, y in zip(c["px"], c["py"]))


def test_fuse_highest_confidence_wins():  # :87-112
    st = O.OracleState(O.make_config(**{**CENT, "fx": 570.0, "fy": 570.0}))
    const_frame(st, 1000, 2)
    st.set_model(O.model_from_surfels([O.make_surfel((-0.0004, 0, 1.0), (0, 0, -1), 0.004, 5.0),
                                       O.make_surfel((0.0004, 0, 1.0), (0, 0, -1), 0.004, 9.0)]))
    idx, _ = st.render_index_map(O.pose_identity(), 4)
    fused, _ = st.fuse_depth(idx, 4, O.pose_identity(), 2)
    m = st.get_model()
    assert fused >= 1 and m["live_conf"][1] > 9.0 and m["live_conf"][0] == 5.0


def test_skin_appended_rigid_keeps_all():  # :114-131
    rng = np.random.default_rng(5)
    rig = O.random_se3(rng, 0.6, 0.15)
    P = np.array([O.random_point(rng, 0.05) for _ in range(6)])
    st = O.OracleState(O.test_config())
    st.set_nodes(O.make_nodes(P, dq=[O.dq_from_se3(rig)] * 6))
    nl = np.array([O.se3_apply(rig, p) for p in P])
    idx, w = st.skin_appended(O.se3_apply(rig, [0.01, 0.005, 0.0]), nl)
    assert len(idx) == 4


def test_skin_appended_inconsistent_removed():  # :133-152
    st = O.OracleState(O.test_config())
    st.set_nodes(O.make_nodes([[0, 0, 0], [0.02, 0, 0], [0.30, 0, 0]],
                              dq=[O.IDENTITY_DQ, O.IDENTITY_DQ,
                                  O.dq_from_se3(O.make_se3([0, 0, 0], [-0.27, 0, 0]))]))
    nl = np.array([[0, 0, 0], [0.02, 0, 0], [0.03, 0, 0]])
    idx, w = st.skin_appended([0.005, 0.002, 0], nl)
    assert 2 not in idx and len(idx) == 2


def test_skin_appended_far_rejected():  # :154-165
    st = O.OracleState(O.test_config())
    P = np.array([[0.01 * j, 0, 0] for j in range(4)])
    st.set_nodes(O.make_nodes(P))
    assert st.skin_appended([1.0, 1.0, 1.0], P) is None


def axis_rig(sigma, off, tr):  # :175-192
    st = O.OracleState(O.test_config())
    nodes = O.make_nodes([[-(off + tr), 0, 0], [off + tr, 0, 0]], sigma=sigma,
                         dq=[O.dq_from_se3(O.make_se3([0, 0, 0], [tr, 0, 0])),
                             O.dq_from_se3(O.make_se3([0, 0, 0], [-tr, 0, 0]))])
    st.set_nodes(nodes)
    nl = np.array([O.dq_apply(nodes["dq"][j], nodes["pos"][j]) for j in range(2)])
    w = [O.skinning_weight([0, 0, 0], nl[j], sigma) for j in range(2)]
    return st, nl, [0, 1], w


def test_compressive_identity_kept():  # :194-202
    st, nl, idx, w = axis_rig(0.025, 0.025, 0.0)
    assert st.check_compressive([0, 0, 0], idx, w, nl)
    assert np.abs(st.inverse_warp_strain([0, 0, 0], idx, w, nl) - np.eye(3)).max() < 1e-9


def test_compressive_half_scale_discarded():  # :204-215
    st, nl, idx, w = axis_rig(0.025, 0.025, 0.025)
    s = st.inverse_warp_strain([0, 0, 0], idx, w, nl)
    assert abs(s[0, 0] - 2.0) < 5e-3 and not st.check_compressive([0, 0, 0], idx, w, nl)


def test_compressive_pure_rotation_kept():  # :217-238
    rng = np.random.default_rng(11)
    rot = O.make_se3([0.3, -0.2, 0.5], [0, 0, 0])
    P = np.array([O.random_point(rng, 0.03) for _ in range(3)])
    st = O.OracleState(O.test_config())
    st.set_nodes(O.make_nodes(P, dq=[O.dq_from_se3(rot)] * 3))
    nl = np.array([O.se3_apply(rot, p) for p in P])
    w = [0.3 + 0.2 * j for j in range(3)]
    s = st.inverse_warp_strain([0.01, 0, 0.01], [0, 1, 2], w, nl)
    assert abs(np.linalg.svd(s, compute_uv=False)[0] - 1.0) < 1e-6
    assert st.check_compressive([0.01, 0, 0.01], [0, 1, 2], w, nl)


def test_remove_surfels_rules():  # :240-272
    st = O.OracleState(O.make_config(**CENT))
    st.set_model(O.model_from_surfels([O.make_surfel((0, 0, 1.0), (0, 0, -1), 0.004, 9.0, 0),
                                       O.make_surfel((0.05, 0, 1.0), (0, 0, -1), 0.004, 11.0, 0)]))
    idx, _ = st.render_index_map(O.pose_identity(), 4)
    assert list(st.remove_surfels(idx, 4, O.pose_identity(), 31)) == [1, 0]
    st.set_model(O.model_from_surfels([O.make_surfel((0, 0, 1.0), (0, 0, -1), 0.004, 15.0, 0),
                                       O.make_surfel((0.0002, 0, 1.0), (0, 0, -1), 0.004, 12.0, 0)]))
    idx, _ = st.render_index_map(O.pose_identity(), 4)
    assert list(st.remove_surfels(idx, 4, O.pose_identity(), 5)) == [0, 1]


def plane_fusion_state(x1):  # ApplyFusionTest, :274-305
    cfg = O.test_config()
    seq = synth("static_plane", 3, cfg)
    st = O.OracleState(cfg)
    st.build_frame(seq.render_depth(1), 1)
    fr = st.get_frame()
    st.set_model(O.model_from_surfels(Hh.surfels_from_frame(fr, None, 0, (0, x1))))
    st.init_warp_field()
    return st, fr


def test_refeed_fuses_everything():  # :307-327
    st, fr = plane_fusion_state(160)
    n0 = st.size()
    before = st.get_model()["live_conf"].copy()
    oc = st.apply_fusion(O.pose_identity(), 1)
    m = st.get_model()
    assert oc.appended == 0 and oc.fused == fr["valid_count"] and oc.removed == 0
    assert st.size() == n0 and (m["live_conf"] >= before).all() and (m["live_t_obs"] == 1).all()
    assert np.array_equal(m["live_conf"], m["ref_conf"])


def test_new_region_appends():  # :329-344
    st, fr = plane_fusion_state(80)
    oc = st.apply_fusion(O.pose_identity(), 1)
    assert oc.appended > 0 and oc.new_nodes > 0
    assert oc.appended + oc.low_support_rejected + oc.compressive_rejected == \
        fr["valid_count"] - oc.fused
    assert (st.get_model()["live_t_init"] == 1).sum() == oc.appended


def test_exact_refeed_in_place_and_convex():  # :346-374
    st, fr = plane_fusion_state(160)
    before = st.get_model()
    st.apply_fusion(O.pose_identity(), 1)
    m = st.get_model()
    assert np.abs(m["live_pos"] - before["live_pos"]).max() < 1e-9
    assert np.abs(m["live_radius"] - before["live_radius"]).max() < 1e-12
    st2, fr2 = plane_fusion_state(160)
    st2.set_config(O.test_config(delta_distance=0.02))
    sh = dict(fr2)
    sh["vert"] = fr2["vert"].copy()
    sh["vert"][fr2["valid"] > 0, 2] += 0.004
    st2.set_frame(sh, 1)
    b2 = st2.get_model()
    st2.apply_fusion(O.pose_identity(), 1)
    z = st2.get_model()["live_pos"][:len(b2["live_pos"]), 2]
    assert (z >= b2["live_pos"][:, 2] - 1e-12).all() and (z <= b2["live_pos"][:, 2] + 0.004 + 1e-9).all()


def test_fusion_deterministic():  # :376-400
    a, _ = plane_fusion_state(80)
    b, _ = plane_fusion_state(80)
    oa, ob = a.apply_fusion(O.pose_identity(), 1), b.apply_fusion(O.pose_identity(), 1)
    assert (oa.fused, oa.appended, oa.removed) == (ob.fused, ob.appended, ob.removed)
    assert np.array_equal(a.get_model()["live_pos"], b.get_model()["live_pos"])


# ------------------------------------------------------------------ reinit
def test_should_reinitialize():  # test_reinit.cpp:25-63
    cfg = O.test_config()
    assert not O.should_reinitialize([0.0] * 3, [0] * 3, 10, 0, cfg)
    assert O.should_reinitialize([0.010] * 3, [8000] * 3, 10, 0, cfg)
    assert not O.should_reinitialize([0.010] * 2, [8000] * 2, 10, 0, cfg)
    assert not O.should_reinitialize([0.010, 0.001, 0.010], [8000] * 3, 10, 0, cfg)
    c5 = O.test_config(periodic_reinit_interval=5)
    assert not O.should_reinitialize([0.0] * 3, [0] * 3, 9, 5, c5)
    assert O.should_reinitialize([0.0] * 3, [0] * 3, 10, 5, c5)


def clean_state(extra):
    cfg = O.test_config()
    seq = synth("static_plane", 2, cfg)
    st = O.OracleState(cfg)
    st.build_frame(seq.render_depth(0), 0)
    surf = Hh.surfels_from_frame(st.get_frame(), 15.0) + extra
    st.set_model(O.model_from_surfels(surf))
    return st, len(surf) - len(extra)


def test_clean_and_reset_cases():  # :97-191
    st, n = clean_state([])
    code, rem, surv = st.clean_and_reset(O.pose_identity())
    m = st.get_model()
    assert code == 0 and rem == 0 and surv == n and np.array_equal(m["ref_pos"], m["live_pos"])
    for dq in st.get_nodes()["dq"]:
        assert np.abs(dq - O.IDENTITY_DQ).max() < 1e-12
    st, n = clean_state([O.make_surfel((0, 0, 0.9), (0, 0, -1), 0.004, 15.0),
                         O.make_surfel((0, 0, 1.1), (0, 0, -1), 0.004, 15.0)])
    code, rem, surv = st.clean_and_reset(O.pose_identity())
    assert rem == 1 and surv == n + 1
    st, n = clean_state([O.make_surfel((0.02, 0, 0.9), (0, 0, 1), 0.004, 15.0),
                         O.make_surfel((5.0, 0, 1.0), (0, 0, -1), 0.004, 15.0),
                         O.make_surfel((0, 0, -0.5), (0, 0, -1), 0.004, 15.0)])
    code, rem, surv = st.clean_and_reset(O.pose_identity())
    assert rem == 0 and surv == n + 3
    st = O.OracleState(O.test_config())
    seq = synth("static_plane", 2, O.test_config())
    st.build_frame(seq.render_depth(0), 0)
    st.set_model(O.model_from_surfels([O.make_surfel((0.01 * i - 0.1, 0, 0.8), (0, 0, -1),
                                                     0.004, 15.0) for i in range(20)]))
    assert st.clean_and_reset(O.pose_identity())[0] == 2  # EmptyGeometry


def test_oracle_pipeline_runs_and_mirror_is_close():
    cfg = O.test_config()
    seq = synth("articulated_two_part", 60, cfg)
    a, b = O.OraclePipeline(cfg), O.OraclePipeline(cfg, mirror=True)
    for t in range(3):
        d = seq.render_depth(t)
        sa, sb = a.process_frame(d, t), b.process_frame(d, t)
        assert sa.valid_pixels == sb.valid_pixels
        if t:
            assert sa.solver.correspondences > 100
            assert abs(sa.surfel_count - sb.surfel_count) <= 0.01 * sa.surfel_count + 2
