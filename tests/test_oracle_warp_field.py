"""Oracle pinned against proj/tests/test_warp_field.cpp known answers."""
import numpy as np
import pytest

import oracle_py as O


def cfg_sigma(s):
    return O.test_config(node_sigma=s)


def cube_grid(extent, step):  # :25-32
    out = []
    n = int(round(extent / step)) + 1
    for z in range(n):
        for y in range(n):
            for x in range(n):
                out.append(O.make_surfel((x * step, y * step, z * step)))
    return out


def state_with(surfels, sigma):
    st = O.OracleState(cfg_sigma(sigma))
    st.set_model(O.model_from_surfels(surfels))
    return st


def test_voxel_knn_matches_brute_force():  # :41-60
    rng = np.random.default_rng(101)
    for _ in range(30):
        n = 1 + int(rng.integers(200))
        pts = np.array([O.random_point(rng, 0.15) for _ in range(n)])
        for _ in range(20):
            q = O.random_point(rng, 0.2)
            k = 1 + int(rng.integers(6))
            assert O.voxel_knn(pts, 0.025, q, k) == O.brute_force_knn(q, pts, k)


def test_nodes_respect_sampling_distance():  # :62-77
    st = state_with(cube_grid(0.10, 0.01), 0.025)
    assert st.init_warp_field() == 0
    nd = st.get_nodes()
    P = nd["pos"]
    assert len(P) > 10
    D = np.linalg.norm(P[:, None] - P[None], axis=-1) + np.eye(len(P)) * 9
    assert D.min() >= 0.025 - 1e-12
    assert np.all(nd["sigma"] == 0.025)
    for dq in nd["dq"]:
        p = O.dq_to_se3(dq)
        assert np.abs(O.pose_R(p) - np.eye(3)).max() < 1e-12 and np.linalg.norm(O.pose_t(p)) < 1e-12
    assert st.size() == len(cube_grid(0.10, 0.01))


def test_single_surfel_skins_to_itself():  # :79-88
    st = state_with([O.make_surfel((0.1, 0.2, 0.9))], 0.025)
    st.init_warp_field()
    nd, m = st.get_nodes(), st.get_model()
    assert len(nd["pos"]) == 1 and np.linalg.norm(nd["pos"][0] - [0.1, 0.2, 0.9]) < 1e-15
    assert m["skin_count"][0] == 1 and m["skin_idx"][0, 0] == 0
    assert abs(m["skin_w"][0, 0] - 1.0) < 1e-12


def test_empty_input_throws():  # :90-92
    st = state_with([], 0.025)
    assert st.init_warp_field() == 2  # EmptyGeometry


def test_skinning_matches_brute_force():  # :94-113
    rng = np.random.default_rng(211)
    surf = [O.make_surfel(O.random_point(rng, 0.2) + [0, 0, 1.0]) for _ in range(400)]
    st = state_with(surf, 0.025)
    st.init_warp_field()
    P = st.get_nodes()["pos"]
    m = st.get_model()
    for i, s in enumerate(surf):
        exp = O.brute_force_knn(s["pos"], P, 4)
        assert m["skin_count"][i] == len(exp)
        assert list(m["skin_idx"][i, :len(exp)]) == exp
        for k, j in enumerate(exp):
            assert abs(m["skin_w"][i, k] - O.skinning_weight(s["pos"], P[j], 0.025)) < 1e-15


def _with_field(st, fn):
    nd = st.get_nodes()
    for j in range(len(nd["pos"])):
        nd["dq"][j] = fn(j)
    st.set_nodes(nd)
    return nd


def test_forward_warp_identity():  # :115-127
    st = state_with(cube_grid(0.05, 0.01), 0.02)
    st.init_warp_field()
    assert st.forward_warp() == 0
    m = st.get_model()
    assert np.abs(m["live_pos"] - m["ref_pos"]).max() < 1e-12
    assert np.abs(m["live_nrm"] - m["ref_nrm"]).max() < 1e-12


def test_forward_warp_uniform_rigid():  # :129-145
    rng = np.random.default_rng(307)
    rig = O.random_se3(rng, 0.8, 0.3)
    st = state_with(cube_grid(0.05, 0.01), 0.02)
    st.init_warp_field()
    _with_field(st, lambda j: O.dq_from_se3(rig))
    st.forward_warp()
    m = st.get_model()
    for i in range(len(m["ref_pos"])):
        assert np.linalg.norm(m["live_pos"][i] - O.se3_apply(rig, m["ref_pos"][i])) < 1e-9
        assert np.linalg.norm(m["live_nrm"][i] - O.pose_R(rig) @ m["ref_nrm"][i]) < 1e-9


def test_forward_warp_midpoint_of_two_translations():  # :147-167
    st = O.OracleState(O.test_config())
    t1, t2 = np.array([0.01, 0, 0]), np.array([0, 0.02, 0])
    nodes = O.make_nodes([[-0.02, 0, 0], [0.02, 0, 0]],
                         dq=[O.dq_from_se3(O.make_se3([0, 0, 0], t1)),
                             O.dq_from_se3(O.make_se3([0, 0, 0], t2))])
    w = [O.skinning_weight([0, 0, 0], p, 0.025) for p in nodes["pos"]]
    idx = np.full((1, 8), -1)
    idx[0, :2] = [0, 1]
    ww = np.zeros((1, 8))
    ww[0, :2] = w
    st.set_model(O.model_from_surfels([O.make_surfel((0, 0, 0))], idx, ww, [2]))
    st.set_nodes(nodes)
    st.forward_warp()
    assert np.linalg.norm(st.get_model()["live_pos"][0] - 0.5 * (t1 + t2)) < 1e-12


def test_forward_warp_preserves_shared_attributes():  # :169-193
    rng = np.random.default_rng(401)
    surf = []
    for i in range(50):
        s = O.make_surfel(O.random_point(rng, 0.1), (0, 0, -1), 0.003 + 0.001 * i, 0.5 * i, i)
        s["t_obs"] = i + 3
        surf.append(s)
    st = state_with(surf, 0.02)
    st.init_warp_field()
    rng2 = np.random.default_rng(402)
    _with_field(st, lambda j: O.dq_from_se3(O.random_se3(rng2, 0.3, 0.05)))
    st.forward_warp()
    m = st.get_model()
    for k in ("radius", "conf", "t_init", "t_obs"):
        assert np.array_equal(m["live_" + k], m["ref_" + k])


def test_inverse_warp_round_trip():  # :195-213
    rng = np.random.default_rng(499)
    st = state_with([O.make_surfel(O.random_point(rng, 0.15)) for _ in range(200)], 0.025)
    st.init_warp_field()
    _with_field(st, lambda j: O.dq_from_se3(O.random_se3(rng, 0.4, 0.08)))
    st.forward_warp()
    m = st.get_model()
    for i in range(200):
        p, n = st.inverse_warp_surfel(i)
        assert np.linalg.norm(p - m["ref_pos"][i]) < 1e-9 and np.linalg.norm(n - m["ref_nrm"][i]) < 1e-9


def test_inverse_warp_single_node_exact():  # :215-232
    rng = np.random.default_rng(503)
    tr = O.random_se3(rng, 0.9, 0.2)
    st = O.OracleState(O.test_config())
    idx = np.full((1, 8), -1)
    idx[0, 0] = 0
    w = np.zeros((1, 8))
    w[0, 0] = 0.4
    m = O.model_from_surfels([O.make_surfel((0.05, -0.02, 0.01), (0, 1, 0))], idx, w, [1])
    st.set_model(m)
    st.set_nodes(O.make_nodes([[0.01, 0.02, 0.03]], dq=[O.dq_from_se3(tr)]))
    p, n = st.inverse_warp_surfel(0)
    inv = O.se3_inverse(tr)
    assert np.linalg.norm(p - O.se3_apply(inv, [0.05, -0.02, 0.01])) < 1e-12
    assert np.linalg.norm(n - O.pose_R(inv) @ [0, 1, 0]) < 1e-12


def test_warp_locality_bit_identical():  # :248-270
    rng = np.random.default_rng(601)
    surf = [O.make_surfel(O.random_point(rng, 0.1)) for _ in range(100)]
    surf.append(O.make_surfel((2.0, 2.0, 2.0)))
    st = state_with(surf, 0.025)
    st.init_warp_field()
    st.forward_warp()
    before = st.get_model()["live_pos"][0].copy()
    nd = st.get_nodes()
    nd["dq"][-1] = O.dq_from_se3(O.make_se3([0.1, 0.2, 0.3], [1, 2, 3]))
    st.set_nodes(nd)
    st.forward_warp()
    assert np.array_equal(st.get_model()["live_pos"][0], before)


def test_extend_covered_adds_nothing():  # :272-278
    surf = cube_grid(0.05, 0.01)
    st = state_with(surf, 0.025)
    st.init_warp_field()
    n0 = st.num_nodes()
    assert st.extend_warp_field([s["pos"] for s in surf]) == 0 and st.num_nodes() == n0


def test_extend_isolated_becomes_identity_node():  # :280-296
    st = state_with(cube_grid(0.05, 0.01), 0.025)
    st.init_warp_field()
    n0 = st.num_nodes()
    assert st.extend_warp_field([[1.0, 1.0, 1.0]]) == 1
    nd = st.get_nodes()
    assert len(nd["pos"]) == n0 + 1 and np.linalg.norm(nd["pos"][-1] - 1.0) < 1e-15
    p = O.dq_to_se3(nd["dq"][-1])
    assert np.abs(O.pose_R(p) - np.eye(3)).max() < 1e-12 and np.linalg.norm(O.pose_t(p)) < 1e-12
    assert np.all(nd["nbr_count"] == min(8, len(nd["pos"]) - 1))


def test_extend_spacing_invariant():  # :298-314
    rng = np.random.default_rng(701)
    st = state_with([O.make_surfel(O.random_point(rng, 0.1)) for _ in range(300)], 0.025)
    st.init_warp_field()
    st.extend_warp_field([O.random_point(rng, 0.1) + [0.18, 0, 0] for _ in range(200)])
    P = st.get_nodes()["pos"]
    D = np.linalg.norm(P[:, None] - P[None], axis=-1) + np.eye(len(P)) * 9
    assert D.min() >= 0.025 - 1e-12


def test_extend_new_node_transform_matches_blend_oracle():  # :316-342
    rng = np.random.default_rng(809)
    st = state_with([O.make_surfel(O.random_point(rng, 0.08)) for _ in range(150)], 0.025)
    st.init_warp_field()
    before = _with_field(st, lambda j: O.dq_from_se3(O.random_se3(rng, 0.3, 0.05)))
    probe = np.array([0.08, 0.08, 0.08]) + [0.03, 0.02, 0.025]
    assert st.extend_warp_field([probe]) == 1
    idx = O.brute_force_knn(probe, before["pos"], 4)
    exp = O.blend([before["dq"][j] for j in idx],
                  [O.skinning_weight(probe, before["pos"][j], 0.025) for j in idx])
    got = st.get_nodes()["dq"][-1]
    s = -1.0 if exp[:4] @ got[:4] < 0 else 1.0
    assert np.linalg.norm(s * got[:4] - exp[:4]) < 1e-12
    assert np.linalg.norm(s * got[4:] - exp[4:]) < 1e-12


def test_incremental_no_new_nodes_noop():  # :344-359
    rng = np.random.default_rng(901)
    st = state_with([O.make_surfel(O.random_point(rng, 0.08)) for _ in range(60)], 0.025)
    st.init_warp_field()
    before = st.get_model()
    st.update_skinning_incremental(st.num_nodes())
    after = st.get_model()
    for k in ("skin_idx", "skin_w", "skin_count"):
        assert np.array_equal(before[k], after[k])


def test_incremental_node_at_surfel_enters():  # :361-384
    rng = np.random.default_rng(907)
    surf = [O.make_surfel(O.random_point(rng, 0.08)) for _ in range(60)]
    st = state_with(surf, 0.025)
    st.init_warp_field()
    nd = st.get_nodes()
    first = len(nd["pos"])
    nd2 = O.make_nodes(np.vstack([nd["pos"], surf[7]["pos"]]),
                       dq=np.vstack([nd["dq"], O.IDENTITY_DQ]))
    nd2["nbr"][:first] = nd["nbr"]
    nd2["nbr_count"][:first] = nd["nbr_count"]
    st.set_nodes(nd2)
    st.update_skinning_incremental(first)
    m = st.get_model()
    row = list(m["skin_idx"][7, :m["skin_count"][7]])
    assert first in row
    assert abs(m["skin_w"][7, row.index(first)] - 1.0) < 1e-12


def test_incremental_matches_brute_force():  # :386-430
    rng = np.random.default_rng(911)
    cfg = cfg_sigma(0.025)
    for _ in range(20):
        surf = [O.make_surfel(O.random_point(rng, 0.1)) for _ in range(100)]
        P = np.array([O.random_point(rng, 0.12) for _ in range(25)])
        idx = np.full((100, 8), -1, np.int32)
        w = np.zeros((100, 8))
        cnt = np.zeros(100, np.int32)
        for i, s in enumerate(surf):
            e = O.brute_force_knn(s["pos"], P[:20], 4)
            idx[i, :len(e)] = e
            w[i, :len(e)] = [O.skinning_weight(s["pos"], P[j], 0.025) for j in e]
            cnt[i] = len(e)
        st = O.OracleState(cfg)
        st.set_model(O.model_from_surfels(surf, idx, w, cnt))
        st.set_nodes(O.make_nodes(P))
        st.update_skinning_incremental(20)
        m = st.get_model()
        for i, s in enumerate(surf):
            e = O.brute_force_knn(s["pos"], P, 4)
            assert m["skin_count"][i] == len(e)
            assert list(m["skin_idx"][i, :len(e)]) == e
            for k, j in enumerate(e):
                assert abs(m["skin_w"][i, k] - O.skinning_weight(s["pos"], P[j], 0.025)) < 1e-15


@pytest.mark.parametrize("k", [1, 4, 8])
def test_node_edges_match_brute_force(k):
    rng = np.random.default_rng(k)
    P = np.array([O.random_point(rng, 0.2) for _ in range(60)])
    st = O.OracleState(O.test_config())
    st.set_nodes(O.make_nodes(P))
    st.compute_node_edges(k)
    nd = st.get_nodes()
    for j in range(60):
        others = [i for i in range(60) if i != j]
        exp = [others[i] for i in O.brute_force_knn(P[j], P[others], k)]
        assert list(nd["nbr"][j, :nd["nbr_count"][j]]) == exp
