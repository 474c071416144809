"""Oracle pinned against proj/tests/test_raster.cpp and test_depth_processing.cpp."""
import math

import numpy as np

import harness as Hh
import oracle_py as O

pkg = __import__("paper_1904_13073_b200")


def ss(u, f):  # raster.hpp:39-41
    return int(math.floor(f * (u + 0.5)))


def live_state(surfels, cfg=None):
    st = O.OracleState(cfg or O.test_config())
    st.set_model(O.model_from_surfels(surfels))
    return st


def test_index_map_nearest_wins():  # test_raster.cpp:16-23
    st = live_state([O.make_surfel((0, 0, 2.0)), O.make_surfel((0, 0, 1.0))])
    idx, _ = st.render_index_map(O.pose_identity(), 4)
    assert idx[ss(59.5, 4), ss(79.5, 4)] == 1


def test_index_map_tie_lower_index():  # :25-30
    st = live_state([O.make_surfel((0, 0, 1.0)), O.make_surfel((0, 0, 1.0))])
    idx, _ = st.render_index_map(O.pose_identity(), 4)
    assert idx[ss(59.5, 4), ss(79.5, 4)] == 0


def test_index_map_behind_camera():  # :32-38
    st = live_state([O.make_surfel((0, 0, -1.0))])
    idx, _ = st.render_index_map(O.pose_identity(), 4)
    assert (idx == -1).all()


def test_index_map_unique_and_own_block():  # :40-79
    rng = np.random.default_rng(5)
    surf = [O.make_surfel(O.random_point(rng, 0.2) + [0, 0, 1.0]) for _ in range(500)]
    idx, _ = live_state(surf).render_index_map(O.pose_identity(), 4)
    v = idx[idx >= 0]
    assert len(v) == len(set(v.tolist())) <= 500
    rng = np.random.default_rng(7)
    surf = [O.make_surfel(O.random_point(rng, 0.25) + [0, 0, 1.2]) for _ in range(300)]
    idx, _ = live_state(surf).render_index_map(O.pose_identity(), 4)
    for sy, sx in zip(*np.nonzero(idx >= 0)):
        p = surf[idx[sy, sx]]["pos"]
        u, v_ = 140 * p[0] / p[2] + 79.5, 140 * p[1] / p[2] + 59.5
        assert sx // 4 == math.floor(u + 0.5) and sy // 4 == math.floor(v_ + 0.5)


def test_splat_covers_25_pixels():  # :81-99
    cfg = O.test_config(fx=570.0, fy=570.0, width=200, height=200, cx=100.0, cy=100.0)
    st = live_state([O.make_surfel((0, 0, 1.0), (0, 0, -1), 0.005, 20.0)], cfg)
    mm = st.render_model_maps(O.pose_identity(), 10, 0)
    assert mm["valid"].sum() == 25


def test_stability_gate_strict():  # :101-127
    s = O.make_surfel((0, 0, 1.0), (0, 0, -1), 0.004, 10.0)
    st = live_state([s])
    assert st.render_model_maps(O.pose_identity(), 50, 0)["valid"].sum() == 0
    s["conf"] = 10.001
    st = live_state([s])
    assert st.render_model_maps(O.pose_identity(), 50, 0)["valid"].sum() > 0


def test_recent_in_bootstrap_window():  # :129-140
    s = O.make_surfel((0, 0, 1.0), (0, 0, -1), 0.004, 1.0)
    s["t_obs"] = 11
    assert live_state([s]).render_model_maps(O.pose_identity(), 11, 10)["valid"].sum() > 0


def test_backfacing_culled():  # :142-149
    st = live_state([O.make_surfel((0, 0, 1.0), (0, 0, 1), 0.004, 20.0)])
    assert st.render_model_maps(O.pose_identity(), 50, 0)["valid"].sum() == 0


def test_point_and_splat_agree_on_tiny_splats():  # :151-170
    rng = np.random.default_rng(11)
    surf = [O.make_surfel(O.random_point(rng, 0.2) + [0, 0, 1.1], (0, 0, -1), 1e-5, 20.0)
            for _ in range(400)]
    st = live_state(surf)
    pts, _ = st.render_index_map(O.pose_identity(), 1)
    mm = st.render_model_maps(O.pose_identity(), 50, 0)
    both = (pts >= 0) & (mm["valid"] > 0)
    assert both.any()
    assert np.array_equal(pts[both], mm["idx"][both])


def test_model_maps_deterministic():  # :172-184
    rng = np.random.default_rng(13)
    surf = [O.make_surfel(O.random_point(rng, 0.2) + [0, 0, 1.0], (0, 0, -1), 0.01, 20.0)
            for _ in range(300)]
    st = live_state(surf)
    a = st.render_model_maps(O.pose_identity(), 50, 0)["idx"]
    b = st.render_model_maps(O.pose_identity(), 50, 0)["idx"]
    assert np.array_equal(a, b)


# ------------------------------------------------------------ depth processing
SMALL_K = dict(fx=120.0, fy=130.0, cx=31.5, cy=23.5, width=64, height=48)


def small_cfg(**kw):
    return O.make_config(**{**SMALL_K, **kw})


def test_backproject_principal_point():  # test_depth_processing.cpp:29-45
    cfg = small_cfg()
    d = np.zeros((48, 64), np.uint16)
    d[24, 32] = d[23, 31] = 1000
    st, v, vv = O.backproject(d, cfg)
    assert st == 0 and vv[23, 31]
    assert abs(v[23, 31, 2] - 1.0) < 1e-12
    assert abs(v[23, 31, 0] - (31 - 31.5) / 120.0) < 1e-12
    assert abs(v[23, 31, 1] - (23 - 23.5) / 130.0) < 1e-12


def test_backproject_unit_slope():  # :47-59
    cfg = small_cfg(cx=10.0, cy=20.0, fx=40.0, fy=40.0)
    d = np.zeros((48, 64), np.uint16)
    d[20, 50] = 2000
    _, v, vv = O.backproject(d, cfg)
    assert vv[20, 50] and np.linalg.norm(v[20, 50] - [2.0, 0.0, 2.0]) < 1e-12


def test_backproject_zero_and_range():  # :61-83
    cfg = small_cfg()
    _, _, vv = O.backproject(np.zeros((48, 64), np.uint16), cfg)
    assert not vv.any()
    d = np.zeros((48, 64), np.uint16)
    d[1, 1], d[2, 2], d[3, 3] = 50, 5500, 500
    _, _, vv = O.backproject(d, cfg)
    assert not vv[1, 1] and not vv[2, 2] and vv[3, 3]


def test_backproject_dimension_mismatch():  # :85-92
    st, _, _ = O.backproject(np.full((48, 65), 1000, np.uint16), small_cfg())
    assert st == 1


def test_projection_round_trip():  # :94-108
    cfg = small_cfg()
    _, v, vv = O.backproject(np.full((48, 64), 1234, np.uint16), cfg)
    assert vv.all()
    u = 120.0 * v[..., 0] / v[..., 2] + 31.5
    w = 130.0 * v[..., 1] / v[..., 2] + 23.5
    ys, xs = np.mgrid[0:48, 0:64]
    assert np.abs(u - xs).max() < 1e-4 and np.abs(w - ys).max() < 1e-4


def test_normals_fronto_parallel_and_facing():  # :110-167
    cfg = small_cfg()
    _, v, vv = O.backproject(np.full((48, 64), 1000, np.uint16), cfg)
    n, nv = O.estimate_normals(v, vv)
    assert nv[1:-1, 1:-1].all() and not nv[0, 0]
    assert np.abs(n[1:-1, 1:-1] - [0, 0, -1]).max() < 1e-9
    _, v8, vv8 = O.backproject(np.full((48, 64), 800, np.uint16), cfg)
    n8, _ = O.estimate_normals(v8, vv8)
    assert ((n8[1:-1, 1:-1] * v8[1:-1, 1:-1]).sum(-1) < 0).all()


def test_normals_tilted_plane():  # :124-150
    ys, xs = np.mgrid[0:48, 0:64]
    sx, sy = (xs - 31.5) / 120.0, (ys - 23.5) / 130.0
    z = 1.0 / (1.0 - sx)
    v = np.stack([z * sx, z * sy, z], -1)
    n, nv = O.estimate_normals(v, np.ones((48, 64), np.uint8))
    exp = np.array([1, 0, -1]) / math.sqrt(2)
    assert nv[1:-1, 1:-1].all()
    assert np.linalg.norm(n[1:-1, 1:-1] - exp, axis=-1).max() < 1e-3


def test_confidence_reference_values():  # :169-196
    cfg = O.make_config(fx=100.0, fy=100.0, width=201, height=201, cx=100.0, cy=100.0)
    assert abs(O.compute_confidence(100, 100, cfg) - 1.0) < 1e-15
    mr = math.hypot(100, 100)
    assert abs(O.compute_confidence(100 + 0.6 * mr, 100, cfg) - math.exp(-0.5)) < 1e-12
    assert abs(O.compute_confidence(0, 0, cfg) - math.exp(-1.0 / 0.72)) < 1e-12
    assert abs(O.compute_confidence(0, 0, cfg) - 0.24935) < 1e-5
    cs = small_cfg()
    prev = 2.0
    for step in range(20):
        c = O.compute_confidence(31.5 + step * 1.7, 23.5 + step * 0.9, cs)
        assert c <= prev + 1e-15
        prev = c


def test_radius_reference_values():  # :198-207
    assert abs(O.compute_radius(1.0, 570.0, -1.0) - 2.4810e-3) < 1e-6
    lim = O.compute_radius(1.0, 570.0, -math.cos(75 * math.pi / 180))
    assert abs(O.compute_radius(1.0, 570.0, -0.1) - lim) < 1e-15
    assert abs(O.compute_radius(2.0, 570.0, -1.0) - 2 * O.compute_radius(1.0, 570.0, -1.0)) < 1e-15


def test_frame_maps_sphere_interior_and_empty():  # :209-246
    cfg = O.test_config()
    seq = pkg.SyntheticSequence("rigid_orbit", 5, pkg.make_config(**{
        k: cfg[k] for k in ("fx", "fy", "cx", "cy", "width", "height")}))
    st = O.OracleState(cfg)
    st.build_frame(seq.render_depth(0), 0)
    f = st.get_frame()
    assert f["valid_count"] > 500
    va = f["valid"] > 0
    assert np.abs(np.linalg.norm(f["nrm"][va], axis=-1) - 1).max() < 1e-9
    assert (f["conf"][va] > 0).all() and (f["conf"][va] <= 1).all() and (f["radius"][va] > 0).all()
    st2 = O.OracleState(small_cfg())
    st2.build_frame(np.zeros((48, 64), np.uint16), 0)
    assert st2.get_frame()["valid_count"] == 0
    d = np.zeros((48, 64), np.uint16)
    d[20, 20] = 1500
    st2.build_frame(d, 0)
    f2 = st2.get_frame()
    assert f2["vertex_valid"][20, 20] and not f2["valid"][20, 20] and f2["valid_count"] == 0


def test_bilateral():  # :248-256
    d = np.full((48, 64), 1000, np.uint16)
    d[10, 10] = 1008
    d[0, 0] = 0
    o = O.bilateral_filter(d, 4.5, 30.0)
    assert o[0, 0] == 0 and abs(int(o[10, 10]) - 1000) < 8 and o[30, 30] == 1000
