"""Stage-level parity: CUDA path vs the CPU oracle on identical (fp32-rounded) inputs.

Discrete outputs (valid masks, node sets, edges, KNN/skinning indices, z-buffer
winners, correspondence pairs, JtJ block pattern) must match bit-exactly;
continuous ones within the fp32 storage tolerance stated per test.
"""
import numpy as np
import pytest

import harness as Hh
import oracle_py as O

pytestmark = pytest.mark.gpu

pkg = pytest.importorskip("paper_1904_13073_b200")

SMALL = dict(fx=140.0, fy=140.0, cx=79.5, cy=59.5, width=160, height=120)


def scene(name="rigid_orbit", frames=5, **kw):
    cfg = pkg.make_config(**{**SMALL, **kw})
    return cfg, pkg.SyntheticSequence(name, frames, cfg)


def frame_model(cfg, depth, conf=20.0, x_range=None, mutate=None):
    st = O.OracleState(Hh.oracle_cfg(cfg))
    st.build_frame(depth, 0)
    fr = st.get_frame()
    surf = Hh.surfels_from_frame(fr, confidence=conf, x_range=x_range)
    if mutate:
        for s in surf:
            mutate(s)
    return O.model_from_surfels(surf), st


@pytest.fixture(scope="module")
def ctx_small():
    cfg, _ = scene()
    c = pkg.Context(cfg)
    yield c
    c.close()


def test_frame_maps_bit_exact():
    for name in ("rigid_orbit", "static_plane", "bending_sheet"):
        cfg, seq = scene(name, 20)
        ctx = pkg.Context(cfg)
        for t in (0, 7):
            d = seq.render_depth(t)
            vc = ctx.frame_maps(d, t)
            g = ctx.download_frame()
            st = O.OracleState(Hh.oracle_cfg(cfg))
            st.build_frame(d, t)
            o = st.get_frame()
            assert vc == o["valid_count"]
            assert np.array_equal(g["valid"], o["valid"])
            assert np.array_equal(g["vertex_valid"], o["vertex_valid"])
            assert np.array_equal(g["vert"], o["vert"])  # same fp64 expression
            assert np.abs(g["nrm"] - o["nrm"]).max() == 0.0
            assert np.abs(g["radius"] - o["radius"]).max() == 0.0
            assert np.abs(g["conf"] - o["conf"]).max() < 1e-15  # exp/hypot ulps
        ctx.close()


def test_frame_maps_dimension_mismatch(ctx_small):
    with pytest.raises(pkg.DimensionMismatch):
        ctx_small.frame_maps(np.zeros((120, 161), np.uint16))


def _init_both(cfg, model):
    ctx = pkg.Context(cfg)
    rm, _ = Hh.round_trip(ctx, model)
    ctx.init_warp_field()
    st = O.OracleState(Hh.oracle_cfg(cfg))
    st.set_model(rm)
    assert st.init_warp_field() == 0
    return ctx, st


def test_init_warp_field_bit_exact():
    cfg, seq = scene()
    model, _ = frame_model(cfg, seq.render_depth(0))
    ctx, st = _init_both(cfg, model)
    gn, on = ctx.download_nodes(), st.get_nodes()
    assert len(gn["pos"]) == len(on["pos"]) > 10
    assert np.array_equal(gn["pos"], on["pos"])
    assert np.array_equal(gn["nbr"], on["nbr"])
    assert np.array_equal(gn["nbr_count"], on["nbr_count"])
    gm, om = ctx.download_model(), st.get_model()
    assert np.array_equal(gm["skin_count"], om["skin_count"])
    assert np.array_equal(gm["skin_idx"], om["skin_idx"])
    # fp32 weight storage: relative 2^-24
    assert np.allclose(gm["skin_w"], om["skin_w"], rtol=1.2e-7, atol=1e-30)
    ctx.close()


def test_init_warp_field_empty_raises(ctx_small):
    ctx_small.upload_model(Hh.oracle_to_device_model(O.model_from_surfels([])))
    with pytest.raises(pkg.EmptyGeometry):
        ctx_small.init_warp_field()


def _random_field(ctx, st, rng, angle=0.3, shift=0.05):
    nd = st.get_nodes()
    for j in range(len(nd["pos"])):
        nd["dq"][j] = O.dq_from_se3(O.random_se3(rng, angle, shift))
    ctx.upload_nodes(nd)
    st.set_nodes(nd)
    return nd


def test_forward_warp_matches():
    cfg, seq = scene()
    model, _ = frame_model(cfg, seq.render_depth(0))
    ctx, st = _init_both(cfg, model)
    _random_field(ctx, st, np.random.default_rng(3))
    # the device's fp32 skinning weights on both sides (mirror input)
    st.set_model(Hh.device_to_oracle_model(ctx.download_model()))
    assert ctx.forward_warp() == st.forward_warp() == 0
    g, o = ctx.download_model(), st.get_model()
    # fp64 arithmetic rounded to the fp32 store: the stored live state is the
    # one the reference chain rounds to (ds_blend.cuh warp_surfel)
    f32 = lambda a: np.asarray(a).astype(np.float32).astype(np.float64)  # noqa: E731
    assert np.array_equal(g["live_pos"], f32(o["live_pos"]))
    assert np.array_equal(g["live_nrm"], f32(o["live_nrm"]))
    ctx.close()


def test_model_maps_and_association_bit_exact():
    cfg, seq = scene()
    d0 = seq.render_depth(0)
    model, _ = frame_model(cfg, d0)
    ctx, st = _init_both(cfg, model)
    _random_field(ctx, st, np.random.default_rng(5), angle=0.01, shift=0.002)
    ctx.forward_warp()
    st.forward_warp()
    # share the device's fp32 live state with the oracle
    om = Hh.device_to_oracle_model(ctx.download_model())
    st.set_model(om)
    pose = O.pose_identity()
    ctx.frame_maps(d0, 1)
    st.build_frame(d0, 1)
    for t_now, t_last in ((1, 0), (50, 0)):
        g = ctx.render_model_maps(pose, t_now, t_last)
        o = st.render_model_maps(pose, t_now, t_last)
        assert np.array_equal(g["valid"], o["valid"])
        assert np.array_equal(g["idx"], o["idx"])
        assert np.array_equal(g["depth"][o["valid"] > 0], o["depth"][o["valid"] > 0])
        gp = ctx.associate(pose)
        op = st.find_correspondences(o, pose)
        assert len(gp["surfel"]) == len(op["surfel"]) > 500 or t_now == 50
        for k in ("surfel", "px", "py"):
            assert np.array_equal(gp[k], op[k])
        for k in ("v_model", "v_depth", "n_depth"):
            assert np.array_equal(gp[k], op[k])
    ctx.close()


def test_index_map_bit_exact():
    cfg, seq = scene()
    model, _ = frame_model(cfg, seq.render_depth(0))
    ctx, st = _init_both(cfg, model)
    om = Hh.device_to_oracle_model(ctx.download_model())
    st.set_model(om)
    pose = O.make_se3([0.01, -0.02, 0.005], [0.003, 0.001, -0.002])
    for f in (4, 1):
        g = ctx.render_index_map(pose, f)
        o, _ = st.render_index_map(pose, f)
        assert np.array_equal(g, o)
    ctx.close()


def test_normal_equations_pattern_and_values():
    cfg, seq = scene()
    d0 = seq.render_depth(0)
    model, _ = frame_model(cfg, d0)
    ctx, st = _init_both(cfg, model)
    _random_field(ctx, st, np.random.default_rng(7), angle=0.02, shift=0.003)
    om = Hh.device_to_oracle_model(ctx.download_model())
    st.set_model(om)
    ctx.frame_maps(d0, 1)
    st.build_frame(d0, 1)
    pose = O.pose_identity()
    g = ctx.build_normal_equations(pose, 1, 0)
    o = st.normal_equations(pose, 1, 0)
    N = ctx.num_nodes()
    Hg, Tg = Hh.bsr_to_dense(g, N)
    assert g["n_pairs"] == o["n_pairs"]
    assert np.array_equal(Tg, o["touched"])  # JtJ sparsity pattern bit-exact
    scale = np.abs(o["h"]).max()
    assert np.abs(Hg - o["h"]).max() <= 2e-6 * scale  # fp32 block storage
    gs = np.abs(o["g"]).max()
    assert np.abs(g["g"] - o["g"]).max() <= 1e-5 * gs
    assert abs(g["e_pre"] - o["e_pre"]) <= 1e-9 * max(o["e_pre"], 1e-30) + 1e-18
    ctx.close()


def test_pcg_converges_to_ldlt():
    cfg, seq = scene()
    d0 = seq.render_depth(0)
    model, _ = frame_model(cfg, d0)
    ctx, st = _init_both(cfg, model)
    _random_field(ctx, st, np.random.default_rng(9), angle=0.02, shift=0.003)
    om = Hh.device_to_oracle_model(ctx.download_model())
    st.set_model(om)
    ctx.frame_maps(d0, 1)
    st.build_frame(d0, 1)
    pose = O.pose_identity()
    g = ctx.build_normal_equations(pose, 1, 0)
    N = ctx.num_nodes()
    Hg, _ = Hh.bsr_to_dense(g, N)
    mu = 1e-6 * np.trace(Hg) / (6 * N) * 10
    delta, it, rel = ctx.pcg_solve(mu, 2000, 1e-10)
    assert rel <= 1e-9, (it, rel)
    ref = O.ldlt_solve(Hg + mu * np.eye(6 * N), -g["g"])
    assert np.abs(delta - ref).max() <= 1e-5 * np.abs(ref).max()
    ctx.close()


@pytest.mark.parametrize("noise", [0.0, 2.0])
def test_bilateral_prefilter_bit_exact(noise):
    """the 5x5 bilateral prefilter (depth_processing.cpp:71-101,
    sigma_s 4.5 px, sigma_d 30 mm) ahead of build_frame_maps, on noisy and clean
    depth: the filtered frame maps are bit-exact against the oracle's."""
    for name, size in (("bending_sheet", SMALL), ("articulated_body",
                                                 dict(fx=280.0, fy=280.0, cx=159.5, cy=119.5,
                                                      width=320, height=240))):
        cfg = pkg.make_config(**{**size, "bilateral_filter": 1})
        seq = pkg.SyntheticSequence(name, 20, cfg, noise_sigma_mm=noise)
        ctx = pkg.Context(cfg)
        st = O.OracleState(Hh.oracle_cfg(cfg))
        for t in (0, 5):
            d = seq.render_depth(t)
            vc = ctx.frame_maps(d, t)
            st.build_frame(d, t)
            g, o = ctx.download_frame(), st.get_frame()
            assert vc == o["valid_count"] > 0
            assert np.array_equal(g["valid"], o["valid"])
            assert np.array_equal(g["vert"], o["vert"])
            assert np.array_equal(g["nrm"], o["nrm"])
            assert np.array_equal(g["radius"], o["radius"])
        # the filter changes the maps relative to the unfiltered path
        raw = pkg.Context(pkg.make_config(**size))
        raw.frame_maps(d, 5)
        if noise > 0:
            assert not np.array_equal(raw.download_frame()["vert"], g["vert"])
        raw.close()
        ctx.close()


def test_assert_normal_equations_on_device(monkeypatch):
    """d4: assert_normal_equations (solver.cpp:157-167) on the device BSR system:
    the assembled H passes; an asymmetric entry or a diagonal block with a
    negative eigenvalue raises the reference's dynsurf::Error (DS_ERR_NUMERICAL)
    -- through the stage call, and inside solve_nonrigid with DS_CHECK_NE=1."""
    cfg, seq = scene()
    d0 = seq.render_depth(0)
    model, _ = frame_model(cfg, d0)
    ctx, st = _init_both(cfg, model)
    _random_field(ctx, st, np.random.default_rng(11), angle=0.02, shift=0.003)
    ctx.frame_maps(d0, 1)
    pose = O.pose_identity()
    ne = ctx.build_normal_equations(pose, 1, 0)
    ctx.check_normal_equations()  # the assembled system is symmetric PSD
    vals = ne["values"].copy()
    r = 0
    diag = [k for k in range(ne["row_ptr"][r], ne["row_ptr"][r + 1]) if ne["col"][k] == r][0]
    off = [k for k in range(ne["row_ptr"][r], ne["row_ptr"][r + 1]) if ne["col"][k] != r][0]
    scale = max(1.0, np.abs(vals).max())
    bad = vals.copy()
    bad[off, 0, 1] += 1e-3 * scale  # the mirror block no longer matches
    ctx.set_normal_equation_values(bad)
    with pytest.raises(pkg.errors.Error, match="symmetry"):
        ctx.check_normal_equations()
    bad = vals.copy()
    bad[diag] -= 2.0 * np.abs(bad[diag]).max() * np.eye(6)  # negative definite block
    ctx.set_normal_equation_values(bad)
    with pytest.raises(pkg.errors.Error, match="PSD"):
        ctx.check_normal_equations()
    ctx.set_normal_equation_values(vals)
    ctx.check_normal_equations()
    ctx.close()
    # the debug switch runs the check on every GN linearisation of the solve
    monkeypatch.setenv("DS_CHECK_NE", "1")
    pipe = pkg.Pipeline(cfg)
    for t in range(3):
        pipe.process_frame(seq.render_depth(t), t)
    pipe.close()
