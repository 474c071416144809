"""Oracle pinned against the reference's DQ-algebra known answers
(proj/tests/test_geometry.cpp:16-207)."""
import math

import numpy as np
import pytest

import oracle_py as O


def R(p):
    return O.pose_R(p)


def t(p):
    return O.pose_t(p)


def test_identity_transform():  # :16-21
    dq = O.dq_from_se3(O.pose_identity())
    assert abs(dq[0] - 1.0) < 1e-15 and np.linalg.norm(dq[1:4]) < 1e-15
    assert np.linalg.norm(dq[4:]) < 1e-15


def test_pure_translation():  # :23-28
    dq = O.dq_from_se3(O.make_se3([0, 0, 0], [1, 0, 0]))
    assert np.linalg.norm(dq[:4] - [1, 0, 0, 0]) < 1e-15
    assert np.linalg.norm(dq[4:] - [0, 0.5, 0, 0]) < 1e-15


def test_half_turn_about_z():  # :30-36
    dq = O.dq_from_se3(O.make_se3([0, 0, math.pi], [0, 0, 0]))
    assert abs(abs(dq[3]) - 1.0) < 1e-12
    assert np.linalg.norm(dq[:3]) < 1e-12 and np.linalg.norm(dq[4:]) < 1e-12


def test_round_trip():  # :38-47
    rng = np.random.default_rng(7)
    for _ in range(200):
        p = O.random_se3(rng, 3.0, 1.0)
        b = O.dq_to_se3(O.dq_from_se3(p))
        assert np.abs(R(b) - R(p)).max() < 1e-9
        assert np.linalg.norm(t(b) - t(p)) < 1e-9


def test_apply_matches_se3():  # :49-56
    rng = np.random.default_rng(11)
    for _ in range(100):
        p = O.random_se3(rng, 3.0, 1.0)
        x = O.random_point(rng, 1.0)
        assert np.linalg.norm(O.dq_apply(O.dq_from_se3(p), x) - O.se3_apply(p, x)) < 1e-9


def test_composition_matches_product():  # :58-71
    rng = np.random.default_rng(13)
    for _ in range(100):
        a = O.random_se3(rng, 2.0, 0.7)
        b = O.random_se3(rng, 2.0, 0.7)
        prod = O.dq_mul(O.dq_from_se3(a), O.dq_from_se3(b))
        direct = O.dq_from_se3(O.se3_mul(a, b))
        s = -1.0 if prod[:4] @ direct[:4] < 0 else 1.0
        assert np.linalg.norm(s * prod[:4] - direct[:4]) < 1e-9
        assert np.linalg.norm(s * prod[4:] - direct[4:]) < 1e-9


def test_normalization_invariants():  # :73-84
    rng = np.random.default_rng(17)
    for _ in range(100):
        raw = np.concatenate([[rng.uniform(-1, 1) + 1.5], rng.uniform(-1, 1, 3),
                              rng.uniform(-1, 1, 4)])
        n = O.dq_normalized(raw)
        assert abs(np.linalg.norm(n[:4]) - 1) < 1e-12
        assert abs(n[:4] @ n[4:]) < 1e-12


def test_blend_identity():  # :86-93
    b = O.blend(np.tile(O.IDENTITY_DQ, (3, 1)), [0.2, 0.5, 1.3])
    p = O.dq_to_se3(b)
    assert np.abs(R(p) - np.eye(3)).max() < 1e-12 and np.linalg.norm(t(p)) < 1e-12


def test_blend_equal_inputs():  # :95-104
    rng = np.random.default_rng(23)
    tr = O.random_se3(rng)
    p = O.dq_to_se3(O.blend(np.tile(O.dq_from_se3(tr), (4, 1)), [0.1, 0.9, 0.4, 2.0]))
    assert np.abs(R(p) - R(tr)).max() < 1e-9 and np.linalg.norm(t(p) - t(tr)) < 1e-9


def test_blend_two_translations_average():  # :106-115
    dqs = [O.dq_from_se3(O.make_se3([0, 0, 0], [1, 0, 0])),
           O.dq_from_se3(O.make_se3([0, 0, 0], [0, 1, 0]))]
    p = O.dq_to_se3(O.blend(dqs, [0.7, 0.7]))
    assert np.linalg.norm(t(p) - [0.5, 0.5, 0]) < 1e-12
    assert np.abs(R(p) - np.eye(3)).max() < 1e-12


def test_blend_single_neighbor_exact():  # :117-126
    rng = np.random.default_rng(29)
    tr = O.random_se3(rng)
    p = O.dq_to_se3(O.blend([O.dq_from_se3(tr)], [0.3]))
    assert np.abs(R(p) - R(tr)).max() < 1e-12 and np.linalg.norm(t(p) - t(tr)) < 1e-12


def test_blend_weight_scale_invariance():  # :128-142
    rng = np.random.default_rng(31)
    dqs = [O.dq_from_se3(O.random_se3(rng)) for _ in range(4)]
    w = [0.1 + i * 0.2 for i in range(4)]
    a = O.dq_to_se3(O.blend(dqs, w))
    b = O.dq_to_se3(O.blend(dqs, [x * 37.5 for x in w]))
    assert np.abs(R(a) - R(b)).max() < 1e-12 and np.linalg.norm(t(a) - t(b)) < 1e-12


def test_blend_antipodal_sign_fix():  # :144-156
    rng = np.random.default_rng(37)
    tr = O.random_se3(rng)
    d = O.dq_from_se3(tr)
    p = O.dq_to_se3(O.blend([d, -d], [1.0, 1.0]))
    assert np.abs(R(p) - R(tr)).max() < 1e-9 and np.linalg.norm(t(p) - t(tr)) < 1e-9


def test_blend_degenerate():  # :158-162
    assert O.blend(np.tile(O.IDENTITY_DQ, (2, 1)), [1e-12, 1e-12]) is None


def test_blend_orthogonal_half_turns():  # :164-177
    a = O.dq_from_se3(O.make_se3([0, 0, math.pi], [0, 0, 0]))
    c = O.dq_from_se3(O.make_se3([math.pi, 0, 0], [0, 0, 0]))
    assert O.blend([a, c], [1.0, 1.0]) is not None


def test_skinning_weight_reference_values():  # :179-188
    p = np.array([0.1, 0.2, 0.3])
    assert abs(O.skinning_weight(p, p, 0.025) - 1.0) < 1e-15
    a = p + [0.025, 0, 0]
    assert abs(O.skinning_weight(a, p, 0.025) - math.exp(-0.5)) < 1e-12
    assert abs(O.skinning_weight(a, p, 0.025) - 0.60653) < 1e-5
    b = p + [0, 0.075, 0]
    assert abs(O.skinning_weight(b, p, 0.025) - math.exp(-4.5)) < 1e-12
    assert abs(O.skinning_weight(b, p, 0.025) - 0.011109) < 1e-6


def test_se3_increment_matches_composition():  # :190-199
    rng = np.random.default_rng(41)
    base = O.random_se3(rng)
    om, sh = np.array([0.01, -0.02, 0.005]), np.array([0.001, 0.002, -0.003])
    inc = O.se3_increment(om, sh, base)
    exp = O.se3_mul(O.make_se3(om, sh), base)
    assert np.abs(R(inc) - R(exp)).max() < 1e-9 and np.linalg.norm(t(inc) - t(exp)) < 1e-12


@pytest.mark.parametrize("angle", [0.0, 1e-13, 0.3, 2.5, math.pi])
def test_quat_matrix_round_trip(angle):
    axis = np.array([0.3, -0.5, 0.8])
    axis /= np.linalg.norm(axis)
    q = O.quat_from_rotvec(axis * angle)
    Rm = O.matrix_from_quat(q)
    assert abs(np.linalg.det(Rm) - 1) < 1e-12 and np.abs(Rm @ Rm.T - np.eye(3)).max() < 1e-12
    q2 = O.quat_from_matrix(Rm)
    assert q2[0] >= 0
    s = 1.0 if q2 @ q >= 0 else -1.0
    assert np.abs(s * q2 - q).max() < 1e-9


def test_ldlt_matches_numpy_and_handles_zero_pivots():
    rng = np.random.default_rng(3)
    A = rng.normal(size=(12, 12))
    A = A @ A.T + 0.1 * np.eye(12)
    b = rng.normal(size=12)
    assert np.allclose(O.ldlt_solve(A, b), np.linalg.solve(A, b), rtol=1e-10, atol=1e-12)
    # plane-like rank deficiency (exact zero rows/cols): Eigen pseudo-inverse semantics
    B = np.zeros((6, 6))
    J = rng.normal(size=(50, 3))
    B[np.ix_([0, 1, 5], [0, 1, 5])] = J.T @ J
    rhs = np.zeros(6)
    rhs[[0, 1, 5]] = rng.normal(size=3)
    x = O.ldlt_solve(B, rhs)
    assert np.all(np.isfinite(x)) and np.allclose(x[[2, 3, 4]], 0.0)
    assert np.allclose(B @ x, rhs, atol=1e-10)


def test_sigma_max3():
    rng = np.random.default_rng(4)
    for _ in range(20):
        M = rng.normal(size=(3, 3))
        assert abs(O.sigma_max3(M) - np.linalg.svd(M, compute_uv=False)[0]) < 1e-12
