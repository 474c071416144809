"""PCG iterates of the device solver against a numpy restatement of the same
block-Jacobi PCG on (H + mu I) x = -g, x0 = 0, on a system assembled by the
device from a synthetic frame pair.

The reference solves each LM step with a dense LDLT (solver.cpp:383-386); the
B200 path replaces that step with this PCG, so there is no reference PCG to
match: `reference_pcg` below is the textbook recurrence written in numpy as an
fp64 check of the kernels' arithmetic, and test_pcg_converges_to_direct_solve
ties the converged PCG to the direct solve the reference performs.

Three device kernels run it: the cluster kernel (k_pcg_cluster.cu, one
thread-block cluster, fixed iteration budget; opt-in, DS_PCG_CLUSTER),
the cooperative grid kernel with pipelined recurrences (fixed
budget; the production path) and with the classic two-barrier
recurrences (tolerance stopping). All must reproduce the restated iterates
after k iterations up to fp64 rounding (relative 1e-8 on x, tolerance written
here; the matrix is the same fp32 BSR).
"""
import numpy as np
import pytest

import harness as Hh

pytestmark = pytest.mark.gpu
pkg = pytest.importorskip("paper_1904_13073_b200")


def reference_pcg(H, g, mu, iters):
    """solver.cpp:180-214 restated: z = M^-1 r with 6x6 diagonal-block inverses."""
    n = H.shape[0]
    A = H + mu * np.eye(n)
    Minv = np.zeros_like(A)
    for j in range(n // 6):
        s = slice(6 * j, 6 * j + 6)
        Minv[s, s] = np.linalg.inv(A[s, s])
    x = np.zeros(n)
    r = -g.copy()
    z = Minv @ r
    p = z.copy()
    rz = r @ z
    for _ in range(iters):
        q = A @ p
        alpha = rz / (p @ q)
        x += alpha * p
        r -= alpha * q
        z = Minv @ r
        rz_new = r @ z
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x


@pytest.fixture(scope="module")
def system():
    cfg = pkg.camera_config(160, 120, 140.0, pcg_max_iters=10)
    seq = pkg.SyntheticSequence("bending_sheet", 10, cfg)
    ctx = pkg.Context(cfg)
    ctx.process_frame(seq.render_depth(0), 0)
    ctx.frame_maps(seq.render_depth(2), 2)
    ne = ctx.build_normal_equations(np.eye(3).reshape(9).tolist() + [0.0, 0.0, 0.0], 2, 0)
    N = ctx.num_nodes()
    H, _ = Hh.bsr_to_dense(ne, N)
    yield ctx, H, ne["g"].copy()
    ctx.close()


def make_system(width=160, height=120, focal=140.0, scene="bending_sheet", frames=(0, 2)):
    cfg = pkg.camera_config(width, height, focal, pcg_max_iters=10)
    seq = pkg.SyntheticSequence(scene, 10, cfg)
    ctx = pkg.Context(cfg)
    ctx.process_frame(seq.render_depth(frames[0]), frames[0])
    ctx.frame_maps(seq.render_depth(frames[1]), frames[1])
    ne = ctx.build_normal_equations(np.eye(3).reshape(9).tolist() + [0.0, 0.0, 0.0], frames[1], 0)
    H, _ = Hh.bsr_to_dense(ne, ctx.num_nodes())
    return ctx, H, ne["g"].copy()


@pytest.mark.parametrize("iters", [1, 2, 5, 10])
@pytest.mark.parametrize("mode", ["cluster", "pipelined", "classic"])
def test_pcg_iterates_match_reference(system, monkeypatch, iters, mode):
    ctx, H, g = system
    if mode == "cluster":  # the cluster kernel: a context with DS_PCG_CLUSTER set
        monkeypatch.setenv("DS_PCG_CLUSTER", "8")  # read at context creation
        ctx, H, g = make_system()
    mu = 1e-6 * np.trace(H) / H.shape[0] * 10.0
    tol = 0.0 if mode != "classic" else 1e-150  # tol > 0 selects the classic recurrences
    x, it, _ = ctx.pcg_solve(mu, iters, tol)
    ref = reference_pcg(H, g, mu, iters)
    assert it == iters
    err = np.abs(x - ref).max() / max(np.abs(ref).max(), 1e-300)
    assert err < 1e-8, (mode, iters, err)
    if mode == "cluster":
        ctx.close()


@pytest.mark.parametrize("csize,cap", [("2", None), ("4", None), ("16", None), ("8", "6000"),
                                       ("8", "3000")])
def test_cluster_pcg_shapes_and_spill_paths(monkeypatch, csize, cap):
    """Cluster sizes 2..16, and a shrunken carve (DS_PCGC_SMEM) that forces
    the blocks to stream from L2 (6000 B), then the index lists to global
    scratch with the remote columns read straight through DSMEM (3000 B)."""
    monkeypatch.setenv("DS_PCG_CLUSTER", csize)
    if cap:
        monkeypatch.setenv("DS_PCGC_SMEM", cap)
    ctx, H, g = make_system()
    mu = 1e-5 * np.trace(H) / H.shape[0]
    x, it, _ = ctx.pcg_solve(mu, 10, 0.0)
    ref = reference_pcg(H, g, mu, 10)
    assert it == 10
    assert np.abs(x - ref).max() / max(np.abs(ref).max(), 1e-300) < 1e-8
    ctx.close()


def test_cluster_pcg_on_config2_system(monkeypatch):
    """BASELINE config 2 (articulated body, 640x480, ~1.5k nodes, ~14 blocks per
    row): the cluster kernel (16 CTAs, two row passes per thread) against the
    cooperative kernel and the numpy restatement."""
    monkeypatch.setenv("DS_PCG_CLUSTER", "16")
    ctx, H, g = make_system(640, 480, 560.0, "articulated_body", (0, 1))
    N = ctx.num_nodes()
    assert N > 1000
    mu = 1e-6 * np.trace(H) / H.shape[0]
    x, it, _ = ctx.pcg_solve(mu, 10, 0.0)
    ref = reference_pcg(H, g, mu, 10)
    assert it == 10
    assert np.abs(x - ref).max() / np.abs(ref).max() < 1e-8
    monkeypatch.setenv("DS_PCG_CLUSTER", "0")
    ctx2, H2, g2 = make_system(640, 480, 560.0, "articulated_body", (0, 1))
    assert np.array_equal(H, H2) and np.array_equal(g, g2)
    x2, _, _ = ctx2.pcg_solve(mu, 10, 0.0)
    assert np.abs(x - x2).max() / np.abs(x2).max() < 1e-9  # dot products in another tree
    ctx.close()
    ctx2.close()


def test_pcg_converges_to_direct_solve(system):
    ctx, H, g = system
    mu = 1e-3 * np.trace(H) / H.shape[0]
    x, it, rel = ctx.pcg_solve(mu, 5000, 1e-12)
    ref = np.linalg.solve(H + mu * np.eye(H.shape[0]), -g)
    assert rel <= 1e-12 and it < 5000
    assert np.abs(x - ref).max() / np.abs(ref).max() < 1e-8


def test_bsr_spmv_matches_dense(system):
    ctx, H, g = system
    x = np.random.default_rng(3).normal(size=H.shape[0])
    mu = 0.25
    y, ms = ctx.bsr_spmv(x, mu, 2)
    ref = H @ x + mu * x
    assert ms > 0
    assert np.abs(y - ref).max() <= 1e-12 * np.abs(ref).max() + 1e-300


@pytest.mark.parametrize("smem", ["0", "12000"])
@pytest.mark.parametrize("mode", ["pipelined", "classic"])
def test_pcg_global_scratch_path_matches_reference(monkeypatch, mode, smem):
    """Slices too large for shared memory (very large N) run the same
    recurrences with the matrix streamed from global memory (vectors still in
    shared memory, DS_PCG_SMEM=12000 at this size) or entirely on global
    scratch (DS_PCG_SMEM=0)."""
    monkeypatch.setenv("DS_PCG_SMEM", smem)  # read at context creation
    cfg = pkg.camera_config(160, 120, 140.0, pcg_max_iters=10)
    seq = pkg.SyntheticSequence("bending_sheet", 10, cfg)
    ctx = pkg.Context(cfg)
    ctx.process_frame(seq.render_depth(0), 0)
    ctx.frame_maps(seq.render_depth(2), 2)
    ne = ctx.build_normal_equations(np.eye(3).reshape(9).tolist() + [0.0, 0.0, 0.0], 2, 0)
    H, _ = Hh.bsr_to_dense(ne, ctx.num_nodes())
    g = ne["g"].copy()
    mu = 1e-5 * np.trace(H) / H.shape[0]
    x, it, _ = ctx.pcg_solve(mu, 10, 0.0 if mode == "pipelined" else 1e-150)
    ref = reference_pcg(H, g, mu, 10)
    assert it == 10
    assert np.abs(x - ref).max() / max(np.abs(ref).max(), 1e-300) < 1e-8
    ctx.close()
