"""The oracle pinned against the REFERENCE ITSELF (oracle/_ref).

`make -C oracle ref` compiles the unmodified reference sources
(/root/reference/proj/core/src, read in place) against repo-owned shims for
its absent dependencies (Eigen subset, libpng stub, GTest) -- SURVEY.md 7.1
step 1. Two checks pin the chain device -> oracle -> reference:

* the reference's own unit tests (proj/tests/*.cpp, 106 tests) pass against
  that build, which validates the shims;
* the oracle's `process_frame` (faithful fp64 mode) follows the compiled
  reference's `Pipeline::process_frame` (pipeline.cpp:74-142) frame by frame:
  every discrete count equal, poses / energies / the model and the warp
  field equal to rounding (the only differences are summation orders inside
  Eigen-expression arithmetic).

The device is held to the oracle in lock-step (tests/lockstep.py,
test_gpu_baseline_parity.py); this file closes the chain to the reference.
CPU only; skipped when oracle/_ref cannot be built (no /root/reference and no
prebuilt library).
"""
import os
import subprocess

import numpy as np
import pytest

import oracle_py as O
import ref_py as R

pkg = pytest.importorskip("paper_1904_13073_b200")


@pytest.fixture(scope="module")
def ref_built():
    try:
        ok = R.build()
    except subprocess.CalledProcessError as e:  # pragma: no cover - build failure is a failure
        pytest.fail(f"oracle/_ref build failed: {e}")
    if not ok:
        pytest.skip("oracle/_ref not built (no /root/reference here and no prebuilt library)")
    return True


def test_reference_unit_tests_pass_on_the_ref_build(ref_built):
    if os.path.isdir(R.REF_SRC):
        subprocess.run(["make", "-s", "-j8", "-C", os.path.join(R.REPO, "oracle"), "ref-tests"],
                       check=True)
    if not os.path.exists(R.REF_TESTS):
        pytest.skip("reference unit-test binary not built")
    r = subprocess.run([R.REF_TESTS], capture_output=True, text=True, timeout=900)
    tail = r.stdout[-2000:] + r.stderr[-2000:]
    assert r.returncode == 0, tail
    ran = [ln for ln in r.stdout.splitlines() if ln.startswith("[==========]")]
    assert ran and int(ran[-1].split()[1]) >= 100, tail
    assert "[  FAILED  ]" not in r.stdout


def _compare_sequence(scene, W, H, f, frames, gn):
    cfg = pkg.camera_config(W, H, f, max_gn_iters=gn)
    seq = pkg.SyntheticSequence(scene, frames, cfg)
    ocfg = O.make_config(**{k: v for k, v in cfg.items() if k in O.DEFAULTS})
    op = O.OraclePipeline(ocfg)  # faithful fp64, as shipped
    rp = R.RefPipeline(ocfg)
    counts = ("valid_pixels", "surfel_count", "node_count")
    fusion = ("fused", "appended", "removed", "compressive_rejected", "low_support_rejected",
              "new_nodes", "degenerate_warps")
    tracked = 0
    for t in range(frames):
        d = seq.render_depth(t)
        so = op.process_frame(d, t)
        sr = rp.process_frame(d, t)
        assert bool(so.skipped) == bool(sr["skipped"]), t
        for k in counts:
            assert getattr(so, k) == sr[k], (t, k)
        for k in fusion:
            assert getattr(so.fusion, k) == sr[k], (t, k)
        assert bool(so.reinit) == bool(sr["reinit"]) and so.reinit_removed == sr["reinit_removed"]
        assert so.rigid.correspondences == sr["rigid_correspondences"], t
        assert so.solver.iterations == sr["solver_iterations"], t
        assert so.solver.correspondences == sr["solver_correspondences"], t
        po = np.array(so.pose[:])
        pr = np.concatenate([sr["pose_R"].ravel(), sr["pose_t"]])
        assert np.abs(po - pr).max() <= 1e-10, (t, np.abs(po - pr).max())
        e0 = max(sr["initial_energy"], 1e-30)
        assert abs(so.solver.initial_energy - sr["initial_energy"]) <= 1e-9 * e0, t
        assert abs(so.solver.final_energy - sr["final_energy"]) <= 1e-9 * e0, t
        tracked += so.solver.iterations > 0
    assert tracked >= frames - 2  # the solver ran on the tracked frames
    om, rm = op.state.get_model(), rp.model()
    assert len(om["ref_pos"]) == len(rm["ref_pos"]) > 1000
    for a, b in (("ref_pos", "ref_pos"), ("live_pos", "live_pos"), ("ref_nrm", "ref_nrm"),
                 ("live_nrm", "live_nrm"), ("ref_conf", "confidence"), ("ref_radius", "radius")):
        assert np.abs(np.asarray(om[a]) - rm[b]).max() <= 1e-9, (a, np.abs(om[a] - rm[b]).max())
    assert np.array_equal(om["ref_t_init"], rm["t_init"])
    assert np.array_equal(om["ref_t_obs"], rm["t_obs"])
    assert np.array_equal(om["skin_count"], rm["skin_count"])
    # skinning entries: the same (node, weight) sets; the slot order may differ
    # only where two nodes are equidistant up to rounding (a (d2, index) tie
    # decided by the last bit, e.g. a surfel midway between grid nodes)
    oi, ow = np.asarray(om["skin_idx"])[:, :4], np.asarray(om["skin_w"])[:, :4]
    diff = np.where((oi != rm["skin_idx"]).any(1))[0]
    assert len(diff) <= 1e-3 * len(oi), len(diff)
    for i in diff:
        a, b = np.argsort(oi[i]), np.argsort(rm["skin_idx"][i])
        assert np.array_equal(oi[i][a], rm["skin_idx"][i][b])
        assert np.abs(ow[i][a] - rm["skin_w"][i][b]).max() <= 1e-9
        assert np.abs(np.sort(ow[i]) - np.sort(rm["skin_w"][i])).max() <= 1e-9
    assert np.abs(np.sort(ow, 1) - np.sort(rm["skin_w"], 1)).max() <= 1e-9
    on, rn = op.state.get_nodes(), rp.nodes()
    assert len(on["pos"]) == len(rn["pos"])
    # appended nodes sit at inverse-warped surfels: equal to rounding
    assert np.abs(np.asarray(on["pos"]) - rn["pos"]).max() <= 1e-10
    assert np.array_equal(np.asarray(on["nbr"]), rn["nbr"])
    assert np.abs(np.asarray(on["dq"]).reshape(-1, 8) - rn["dq"]).max() <= 1e-10


@pytest.mark.parametrize("scene", ["rigid_orbit", "bending_sheet"])
def test_oracle_process_frame_matches_reference_160x120(ref_built, scene):
    """6 frames, 10 GN iterations (the reference's default)."""
    _compare_sequence(scene, 160, 120, 140.0, 6, 10)


def test_oracle_process_frame_matches_reference_config1(ref_built):
    """BASELINE config 1 (deforming sphere, 320x240, 3 GN iterations), the
    first 4 frames."""
    _compare_sequence("deforming_sphere", 320, 240, 280.0, 4, 3)
