"""CPU-side checks of the drop-in boundary: the sm_100a library loads without a GPU,
exports every entry point include/dynsurf_b200.h declares, maps statuses to the
reference's exception types, and has no CPU fallback."""
import ctypes as C
import os
import re

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols(header="dynsurf_b200.h"):
    src = open(os.path.join(REPO, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ds_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    import paper_1904_13073_b200._lib as L

    lib = L.load()
    syms = declared_symbols()
    assert len(syms) >= 45
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # and the Python binding declares a signature for each of them
    assert set(syms) <= set(L.SIGNATURES), set(syms) - set(L.SIGNATURES)


def test_synth_library_exports_every_declared_symbol():
    """The scene generator is a host-only library of its own (include/dynsurf_synth.h):
    generating inputs does not map the CUDA library."""
    import paper_1904_13073_b200._lib as L

    lib = L.load_synth()
    syms = declared_symbols("dynsurf_synth.h")
    assert len(syms) == 6
    assert all(hasattr(lib, s) for s in syms)
    assert set(syms) == set(L.SYNTH_SIGNATURES)
    assert not any(s.startswith("ds_synth") for s in declared_symbols())


def test_shared_object_is_sm100a():
    so = os.path.join(REPO, "paper_1904_13073_b200", "lib", "libdynsurf_b200.so")
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {so} 2>&1").read()
    assert "sm_100a" in out, out


def test_config_struct_layout_matches_oracle():
    import oracle_py as O
    from paper_1904_13073_b200._lib import DsConfig

    for (a, ta), (b, tb) in zip(O.OrConfig._fields_, DsConfig._fields_):
        assert a == b and ta == tb
    assert C.sizeof(DsConfig) > C.sizeof(O.OrConfig)


def test_validate_config_errors():
    import paper_1904_13073_b200 as pkg

    good = pkg.make_config(fx=140.0, fy=140.0, cx=79.5, cy=59.5, width=160, height=120)
    pkg.Pipeline.__init__  # noqa: B018
    from paper_1904_13073_b200 import _lib
    from paper_1904_13073_b200.pipeline import to_struct

    assert _lib.load().ds_validate_config(C.byref(to_struct(good))) == 0
    for bad in (dict(node_sigma=0.0), dict(knn_k=9), dict(epsilon=1.0), dict(fx=0.0),
                dict(knn_k=5), dict(node_neighbor_k=9)):
        cfg = dict(good)
        cfg.update(bad)
        st = _lib.load().ds_validate_config(C.byref(to_struct(cfg)))
        assert st == 4, bad  # DS_ERR_CONFIG -> ConfigError
        with pytest.raises(pkg.ConfigError):
            _lib.check(st)


def test_no_cpu_fallback_without_device():
    import paper_1904_13073_b200 as pkg

    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("a CUDA device is present")
    except ImportError:
        pass
    cfg = pkg.make_config(fx=140.0, fy=140.0, cx=79.5, cy=59.5, width=160, height=120)
    with pytest.raises(pkg.CudaError):
        pkg.Pipeline(cfg)


def test_synth_scenes_known_answers():
    import paper_1904_13073_b200 as pkg

    cfg = pkg.make_config(fx=140.0, fy=140.0, cx=79.5, cy=59.5, width=160, height=120)
    plane = pkg.SyntheticSequence("static_plane", 3, cfg).render_depth(1)
    # rect at z = 1 m covering |x| <= 0.4, |y| <= 0.3 (synth.cpp:278): 1000 mm
    assert plane[60, 80] == 1000
    assert set(np.unique(plane)) <= {0, 1000}
    with pytest.raises(pkg.UnknownScenario):
        pkg.SyntheticSequence("nope", 3, cfg)
    orbit = pkg.SyntheticSequence("rigid_orbit", 5, cfg)
    assert (orbit.render_depth(0) > 0).sum() > 500
    p = orbit.camera_pose(3)
    assert abs(np.linalg.det(p[:9].reshape(3, 3)) - 1) < 1e-12
    noisy = pkg.SyntheticSequence("static_plane", 3, cfg, noise_sigma_mm=2.0)
    a, b = noisy.render_depth(1), noisy.render_depth(1)
    assert np.array_equal(a, b) and (a[plane > 0] != 1000).any()


def test_config_scenes_sizes():
    """BASELINE configs: ~30k surfels / ~300 nodes (cfg 1), ~200k / ~1.5k (cfg 2)."""
    import oracle_py as O
    import harness as Hh
    import paper_1904_13073_b200 as pkg

    c1 = pkg.camera_config(320, 240, 280.0)
    d = pkg.SyntheticSequence("deforming_sphere", 10, c1).render_depth(0)
    st = O.OracleState(Hh.oracle_cfg(c1))
    st.build_frame(d, 0)
    assert 25000 < st.get_frame()["valid_count"] < 35000
    c2 = pkg.camera_config(640, 480, 560.0)
    d2 = pkg.SyntheticSequence("articulated_body", 100, c2).render_depth(0)
    st2 = O.OracleState(Hh.oracle_cfg(c2))
    st2.build_frame(d2, 0)
    assert 170000 < st2.get_frame()["valid_count"] < 230000


def test_config3_scene_pans_and_fills_the_frame():
    """BASELINE config 3 (large_scene, 1280x960): ~0.57M valid pixels, a panning
    camera (pose changes every frame) and the contact spheres closing."""
    import paper_1904_13073_b200 as pkg

    c3 = pkg.camera_config(1280, 960, 1120.0)
    seq = pkg.SyntheticSequence("large_scene", 60, c3)
    d0, d1 = seq.render_depth(0), seq.render_depth(1)
    assert (d0 > 0).sum() > 500_000  # ~0.57M per frame; the model passes 1M surfels by frame 2
    assert not np.array_equal(d0, d1)
    p0, p1 = np.array(seq.camera_pose(0)), np.array(seq.camera_pose(1))
    assert np.abs(p1 - p0).max() > 1e-4  # pans
    assert np.allclose(p0, np.eye(3).reshape(9).tolist() + [0, 0, 0])


def test_bench_configs_and_reference_arm_for_config3():
    import argparse
    import bench
    import bench_reference

    assert set(bench.CONFIGS) == {"cfg1", "cfg2", "cfg3"}
    cfg = bench.make_cfg(bench.CFG3)
    assert cfg["width"] == 1280 and cfg["max_nodes"] == 32768 and cfg["max_surfels"] == 20_000_000
    out = bench_reference.run_reference(argparse.Namespace(config="cfg3", steps=1, gpus=1))
    assert out["impl"] == "reference" and "unavailable" in out
