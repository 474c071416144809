"""The C++ host side of SURVEY 8(f) row 2 (include/dynsurf_io.hpp) and the
reference CLI's verbs over it (paper_1904_13073_b200/tools/dynsurf_cli.cpp):
16-bit depth PNG read/write (png_io.cpp:23-70), config files (config.cpp:140-196),
`synth` (synth.cpp:411-440), `check` (tools/main.cpp:74-165) and `run`
(process_sequence, pipeline.cpp:205-295; GPU). Byte formats are compared with
the Python twin, paper_1904_13073_b200/sequence_io.py."""
import json
import os
import shutil
import subprocess

import numpy as np
import pytest

from test_sequence_io import _encode_filtered, _png

pkg = pytest.importorskip("paper_1904_13073_b200")
sio = pkg.sequence_io
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(REPO, "paper_1904_13073_b200", "build", "dynsurf_b200")


@pytest.fixture(scope="module")
def png_check(tmp_path_factory):
    if shutil.which("g++") is None:
        pytest.skip("g++ not available")
    exe = tmp_path_factory.mktemp("bin") / "png_check"
    subprocess.run(["g++", "-std=c++17", "-O1", "-I" + os.path.join(REPO, "include"),
                    "-I/usr/local/cuda/include", "-o", str(exe),
                    os.path.join(REPO, "tests", "cpp", "png_check.cpp"), "-lz"], check=True)
    return str(exe)


@pytest.fixture(scope="module")
def cli():
    if not os.path.exists(CLI):
        subprocess.run(["make", "-s", "-C", os.path.join(REPO, "paper_1904_13073_b200")],
                       check=True)
    return CLI


def _read_cpp(exe, path, out=None):
    args = [exe, str(path)] + ([str(out)] if out else [])
    lines = subprocess.run(args, capture_output=True, text=True, check=True).stdout.split()
    if lines[0] in ("CorruptFrame", "IoFailure"):
        return lines[0]
    w, h = int(lines[0]), int(lines[1])
    return np.array(lines[2:], np.uint16).reshape(h, w)


def test_cpp_png_reader_matches_python(png_check, tmp_path):
    rng = np.random.default_rng(5)
    d = rng.integers(0, 65535, size=(11, 29), dtype=np.uint16)
    filt = tmp_path / "filtered.png"  # every row filter type (PNG spec 9.2)
    filt.write_bytes(_png(29, 11, 16, 0, _encode_filtered(d)))
    assert np.array_equal(_read_cpp(png_check, filt), d)
    assert np.array_equal(sio.read_depth_png(str(filt)), d)
    # the C++ writer writes the Python writer's bytes (filter 0 rows, zlib 6)
    py = tmp_path / "py.png"
    sio.write_depth_png(str(py), d)
    cpp = tmp_path / "cpp.png"
    assert np.array_equal(_read_cpp(png_check, filt, cpp), d)
    assert cpp.read_bytes() == py.read_bytes()


def test_cpp_png_reader_errors(png_check, tmp_path):
    assert _read_cpp(png_check, tmp_path / "missing.png") == "IoFailure"
    bad = tmp_path / "bad.png"
    bad.write_bytes(b"not a png at all")
    assert _read_cpp(png_check, bad) == "CorruptFrame"
    rgb = tmp_path / "rgb.png"
    rgb.write_bytes(_png(4, 4, 8, 2, b"\0" * (4 * (1 + 12))))
    assert _read_cpp(png_check, rgb) == "CorruptFrame"
    good = bytearray(_png(3, 2, 16, 0, b"\0" * (2 * (1 + 6))))
    good[-20] ^= 0xFF  # damaged chunk data (CRC mismatch)
    trunc = tmp_path / "crc.png"
    trunc.write_bytes(bytes(good))
    assert _read_cpp(png_check, trunc) == "CorruptFrame"


def test_cli_synth_writes_the_reference_layout(cli, tmp_path):
    out = tmp_path / "seq"
    r = subprocess.run([cli, "synth", "--scenario", "bending_sheet", "--output", str(out),
                        "--frames", "4", "--noise", "2"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert sorted(os.listdir(out)) == ["config.cfg"] + [f"frame-{t:06d}.png" for t in range(4)]
    cfg = pkg.make_config(fx=140.0, fy=140.0, cx=79.5, cy=59.5, width=160, height=120)
    seq = pkg.SyntheticSequence("bending_sheet", 4, cfg, noise_sigma_mm=2.0)
    for t in range(4):
        assert np.array_equal(sio.read_depth_png(str(out / f"frame-{t:06d}.png")),
                              seq.render_depth(t))
    keys = dict(ln.split() for ln in (out / "config.cfg").read_text().splitlines())
    assert keys["width"] == "160" and keys["height"] == "120" and keys["fx"] == "140"
    assert keys["node_sigma"] == "0.025000000000000001"  # precision 17, config.cpp:47-51
    assert list(keys) == sorted(keys)  # std::map order
    r = subprocess.run([cli, "synth", "--scenario", "nope", "--output", str(tmp_path / "x")],
                       capture_output=True, text=True)
    assert r.returncode == 1 and "unknown scenario" in r.stderr


def _metrics_line(frame, count, appended=0, removed=0, reinit=False, nodes=10, e0=1.0, e1=0.5,
                  valid=100, skipped=False):
    if skipped:
        return json.dumps({"frame": frame, "skipped": True})
    return json.dumps({"frame": frame, "skipped": False, "valid_pixels": valid,
                       "surfel_count": count, "node_count": nodes, "fused": 5,
                       "appended": appended, "removed": removed, "reinit": reinit,
                       "reinit_removed": 0, "initial_energy": e0, "final_energy": e1})


def test_cli_check_invariants(cli, tmp_path):
    good = tmp_path / "good.jsonl"
    good.write_text("\n".join([_metrics_line(0, 100), _metrics_line(1, 110, appended=12,
                                                                      removed=2, nodes=12),
                               _metrics_line(2, 0, skipped=True),
                               _metrics_line(3, 115, appended=5, nodes=12)]) + "\n")
    r = subprocess.run([cli, "check", str(good)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout
    names = [ln.split()[1] for ln in r.stdout.splitlines()]
    assert names == sorted(["parse", "frames_increasing", "counts_nonnegative",
                            "appended_within_valid_pixels", "surfel_count_accounting",
                            "energy_nonincreasing", "nodes_monotonic_between_reinits"])
    assert all(ln.startswith("PASS") for ln in r.stdout.splitlines())
    bad = tmp_path / "bad.jsonl"
    bad.write_text("\n".join([_metrics_line(0, 100), _metrics_line(1, 111, appended=12,
                                                                     removed=2, nodes=9),
                              _metrics_line(1, 111, e0=0.5, e1=0.7), "{not json"]) + "\n")
    r = subprocess.run([cli, "check", str(bad)], capture_output=True, text=True)
    assert r.returncode == 1
    res = {ln.split()[1]: ln.split()[0] for ln in r.stdout.splitlines()}
    assert res["surfel_count_accounting"] == "FAIL" and res["frames_increasing"] == "FAIL"
    assert res["nodes_monotonic_between_reinits"] == "FAIL"
    assert res["energy_nonincreasing"] == "FAIL" and res["parse"] == "FAIL"
    assert res["appended_within_valid_pixels"] == "PASS"
    empty = tmp_path / "empty.jsonl"
    empty.write_text("")
    assert subprocess.run([cli, "check", str(empty)], capture_output=True).returncode == 2
    assert subprocess.run([cli, "check", str(tmp_path / "no.jsonl")],
                          capture_output=True).returncode == 2


@pytest.mark.gpu
def test_cli_run_matches_python_process_sequence(cli, tmp_path):
    """`dynsurf_b200 run` (C++ process_sequence + PNG ingest over the B200
    pipeline) writes the same metrics / nodes logs and PLY files, byte for
    byte, as the Python process_sequence on the same frames; `check` passes."""
    seq_dir = tmp_path / "seq"
    subprocess.run([cli, "synth", "--scenario", "bending_sheet", "--output", str(seq_dir),
                    "--frames", "12"], check=True, capture_output=True)
    (seq_dir / "frame-000005.png").write_bytes(b"corrupt")  # skipped like the reference
    out_cpp = tmp_path / "out_cpp"
    r = subprocess.run([cli, "run", "--input", str(seq_dir), "--output", str(out_cpp),
                        "--ply_every", "4", "--log_nodes"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert "processed 11 frames (1 skipped)" in r.stdout
    assert "skipping frame 5" in r.stderr
    cfg = pkg.make_config(fx=140.0, fy=140.0, cx=79.5, cy=59.5, width=160, height=120)
    out_py = tmp_path / "out_py"
    s = sio.process_sequence(str(seq_dir), cfg, sio.PipelineOptions(str(out_py), 4, True))
    assert s.frames_processed == 11 and s.frames_skipped == 1
    for name in ("metrics.jsonl", "nodes.jsonl", "model-000000.ply", "model-000004.ply",
                 "model-000008.ply", "final_live.ply", "final_reference.ply"):
        assert (out_cpp / name).read_bytes() == (out_py / name).read_bytes(), name
    r = subprocess.run([cli, "check", str(out_cpp / "metrics.jsonl")], capture_output=True,
                       text=True)
    assert r.returncode == 0, r.stdout
