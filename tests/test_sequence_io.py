"""On-disk / log formats: depth PNG, binary PLY,
metrics.jsonl / timings.jsonl lines, and process_sequence over a frame
directory (reference: png_io.cpp, ply_io.cpp:10-95, pipeline.cpp:144-291).

CPU tests pin the formats byte-for-byte against what the reference writes;
the GPU test runs process_sequence on the B200 pipeline and checks its logs
and exports against the device state and the oracle pipeline.
"""
import json
import math
import struct
import zlib

import numpy as np
import pytest

import harness as Hh
import oracle_py as O

pkg = pytest.importorskip("paper_1904_13073_b200")
sio = pkg.sequence_io

SMALL = dict(fx=140.0, fy=140.0, cx=79.5, cy=59.5, width=160, height=120)


def _encode_filtered(img: np.ndarray, bpp=2) -> bytes:
    """Test-side PNG encoder using filter type (y % 5) on row y (PNG spec §9)."""
    h, w = img.shape
    rows = img.astype(">u2").view(np.uint8).reshape(h, w * bpp).astype(np.int64)
    out = bytearray()
    prior = np.zeros(w * bpp, np.int64)
    for y in range(h):
        f, cur = y % 5, rows[y]
        left = np.concatenate([np.zeros(bpp, np.int64), cur[:-bpp]])
        upleft = np.concatenate([np.zeros(bpp, np.int64), prior[:-bpp]])
        if f == 0:
            pred = np.zeros_like(cur)
        elif f == 1:
            pred = left
        elif f == 2:
            pred = prior
        elif f == 3:
            pred = (left + prior) >> 1
        else:
            p = left + prior - upleft
            pa, pb, pc = np.abs(p - left), np.abs(p - prior), np.abs(p - upleft)
            pred = np.where((pa <= pb) & (pa <= pc), left, np.where(pb <= pc, prior, upleft))
        out.append(f)
        out += ((cur - pred) & 0xFF).astype(np.uint8).tobytes()
        prior = cur
    return bytes(out)


def _png(w, h, bit_depth, color, idat: bytes) -> bytes:
    return (sio._PNG_SIG + sio._chunk(b"IHDR", struct.pack(">IIBBBBB", w, h, bit_depth, color,
                                                           0, 0, 0))
            + sio._chunk(b"IDAT", zlib.compress(idat)) + sio._chunk(b"IEND", b""))


def test_depth_png_round_trip(tmp_path):
    rng = np.random.default_rng(7)
    d = rng.integers(0, 65536, size=(37, 53), dtype=np.uint16)
    d[0, 0], d[-1, -1] = 0, 65535
    p = str(tmp_path / "frame-000000.png")
    sio.write_depth_png(p, d)
    back = sio.read_depth_png(p)
    assert back.dtype == np.uint16 and back.shape == d.shape
    assert np.array_equal(back, d)
    # the file is a standard 16-bit grayscale PNG: IHDR right after the signature
    blob = open(p, "rb").read()
    assert blob[:8] == b"\x89PNG\r\n\x1a\n" and blob[12:16] == b"IHDR"
    assert struct.unpack(">IIBB", blob[16:26]) == (53, 37, 16, 0)


def test_depth_png_decodes_every_row_filter(tmp_path):
    rng = np.random.default_rng(3)
    d = rng.integers(0, 5000, size=(11, 29), dtype=np.uint16)
    p = tmp_path / "f.png"
    p.write_bytes(_png(29, 11, 16, 0, _encode_filtered(d)))
    assert np.array_equal(sio.read_depth_png(str(p)), d)


def test_depth_png_full_frame_filters_native_speed(tmp_path):
    """A 640x480 frame with every row filter (libpng's default adaptive
    filtering uses Average / Paeth heavily): decoded exactly by the native
    unfilter (ds_png_unfilter) in well under the GPU frame budget's order of
    magnitude (the Python per-byte loop took ~1 s)."""
    import time

    rng = np.random.default_rng(11)
    d = rng.integers(0, 5000, size=(480, 640), dtype=np.uint16)
    p = tmp_path / "big.png"
    p.write_bytes(_png(640, 480, 16, 0, _encode_filtered(d)))
    sio.read_depth_png(str(p))  # warm (library load)
    t0 = time.perf_counter()
    back = sio.read_depth_png(str(p))
    dt = time.perf_counter() - t0
    assert np.array_equal(back, d)
    assert dt < 0.1, dt
    bad = bytearray(_encode_filtered(d[:2, :4]))
    bad[0] = 7  # invalid filter type
    q = tmp_path / "badfilter.png"
    q.write_bytes(_png(4, 2, 16, 0, bytes(bad)))
    with pytest.raises(pkg.CorruptFrame, match="filter"):
        sio.read_depth_png(str(q))


def test_depth_png_errors(tmp_path):
    with pytest.raises(pkg.IoFailure):
        sio.read_depth_png(str(tmp_path / "missing.png"))
    bad = tmp_path / "bad.png"
    bad.write_bytes(b"not a png at all")
    with pytest.raises(pkg.CorruptFrame, match="not a PNG"):
        sio.read_depth_png(str(bad))
    gray8 = tmp_path / "g8.png"
    gray8.write_bytes(_png(4, 2, 8, 0, b"\x00" * 5 * 2))
    with pytest.raises(pkg.CorruptFrame, match="16-bit grayscale"):
        sio.read_depth_png(str(gray8))
    good = _png(4, 2, 16, 0, b"\x00" * 9 * 2)
    crc = tmp_path / "crc.png"
    crc.write_bytes(good[:-20] + bytes([good[-20] ^ 0xFF]) + good[-19:])
    with pytest.raises(pkg.CorruptFrame):
        sio.read_depth_png(str(crc))
    trunc = tmp_path / "trunc.png"
    trunc.write_bytes(good[:40])
    with pytest.raises(pkg.CorruptFrame):
        sio.read_depth_png(str(trunc))


def _model(n, seed=1):
    rng = np.random.default_rng(seed)
    return dict(ref_pos=rng.normal(size=(n, 3)), ref_nrm=rng.normal(size=(n, 3)),
                live_pos=rng.normal(size=(n, 3)), live_nrm=rng.normal(size=(n, 3)),
                radius=rng.random(n), conf=rng.random(n) * 10)


def test_ply_bytes_and_round_trip(tmp_path):
    m = _model(17)
    p = str(tmp_path / "m.ply")
    sio.export_pointcloud(m, "live", p)
    blob = open(p, "rb").read()
    header = ("ply\nformat binary_little_endian 1.0\nelement vertex 17\n"
              "property double x\nproperty double y\nproperty double z\n"
              "property double nx\nproperty double ny\nproperty double nz\n"
              "property double radius\nproperty double confidence\nend_header\n").encode()
    assert blob[:len(header)] == header and len(blob) == len(header) + 17 * 64
    rec = np.frombuffer(blob[len(header):], "<f8").reshape(17, 8)
    assert np.array_equal(rec[:, 0:3], m["live_pos"]) and np.array_equal(rec[:, 7], m["conf"])
    c = sio.read_pointcloud(p)
    assert np.array_equal(c["positions"], m["live_pos"])
    assert np.array_equal(c["normals"], m["live_nrm"])
    assert np.array_equal(c["radii"], m["radius"]) and np.array_equal(c["confidences"], m["conf"])
    sio.export_pointcloud(m, "reference", p)
    assert np.array_equal(sio.read_pointcloud(p)["positions"], m["ref_pos"])


def test_ply_errors(tmp_path):
    with pytest.raises(pkg.EmptyGeometry):
        sio.export_pointcloud(_model(0), "live", str(tmp_path / "e.ply"))
    p = tmp_path / "m.ply"
    sio.export_pointcloud(_model(3), "live", str(p))
    blob = p.read_bytes()
    p.write_bytes(blob[:-8])
    with pytest.raises(pkg.IoFailure, match="truncated"):
        sio.read_pointcloud(str(p))
    p.write_bytes(blob.replace(b"property double nx", b"property float nx"))
    with pytest.raises(pkg.IoFailure, match="property"):
        sio.read_pointcloud(str(p))
    p.write_bytes(blob.replace(b"binary_little_endian", b"ascii"))
    with pytest.raises(pkg.IoFailure, match="format"):
        sio.read_pointcloud(str(p))
    p.write_bytes(b"plx\n")
    with pytest.raises(pkg.IoFailure, match="not a PLY"):
        sio.read_pointcloud(str(p))
    with pytest.raises(pkg.IoFailure):
        sio.read_pointcloud(str(tmp_path / "missing.ply"))


# nlohmann::json::dump outputs for doubles (Grisu2 digits + format_buffer layout)
NLOHMANN_DOUBLES = [
    (0.0, "0.0"), (-0.0, "-0.0"), (1.0, "1.0"), (0.1, "0.1"), (12.5, "12.5"),
    (100.0, "100.0"), (1e-05, "1e-05"), (0.0001, "0.0001"), (-2.5e-07, "-2.5e-07"),
    (123456789012345.0, "123456789012345.0"), (1e15, "1e+15"), (1.5e300, "1.5e+300"),
    (0.001234, "0.001234"), (5e-324, "5e-324"), (float("nan"), "null"),
    (float("inf"), "null"), (0.30000000000000004, "0.30000000000000004"),
]


@pytest.mark.parametrize("x,text", NLOHMANN_DOUBLES)
def test_json_double_formatting(x, text):
    assert sio._json_double(x) == text


def test_quat_from_matrix_matches_oracle():
    rng = np.random.default_rng(11)
    mats = [np.eye(3), np.diag([1.0, -1.0, -1.0]), np.diag([-1.0, 1.0, -1.0]),
            np.diag([-1.0, -1.0, 1.0])]
    for _ in range(200):
        q = rng.normal(size=4)
        mats.append(O.matrix_from_quat(q / np.linalg.norm(q)))
    for R in mats:
        assert np.array_equal(sio.quat_from_matrix(R), np.asarray(O.quat_from_matrix(R))), R


def _stats(frame=4):
    return dict(frame=frame, skipped=False, valid_pixels=1000, surfel_count=900, node_count=40,
                fused=10, appended=5, removed=1, compressive_rejected=0, low_support_rejected=2,
                new_nodes=3, degenerate_warps=0, gn_iters=10, correspondences=800,
                initial_energy=0.5, final_energy=0.25, mean_residual=0.001, rigid_pairs=700,
                rigid_residual=0.002, rigid_low_confidence=False, reinit=False,
                reinit_removed=0, pose=[1, 0, 0, 0, 1, 0, 0, 0, 1, 0.1, -0.2, 0.0],
                depth_ms=0.5, rigid_ms=1.0, solve_ms=2.0, fusion_ms=0.25, reinit_ms=0.0,
                total_ms=3.75)


def test_metrics_and_timings_lines():
    line = sio.frame_stats_to_json(_stats())
    assert line.startswith('{"frame":4,"skipped":false,"valid_pixels":1000,"surfel_count":900,')
    assert line.endswith('"reinit":false,"reinit_removed":0,"pose":[1.0,0.0,0.0,0.0,0.1,-0.2,0.0]}')
    keys = list(json.loads(line).keys())
    assert keys == ["frame", "skipped"] + list(sio._METRIC_KEYS) + ["pose"]
    assert '"initial_energy":0.5,"final_energy":0.25,"mean_residual":0.001,' in line
    assert sio.frame_stats_to_json({"frame": 3, "skipped": True}) == '{"frame":3,"skipped":true}'
    assert sio.timings_to_json(_stats()) == (
        '{"frame":4,"depth_ms":0.5,"rigid_ms":1.0,"solve_ms":2.0,"fusion_ms":0.25,'
        '"reinit_ms":0.0,"total_ms":3.75}')
    assert " " not in line and "\n" not in line


def test_process_sequence_input_errors(tmp_path):
    cfg = pkg.make_config(**SMALL)
    with pytest.raises(pkg.MissingInput):
        sio.process_sequence(str(tmp_path / "nope"), cfg)
    (tmp_path / "frame-1.png").write_bytes(b"")
    with pytest.raises(pkg.MissingInput):
        sio.process_sequence(str(tmp_path), cfg)


def _write_sequence(d, cfg, scene, frames, corrupt=None):
    seq = pkg.SyntheticSequence(scene, 30, cfg)
    depths = []
    for t in range(frames):
        p = d / f"frame-{t:06d}.png"
        if t == corrupt:
            p.write_bytes(b"\x89PNG\r\n\x1a\ngarbage")
            depths.append(None)
            continue
        depth = seq.render_depth(t)
        sio.write_depth_png(str(p), depth)
        depths.append(depth)
    (d / "notes.txt").write_text("ignored")
    return depths


def test_sequence_frames_decode_to_the_rendered_depth(tmp_path):
    cfg = pkg.make_config(**SMALL)
    depths = _write_sequence(tmp_path, cfg, "bending_sheet", 3)
    for t, dep in enumerate(depths):
        assert np.array_equal(sio.read_depth_png(str(tmp_path / f"frame-{t:06d}.png")), dep)


@pytest.mark.gpu
def test_process_sequence_on_device(tmp_path):
    """process_sequence over PNG frames (one corrupt) on the B200 pipeline:
    the skipped line, one metrics/timings line per frame, PLY exports equal to
    the device model, and frame-0 counts equal to the oracle pipeline's."""
    cfg = pkg.make_config(**SMALL)
    depths = _write_sequence(tmp_path, cfg, "rigid_orbit", 5, corrupt=3)
    out = tmp_path / "out"
    opts = sio.PipelineOptions(output_dir=str(out), ply_every=2, log_nodes=True,
                               debug_dump_maps=True)
    summary = sio.process_sequence(str(tmp_path), cfg, opts)
    assert (summary.frames_processed, summary.frames_skipped) == (4, 1)
    metrics = (out / "metrics.jsonl").read_text().splitlines()
    timings = (out / "timings.jsonl").read_text().splitlines()
    nodes = (out / "nodes.jsonl").read_text().splitlines()
    assert len(metrics) == 5 and len(timings) == 4 and len(nodes) == 4
    assert metrics[3] == '{"frame":3,"skipped":true}'
    recs = [json.loads(m) for m in metrics]
    assert [r["frame"] for r in recs] == [0, 1, 2, 3, 4]
    for r in recs[:3] + recs[4:]:
        assert list(r) == ["frame", "skipped"] + list(sio._METRIC_KEYS) + ["pose"]
    for f in (0, 2, 4):
        assert (out / f"model-{f:06d}.ply").exists()
    assert (out / "debug-normals-000000.png").exists()
    live = sio.read_pointcloud(str(out / "final_live.ply"))
    ref = sio.read_pointcloud(str(out / "final_reference.ply"))
    assert len(live["radii"]) == summary.final_surfel_count == recs[-1]["surfel_count"]
    assert len(ref["radii"]) == summary.final_surfel_count
    assert np.all(np.isfinite(live["positions"]))
    q = np.array(recs[-1]["pose"][:4])
    assert abs(math.sqrt(float(q @ q)) - 1.0) < 1e-12 and q[0] >= 0
    # frame 0 is deterministic: the oracle pipeline reproduces its counts
    ore = O.OraclePipeline(Hh.oracle_cfg(cfg), mirror=True)
    o = ore.process_frame(depths[0], 0)
    assert (recs[0]["valid_pixels"], recs[0]["surfel_count"], recs[0]["node_count"]) == (
        o.valid_pixels, o.surfel_count, o.node_count)
    assert json.loads(nodes[0])["node_count"] == o.node_count


def test_cpp_mirror_writes_the_same_bytes(tmp_path):
    """include/dynsurf_b200.hpp's export_pointcloud / frame_stats_to_json /
    timings_to_json produce the same bytes as sequence_io.py (both restate
    ply_io.cpp:16-37 and pipeline.cpp:144-188)."""
    import os
    import shutil
    import subprocess

    if shutil.which("g++") is None:
        pytest.skip("g++ not available")
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = tmp_path / "formats_check"
    subprocess.run(["g++", "-std=c++17", "-O1", "-I" + os.path.join(repo, "include"),
                    "-I/usr/local/cuda/include", "-o", str(exe),
                    os.path.join(repo, "tests", "cpp", "formats_check.cpp")], check=True)
    live, ref = tmp_path / "live.ply", tmp_path / "ref.ply"
    out = subprocess.run([str(exe), str(live), str(ref)], capture_output=True, text=True,
                         check=True).stdout.splitlines()
    i = np.arange(5)
    pos = np.stack([0.1 * i, -0.25 * i, 1.0 + i / 3.0], 1)
    live_pos = pos.copy()
    live_pos[:, 2] += 1e-7 * i
    nrm = np.tile([0.0, 0.6, -0.8], (5, 1))
    m = dict(ref_pos=pos, ref_nrm=nrm, live_pos=live_pos, live_nrm=nrm,
             radius=0.001 * (i + 1), conf=1.5 * i)
    sio.export_pointcloud(m, "live", str(tmp_path / "py_live.ply"))
    sio.export_pointcloud(m, "reference", str(tmp_path / "py_ref.ply"))
    assert live.read_bytes() == (tmp_path / "py_live.ply").read_bytes()
    assert ref.read_bytes() == (tmp_path / "py_ref.ply").read_bytes()
    st = _stats()
    st.update(rigid_residual=1.0 / 3.0, rigid_ms=1e-5, total_ms=123456789012345.0,
              pose=[0.36, 0.48, -0.8, -0.8, 0.6, 0.0, 0.48, 0.64, 0.6, 0.1, -0.2, 1e-5])
    assert out[0] == sio.frame_stats_to_json(st)
    assert out[1] == sio.timings_to_json(st)
    assert out[2] == '{"frame":4,"skipped":true}'
    xs = [0.0, -0.0, 1.0, 0.1, 1e-05, 0.0001, 1e15, 1.5e300, 5e-324, -2.5e-07, 100.0]
    assert out[3:] == [sio._json_double(x) for x in xs]
