"""On-disk and log formats around the per-frame path.

Host-side I/O that lets a directory of depth frames run through the B200
pipeline exactly as the reference's `process_sequence` runs it:

  depth PNG ingest / export   png_io.hpp:10-15, png_io.cpp (16-bit grayscale,
                              big-endian samples, 0 = invalid); decoded here
                              with zlib + the five PNG row filters because
                              libpng headers are absent from the image
  binary PLY export / import  ply_io.hpp:12-26, ply_io.cpp:10-95 (byte-identical
                              header, 8 little-endian doubles per vertex)
  metrics.jsonl line          pipeline.cpp:144-174 `frame_stats_to_json`
                              (nlohmann::ordered_json::dump formatting)
  timings.jsonl line          pipeline.cpp:178-188 `timings_to_json`
  process_sequence            pipeline.cpp:205-291 (frame-%06d.png discovery,
                              CorruptFrame skip, nodes.jsonl, PLY cadence)

None of this is on the device path: the frames are decoded on the host and
handed to `Pipeline.process_frame` (the C ABI's host-buffer entry point).
"""
from __future__ import annotations

import math
import os
import re
import struct
import sys
import zlib
from dataclasses import dataclass
from decimal import Decimal

import numpy as np

from .errors import CorruptFrame, EmptyGeometry, IoFailure, MissingInput

_PNG_SIG = b"\x89PNG\r\n\x1a\n"

# --------------------------------------------------------------------------- PNG


def _chunk(tag: bytes, data: bytes) -> bytes:
    return struct.pack(">I", len(data)) + tag + data + struct.pack(
        ">I", zlib.crc32(tag + data) & 0xFFFFFFFF)


def _unfilter(data: bytes, width: int, height: int, bpp: int) -> np.ndarray:
    """PNG row filters reversed by the native library (ds_png_unfilter, PNG
    spec 9.2: the Average / Paeth filters libpng writes by default are
    sequential along a row)."""
    from . import _lib

    stride = width * bpp
    if len(data) != height * (stride + 1):
        raise CorruptFrame("PNG image data has the wrong size")
    src = np.frombuffer(data, np.uint8)
    out = np.empty((height, stride), np.uint8)
    rc = _lib.load().ds_png_unfilter(src.ctypes.data, src.size, width, height, bpp,
                                     out.ctypes.data)
    if rc != 0:
        raise CorruptFrame("PNG row filter is invalid")
    return out


def read_depth_png(path: str) -> np.ndarray:
    """`read_depth_png` (png_io.cpp): a (H, W) uint16 depth image in millimetres.

    Same errors as the reference: IoFailure when the file cannot be opened,
    CorruptFrame for a bad signature, a non 16-bit grayscale image, or damaged
    chunk / zlib data (libpng's longjmp path). Interlaced images are rejected
    as corrupt (the reference's writer never produces them).
    """
    try:
        with open(path, "rb") as f:
            blob = f.read()
    except OSError:
        raise IoFailure("cannot open PNG: " + path) from None
    if blob[:8] != _PNG_SIG:
        raise CorruptFrame("not a PNG file: " + path)
    pos, idat, ihdr = 8, [], None
    try:
        while True:
            if pos + 8 > len(blob):
                raise CorruptFrame("corrupt PNG: " + path)
            (n,), tag = struct.unpack(">I", blob[pos:pos + 4]), blob[pos + 4:pos + 8]
            data = blob[pos + 8:pos + 8 + n]
            crc = blob[pos + 8 + n:pos + 12 + n]
            if len(data) != n or len(crc) != 4 or struct.unpack(">I", crc)[0] != (
                    zlib.crc32(tag + data) & 0xFFFFFFFF):
                raise CorruptFrame("corrupt PNG: " + path)
            pos += 12 + n
            if tag == b"IHDR":
                ihdr = struct.unpack(">IIBBBBB", data)
            elif tag == b"IDAT":
                idat.append(data)
            elif tag == b"IEND":
                break
        if ihdr is None:
            raise CorruptFrame("corrupt PNG: " + path)
        width, height, bit_depth, color_type, _comp, _filt, interlace = ihdr
        if bit_depth != 16 or color_type != 0:
            raise CorruptFrame("expected 16-bit grayscale PNG: " + path)
        if interlace != 0 or width == 0 or height == 0:
            raise CorruptFrame("corrupt PNG: " + path)
        raw = zlib.decompress(b"".join(idat))
    except (struct.error, zlib.error):
        raise CorruptFrame("corrupt PNG: " + path) from None
    img = _unfilter(raw, width, height, 2)
    # PNG stores 16-bit samples big-endian (png_set_swap in the reference).
    return img.view(">u2").reshape(height, width).astype(np.uint16)


def write_depth_png(path: str, depth) -> None:
    """`write_depth_png` (png_io.cpp): 16-bit grayscale, samples big-endian."""
    d = np.ascontiguousarray(depth, dtype=np.uint16)
    if d.ndim != 2:
        raise IoFailure("write_depth_png expects a (H, W) image")
    h, w = d.shape
    rows = np.zeros((h, 1 + 2 * w), np.uint8)  # filter byte 0 per row
    rows[:, 1:] = d.astype(">u2").view(np.uint8).reshape(h, 2 * w)
    _write_png(path, w, h, 16, 0, rows.tobytes())


def write_rgb_png(path: str, image) -> None:
    """`write_rgb_png` (png_io.hpp:14): 8-bit RGB, used for debug map dumps."""
    im = np.ascontiguousarray(image, dtype=np.uint8)
    h, w = im.shape[:2]
    rows = np.zeros((h, 1 + 3 * w), np.uint8)
    rows[:, 1:] = im.reshape(h, 3 * w)
    _write_png(path, w, h, 8, 2, rows.tobytes())


def _write_png(path, w, h, bit_depth, color_type, filtered: bytes) -> None:
    blob = (_PNG_SIG + _chunk(b"IHDR", struct.pack(">IIBBBBB", w, h, bit_depth, color_type,
                                                    0, 0, 0))
            + _chunk(b"IDAT", zlib.compress(filtered, 6)) + _chunk(b"IEND", b""))
    try:
        with open(path, "wb") as f:
            f.write(blob)
    except OSError:
        raise IoFailure("cannot create PNG: " + path) from None


# --------------------------------------------------------------------------- PLY

_PLY_PROPS = ("x", "y", "z", "nx", "ny", "nz", "radius", "confidence")  # ply_io.cpp:11


def export_pointcloud(model: dict, side: str, path: str) -> None:
    """`export_pointcloud` (ply_io.cpp:16-37). `model` is `Pipeline.model()`;
    side is "reference" or "live". Header and records byte-identical."""
    if side not in ("reference", "live"):
        raise ValueError("side must be 'reference' or 'live'")
    pre = "ref" if side == "reference" else "live"
    n = len(model["radius"])
    if n == 0:
        raise EmptyGeometry("export_pointcloud: empty model")
    rec = np.empty((n, 8), "<f8")
    rec[:, 0:3] = model[pre + "_pos"]
    rec[:, 3:6] = model[pre + "_nrm"]
    rec[:, 6] = model["radius"]
    rec[:, 7] = model["conf"]
    head = ("ply\nformat binary_little_endian 1.0\n" f"element vertex {n}\n"
            + "".join(f"property double {p}\n" for p in _PLY_PROPS) + "end_header\n")
    try:
        with open(path, "wb") as f:
            f.write(head.encode("ascii"))
            f.write(rec.tobytes())
    except OSError:
        raise IoFailure("cannot create PLY: " + path) from None


def read_pointcloud(path: str) -> dict:
    """`read_pointcloud` (ply_io.cpp:39-93): positions, normals, radii,
    confidences; IoFailure on every header / size violation the reference
    rejects."""
    try:
        with open(path, "rb") as f:
            blob = f.read()
    except OSError:
        raise IoFailure("cannot open PLY: " + path) from None
    pos = 0

    def line():
        nonlocal pos
        e = blob.find(b"\n", pos)
        if e < 0:
            return None
        s = blob[pos:e].decode("latin-1")
        pos = e + 1
        return s

    if line() != "ply":
        raise IoFailure("not a PLY file: " + path)
    count, prop, done = 0, 0, False
    while True:
        s = line()
        if s is None:
            break
        tok = s.split()
        head = tok[0] if tok else ""
        if head == "format":
            if len(tok) < 2 or tok[1] != "binary_little_endian":
                raise IoFailure("unsupported PLY format in " + path)
        elif head == "element":
            if len(tok) < 3 or tok[1] != "vertex":
                raise IoFailure("unsupported PLY element in " + path)
            count = int(tok[2])
        elif head == "property":
            if (len(tok) < 3 or tok[1] != "double" or prop >= 8
                    or tok[2] != _PLY_PROPS[prop]):
                raise IoFailure("unexpected PLY property in " + path)
            prop += 1
        elif head == "end_header":
            done = True
            break
        elif head == "comment":
            continue
        else:
            raise IoFailure("unexpected PLY header line in " + path)
    if not done or prop != 8:
        raise IoFailure("malformed PLY header in " + path)
    body = blob[pos:pos + count * 64]
    if len(body) != count * 64:
        raise IoFailure("truncated PLY: " + path)
    rec = np.frombuffer(body, "<f8").reshape(count, 8).astype(np.float64)
    return dict(positions=rec[:, 0:3].copy(), normals=rec[:, 3:6].copy(),
                radii=rec[:, 6].copy(), confidences=rec[:, 7].copy())


# --------------------------------------------------------------------------- JSON lines


def _json_double(x: float) -> str:
    """nlohmann::json's double serialisation: shortest round-trip digits laid
    out by its `format_buffer` (min_exp = -4, max_exp = 15), non-finite -> null."""
    x = float(x)
    if not math.isfinite(x):
        return "null"
    if x == 0.0:
        return "-0.0" if math.copysign(1.0, x) < 0 else "0.0"
    sign = "-" if x < 0 else ""
    _, dg, exp = Decimal(repr(abs(x))).normalize().as_tuple()  # shortest round-trip digits
    digits = "".join(map(str, dg))
    n = len(digits) + exp  # decimal point position relative to the digit string
    k = len(digits)
    if k <= n <= 15:
        s = digits + "0" * (n - k) + ".0"
    elif 0 < n <= 15:
        s = digits[:n] + "." + digits[n:]
    elif -4 < n <= 0:
        s = "0." + "0" * (-n) + digits
    else:
        e = n - 1
        s = (digits if k == 1 else digits[0] + "." + digits[1:]) + "e" + (
            "-" if e < 0 else "+") + f"{abs(e):02d}"
    return sign + s


def _json_value(v) -> str:
    if isinstance(v, bool):
        return "true" if v else "false"
    if isinstance(v, (int, np.integer)):
        return str(int(v))
    if isinstance(v, (float, np.floating)):
        return _json_double(v)
    if isinstance(v, (list, tuple, np.ndarray)):
        return "[" + ",".join(_json_value(e) for e in v) + "]"
    if isinstance(v, str):
        return '"' + v.replace("\\", "\\\\").replace('"', '\\"') + '"'
    raise TypeError(f"cannot serialise {type(v)!r}")


def _json_object(pairs) -> str:
    return "{" + ",".join(f'"{k}":{_json_value(v)}' for k, v in pairs) + "}"


def quat_from_matrix(r) -> np.ndarray:
    """`quat_from_matrix` (geometry.cpp:44-50): Eigen's Shepperd branch order,
    normalised, w >= 0; returns (w, x, y, z)."""
    m = np.asarray(r, np.float64).reshape(3, 3)
    q = [0.0, 0.0, 0.0, 0.0]
    t = (m[0, 0] + m[1, 1]) + m[2, 2]
    if t > 0.0:
        t = math.sqrt(t + 1.0)
        q[0] = 0.5 * t
        t = 0.5 / t
        q[1] = (m[2, 1] - m[1, 2]) * t
        q[2] = (m[0, 2] - m[2, 0]) * t
        q[3] = (m[1, 0] - m[0, 1]) * t
    else:
        i = 0
        if m[1, 1] > m[0, 0]:
            i = 1
        if m[2, 2] > m[i, i]:
            i = 2
        j = (i + 1) % 3
        k = (j + 1) % 3
        t = math.sqrt(m[i, i] - m[j, j] - m[k, k] + 1.0)
        q[1 + i] = 0.5 * t
        t = 0.5 / t
        q[0] = (m[k, j] - m[j, k]) * t
        q[1 + j] = (m[j, i] + m[i, j]) * t
        q[1 + k] = (m[k, i] + m[i, k]) * t
    nrm = math.sqrt(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3])
    q = [c / nrm for c in q]
    if q[0] < 0:
        q = [-c for c in q]
    return np.array(q)


_METRIC_KEYS = ("valid_pixels", "surfel_count", "node_count", "fused", "appended", "removed",
                "compressive_rejected", "low_support_rejected", "new_nodes",
                "degenerate_warps", "gn_iters", "correspondences", "initial_energy",
                "final_energy", "mean_residual", "rigid_pairs", "rigid_residual",
                "rigid_low_confidence", "reinit", "reinit_removed")
_FLOAT_KEYS = ("initial_energy", "final_energy", "mean_residual", "rigid_residual")


def frame_stats_to_json(stats: dict) -> str:
    """`frame_stats_to_json` (pipeline.cpp:144-174) for a `Pipeline.process_frame`
    dict: same keys, order and number formatting as the reference's line."""
    pairs = [("frame", int(stats["frame"])), ("skipped", bool(stats["skipped"]))]
    if stats["skipped"]:
        return _json_object(pairs)
    for k in _METRIC_KEYS:
        v = stats[k]
        pairs.append((k, float(v) if k in _FLOAT_KEYS else v))
    pose = np.asarray(stats["pose"], np.float64)
    q = quat_from_matrix(pose[:9])
    pairs.append(("pose", [float(c) for c in q] + [float(c) for c in pose[9:12]]))
    return _json_object(pairs)


def timings_to_json(stats: dict) -> str:
    """`timings_to_json` (pipeline.cpp:178-188)."""
    return _json_object([("frame", int(stats["frame"]))] + [
        (k, float(stats[k])) for k in ("depth_ms", "rigid_ms", "solve_ms", "fusion_ms",
                                        "reinit_ms", "total_ms")])


# --------------------------------------------------------------------------- sequences


@dataclass
class PipelineOptions:
    """`PipelineOptions` (pipeline.hpp:64-69)."""
    output_dir: str = ""
    ply_every: int = 10  # also exports the final model; 0 = final only, -1 = never
    log_nodes: bool = False
    debug_dump_maps: bool = False


@dataclass
class SequenceSummary:
    """`SequenceSummary` (pipeline.hpp:71-76)."""
    frames_processed: int = 0
    frames_skipped: int = 0
    reinit_count: int = 0
    final_surfel_count: int = 0


_FRAME_RE = re.compile(r"frame-([0-9]{6})\.png")


def _skipped(index: int) -> dict:
    return {"frame": index, "skipped": True}


def process_sequence(input_dir: str, cfg: dict, options: PipelineOptions | None = None,
                     device: int = 0) -> SequenceSummary:
    """`process_sequence` (pipeline.cpp:205-291) over the B200 pipeline."""
    from .pipeline import Pipeline

    options = options or PipelineOptions()
    if not os.path.isdir(input_dir):
        raise MissingInput("not a directory: " + input_dir)
    frames = []
    for name in os.listdir(input_dir):
        full = os.path.join(input_dir, name)
        m = _FRAME_RE.fullmatch(name)
        if m and os.path.isfile(full):
            frames.append((int(m.group(1)), full))
    if not frames:
        raise MissingInput("no frame-%06d.png files in " + input_dir)
    frames.sort()
    out_dir = options.output_dir or os.path.join(input_dir, "out")
    try:
        os.makedirs(out_dir, exist_ok=True)
    except OSError:
        raise IoFailure("cannot create output directory: " + out_dir) from None
    try:
        metrics = open(os.path.join(out_dir, "metrics.jsonl"), "w")
        timings = open(os.path.join(out_dir, "timings.jsonl"), "w")
        nodes_log = open(os.path.join(out_dir, "nodes.jsonl"), "w") if options.log_nodes else None
    except OSError:
        raise IoFailure("cannot open log files in " + out_dir) from None

    summary = SequenceSummary()
    pipe = Pipeline(cfg, device)
    try:
        for index, path in frames:
            try:
                depth = read_depth_png(path)
                if depth.shape != (cfg["height"], cfg["width"]):
                    raise CorruptFrame("frame size mismatch: " + path)
                stats = pipe.process_frame(depth, index)
            except CorruptFrame as err:
                print(f"warning: skipping frame {index}: {err}", file=sys.stderr)
                summary.frames_skipped += 1
                metrics.write(frame_stats_to_json(_skipped(index)) + "\n")
                continue
            summary.frames_processed += 1
            summary.reinit_count += int(bool(stats["reinit"]))
            metrics.write(frame_stats_to_json(stats) + "\n")
            timings.write(timings_to_json(stats) + "\n")
            if nodes_log is not None:
                pos = pipe.nodes()["pos"]
                nodes_log.write(_json_object([
                    ("frame", int(stats["frame"])), ("node_count", int(len(pos))),
                    ("positions", [[float(c) for c in p] for p in pos])]) + "\n")
            if options.debug_dump_maps:
                f = pipe.context.download_frame()
                rgb = np.zeros(f["nrm"].shape, np.uint8)
                v = f["valid"].astype(bool)
                rgb[v] = (127.5 * (f["nrm"][v] + 1.0)).astype(np.uint8)
                write_rgb_png(os.path.join(out_dir, f"debug-normals-{index:06d}.png"), rgb)
            if options.ply_every > 0 and index % options.ply_every == 0:
                model = pipe.model()
                if len(model["radius"]) > 0:
                    export_pointcloud(model, "live",
                                      os.path.join(out_dir, f"model-{index:06d}.ply"))
        model = pipe.model()
        if options.ply_every >= 0 and len(model["radius"]) > 0:
            export_pointcloud(model, "live", os.path.join(out_dir, "final_live.ply"))
            export_pointcloud(model, "reference", os.path.join(out_dir, "final_reference.ply"))
        summary.final_surfel_count = int(len(model["radius"]))
    finally:
        metrics.close()
        timings.close()
        if nodes_log is not None:
            nodes_log.close()
        pipe.close()
    return summary
