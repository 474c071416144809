#!/usr/bin/env python3
"""BASELINE config 4: solver micro-benchmark — GN term evaluation + JtJ block
assembly + block-Jacobi PCG over a node-count sweep (512 ... 16k), plus the
warp kernel at config-3 scale (>= 1M surfels).

Scene: `sine_sheet` (2 cm waves over the whole field of view at 1.2 m, f = 560),
so the image size sets N at ~130 surfels per node.
Frame 0 initialises model + warp field; frame 1 (waves shifted) is the target.

Per N it prints one JSON line with:
  linearize_ms   one GN linearisation (warp, model maps, association, terms,
                 assembly) — CUDA events on the context stream
  pcg10_ms       10 block-Jacobi PCG iterations (cooperative kernel)
  spmv           standalone BSR SpMV, cold L2 (256 MiB flush between calls),
                 algorithmic bytes 148 B/block + 56 B/row -> GB/s and fraction
                 of the measured HBM peak
  assembly       k_assemble_chunks + finish, GB/s over its algorithmic bytes
  forward_warp   full-model warp (96 B/surfel), cold L2
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)


def dims_for(nodes):
    p = 130 * nodes
    w = max(64, int(round(math.sqrt(p * 4 / 3) / 16)) * 16)
    h = max(48, int(round(p / w / 8)) * 8)
    return w, h


def run(nodes, reps, peak):
    import torch
    import paper_1904_13073_b200 as pkg

    W, H = dims_for(nodes)
    cfg = pkg.camera_config(W, H, 560.0, max_nodes=max(8192, int(nodes * 1.5)),
                            max_surfels=2 * W * H, pcg_max_iters=10)
    seq = pkg.SyntheticSequence("sine_sheet", 10, cfg)
    d0, d1 = seq.render_depth(0), seq.render_depth(1)
    ctx = pkg.Context(cfg)
    ctx.process_frame(d0, 0)
    ctx.frame_maps(d1, 1)
    I = np.eye(4)[:3, :3].reshape(9).tolist() + [0.0, 0.0, 0.0]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def cold():
        flush.fill_(1.0)
        torch.cuda.synchronize()

    ne = ctx.build_normal_equations(I, 1, 0)  # warm-up + pattern
    N = ctx.num_nodes()
    S = ctx.model_size()
    B = len(ne["col"])
    ctx.reset_kernel_stats()
    ctx.set_profiling(True)
    for _ in range(reps):
        cold()
        ctx.build_normal_equations(I, 1, 0)
    ks = ctx.kernel_stats()
    ctx.set_profiling(False)
    asm = ks["block_assembly"]
    lin_ms = sum(v["ms"] for k, v in ks.items()) / reps
    # PCG (10 iterations, cooperative kernel)
    diag = [ne["values"][k] for r in range(N) for k in range(ne["row_ptr"][r], ne["row_ptr"][r + 1])
            if ne["col"][k] == r]
    mu = 1e-6 * float(sum(np.trace(b) for b in diag)) / (6 * N)  # the LM floor (solver.cpp:378)
    ctx.reset_kernel_stats()
    ctx.set_profiling(True)
    for _ in range(reps):
        cold()
        ctx.pcg_solve(mu, 10, 0.0)
    pk = ctx.kernel_stats()["pcg"]
    ctx.set_profiling(False)
    # standalone SpMV, cold L2 per call
    x = np.random.default_rng(0).normal(size=6 * N)
    t = []
    for _ in range(reps):
        cold()
        _, ms = ctx.bsr_spmv(x, mu, 1)
        t.append(ms)
    spmv_ms = float(np.median(t))
    spmv_bytes = 148.0 * B + 56.0 * N
    # forward warp of the whole model, cold L2 per call
    ctx.reset_kernel_stats()
    ctx.set_profiling(True)
    for _ in range(reps):
        cold()
        ctx.forward_warp()
    fw = ctx.kernel_stats()["forward_warp"]
    ctx.set_profiling(False)
    ctx.close()

    def rate(v):
        gbs = v["bytes"] / (v["ms"] * 1e-3) / 1e9 if v["ms"] > 0 else 0.0
        return {"ms": round(v["ms"] / max(v["launches"], 1), 4), "gbs": round(gbs, 1),
                "frac": round(gbs / peak, 4), "launches": v["launches"]}

    spmv_gbs = spmv_bytes / (spmv_ms * 1e-3) / 1e9
    return {
        "config": "cfg4", "nodes": N, "surfels": S, "image": f"{W}x{H}", "blocks": B,
        "pairs": ne["n_pairs"], "linearize_ms": round(lin_ms, 4),
        "pcg10_ms": round(pk["ms"] / max(pk["launches"], 1), 4),
        "gn_iter_ms": round(lin_ms + pk["ms"] / max(pk["launches"], 1), 4),
        "spmv": {"ms": round(spmv_ms, 4), "bytes": int(spmv_bytes), "gbs": round(spmv_gbs, 1),
                 "frac": round(spmv_gbs / peak, 4), "l2": "cold (256 MiB flush)"},
        "assembly": rate(asm), "forward_warp": rate(fw), "peak_gbs": peak,
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nodes", type=int, nargs="*", default=[512, 1024, 2048, 4096, 8192, 16384])
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    try:
        peak = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        peak = 6650.0
    for n in args.nodes:
        print(json.dumps(run(n, args.reps, peak)), flush=True)


if __name__ == "__main__":
    main()
