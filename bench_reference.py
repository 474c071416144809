"""`bench.py --impl reference`: the reference algorithm timed on the host cores.

The reference C++ sources cannot be compiled here (Eigen 3, libpng, GTest and
vendored json/CLI11 are absent), so this arm times the CPU
oracle — the fp64 line-by-line restatement in oracle/ — on the same workload,
config and metric as bench.py's B200 arm. Each step is a bounded sample (see
bench.cpu_sample): real per-stage timings plus the dense 6N x 6N LDLT cost
extrapolated from a measured factorisation rate.
"""
from __future__ import annotations

import os
import time

import numpy as np


def run_reference(args):
    import bench

    spec = bench.CONFIGS[args.config]
    if args.config == "cfg3":
        return {"impl": "reference", "unavailable": "config 3 (~8k nodes): the reference's dense "
                "6N x 6N normal equations need ~18 GB and an O((6N)^3) LDLT per LM attempt"}
    cfg = bench.make_cfg(spec)
    warm = max(1, min(args.warmup, 3))
    for _ in range(warm):  # untimed: pages in the oracle and its buffers
        bench.cpu_sample(spec, cfg)
    samples = [bench.cpu_sample(spec, cfg) for _ in range(max(1, min(args.steps, 10)))]
    values = [1.0 / cs["t_frame"] for cs in samples]
    v = float(np.median(values))
    entry = bench.cpu_baseline_entry(samples[-1])
    entry["value"] = round(v, 6)
    return {
        "impl": "reference", "metric": "frames/s", "value": round(v, 6), "unit": "frames/s",
        "n_gpus": args.gpus, "steps": len(values), "warmup": warm, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "data": "synthetic",
        "config": {"workload": f"{args.config}: {spec['scene']} {spec['width']}x{spec['height']}, "
                               f"10 GN x 10 PCG per frame", "device": "host CPU (1 core)"},
        "cpu_baseline": entry,
        "e2e": {"value": round(v, 6), "unit": "frames/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
