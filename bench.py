#!/usr/bin/env python3
"""Benchmark: SurfelWarp per-frame tracking + fusion on B200 (BASELINE.json metric).

Workload (N=1): BASELINE config 2 — synthetic articulated body, 640x480,
~185k surfels, ~1.5k nodes, 10 GN x 10 PCG per frame. One "step" = one
Pipeline::process_frame on the next frame of the sequence.

  value    frames/s with the depth frames already resident in HBM
           (ds_process_frame_device), CUDA events on the context's stream
           around each step; L2 is flushed (256 MiB write) between steps,
           outside the timed events; total = sum of the K step times.
  e2e      same metric through the public C ABI ds_process_frame with HOST
           depth buffers (H2D of the u16 frame and D2H of the FrameStats
           inside the timed region).
  roofline achieved HBM GB/s of the dominant kernel (algorithmic bytes /
           mean launch time from per-launch CUDA events in a profiled pass).
  cpu_baseline  the reference itself -- its unmodified sources compiled out of
           tree against the repo's Eigen / libpng shims (oracle/_ref; the CPU
           oracle's restatement where that was not built) -- running its own
           Pipeline::process_frame on a bounded sample of the same workload
           (bench_reference.cpu_baseline: cfg2 frame 1 after the init frame).

Multi-GPU: `--gpus N` spawns N processes itself (or runs under torchrun), one
rank per GPU; each rank runs an independent sequence (the scene phase-shifted
by rank), no collective on the data path; the only inter-rank traffic is a
gloo barrier and the max-over-ranks time. value = N*K / max-over-ranks time
("scaling": "weak").

`--impl reference` times the reference on the host cores (oracle/_ref's
Pipeline::process_frame; bench_reference.py) on the same config/metric; rank 0
only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

CFG2 = dict(width=640, height=480, focal=560.0, scene="articulated_body", seq_frames=100)
CFG1 = dict(width=320, height=240, focal=280.0, scene="deforming_sphere", seq_frames=10,
            gn_iters=3)
# BASELINE config 3: large scene with a panning camera (node append + reskinning
# every frame) and an open-to-close contact, 1280x960
# Initial capacities sized for the sequence's peak (9.2 M surfels, 15.2 k nodes)
# with ~2x headroom: the device grows them geometrically at frame boundaries
# when a frame could overflow (ds_capacity), but a growth re-allocates every
# buffer (measured: 120 ms for nodes 16k -> 32k, 0.87 s for surfels 9.8 M ->
# 19.7 M) -- a one-off hitch a real-time user avoids by sizing up front.
CFG3 = dict(width=1280, height=960, focal=1120.0, scene="large_scene", seq_frames=60,
            max_nodes=32768, max_surfels=20_000_000)
CONFIGS = {"cfg1": CFG1, "cfg2": CFG2, "cfg3": CFG3}


def peaks():
    try:
        return json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "source": "fallback"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def make_cfg(spec, **kw):
    import paper_1904_13073_b200 as pkg

    for k in ("max_nodes", "max_surfels"):
        if k in spec:
            kw.setdefault(k, spec[k])
    return pkg.camera_config(spec["width"], spec["height"], spec["focal"],
                             max_gn_iters=spec.get("gn_iters", 10), pcg_max_iters=10, **kw)


def render_frames(spec, cfg, n, phase):
    import paper_1904_13073_b200 as pkg

    seq = pkg.SyntheticSequence(spec["scene"], spec["seq_frames"] + phase, cfg)
    return [seq.render_depth((phase + t) % seq.frame_count()) for t in range(n)]


def run_b200(args, rank, world, local_rank):
    import torch
    import paper_1904_13073_b200 as pkg

    torch.cuda.set_device(local_rank)
    spec = CONFIGS[args.config]
    cfg = make_cfg(spec)
    K, W = args.steps, args.warmup
    frames = render_frames(spec, cfg, 1 + W + K, phase=3 * rank)
    stream = torch.cuda.current_stream()
    dev = torch.device("cuda", local_rank)
    # depth frames resident in HBM (u16 stored in int16 tensors)
    d_frames = torch.stack([torch.from_numpy(f.view(np.int16)) for f in frames]).to(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def ptr(t):
        return d_frames[t].data_ptr()

    # ---------------- device-resident pass (value)
    ctx = pkg.Context(cfg, local_rank, stream.cuda_stream)
    for t in range(1 + W):
        ctx.process_frame_device(ptr(t), t)
    torch.cuda.synchronize()
    dist_barrier(world)
    launches0 = ctx.total_launches()
    step_ms, stats = [], []
    with ClockSampler(local_rank) as clk:
        for t in range(1 + W, 1 + W + K):
            flush.fill_(float(t))  # L2 flush outside the timed events
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            st = ctx.process_frame_device(ptr(t), t)
            ctx.join_deferred()  # the frame's side-stream node / reskin work is timed too
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            stats.append(pkg.stats_to_dict(st))
    torch.cuda.synchronize()
    launches = ctx.total_launches() - launches0
    total_ms = sum(step_ms)
    total_ms = dist_max(total_ms, world)
    dist_barrier(world)

    # ---------------- end-to-end pass through the host-buffer C ABI (e2e)
    pipe = pkg.Pipeline(cfg, local_rank, stream.cuda_stream)
    for t in range(1 + W):
        pipe.process_frame(frames[t], t)
    torch.cuda.synchronize()
    dist_barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for t in range(1 + W, 1 + W + K):
        pipe.process_frame(frames[t], t)
    pipe.context.join_deferred()
    e1.record(stream)
    e1.synchronize()
    e2e_ms = dist_max(e0.elapsed_time(e1), world)
    pipe.close()

    # ---------------- the frames the CPU reference arm times (1..3 after the
    # init frame; bench_reference.py), end to end as above
    n_ref = min(3, len(frames) - 1)
    rp = pkg.Pipeline(cfg, local_rank, stream.cuda_stream)
    rp.process_frame(frames[0], 0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for t in range(1, 1 + n_ref):
        rp.process_frame(frames[t], t)
    rp.context.join_deferred()
    e1.record(stream)
    e1.synchronize()
    ref_frames_ms = e0.elapsed_time(e1)
    rp.close()

    # ---------------- profiled pass (per-kernel CUDA events) for the roofline
    prof = pkg.Context(cfg, local_rank, stream.cuda_stream)
    for t in range(1 + W):
        prof.process_frame_device(ptr(t), t)
    prof.reset_kernel_stats()
    # profile every 8th timed frame so the per-kernel shares cover the whole run
    for t in range(1 + W, 1 + W + K):
        on = (t - 1 - W) % 8 == 0
        prof.set_profiling(on)
        prof.process_frame_device(ptr(t), t)
    prof.set_profiling(False)
    ks = prof.kernel_stats()
    prof.close()
    ctx.close()
    return dict(K=K, W=W, total_ms=total_ms, step_ms=step_ms, stats=stats, launches=launches,
                e2e_ms=e2e_ms, ref_frames=(n_ref, ref_frames_ms), kernels=ks, clocks=clk.summary(), spec=spec, cfg=cfg,
                bytes_in=frames[0].nbytes)


def run_multi(args, rank, world, local_rank):
    """BASELINE config 5: `--sequences S` independent cfg2 sequences per GPU, one
    context + CUDA stream + host thread each (ctypes releases the GIL). The PCG's
    cooperative grid is divided among the S contexts so their solves co-reside.
    Timing: a start event every stream waits on, one end event per stream; the
    job time is the max over streams (and over ranks)."""
    import torch
    import paper_1904_13073_b200 as pkg

    S, K, W = args.sequences, args.steps, args.warmup
    torch.cuda.set_device(local_rank)
    sms = torch.cuda.get_device_properties(local_rank).multi_processor_count
    # measured (S = 8, 16): a quarter of the SMs per PCG beats an even split
    # (418 / 424 vs 385 / 393 aggregate frames/s) -- solves rarely coincide
    os.environ.setdefault("DS_PCG_GRID", str(max(sms // 4, sms // S)))
    spec = CFG2
    cfg = make_cfg(spec)
    seq = pkg.SyntheticSequence(spec["scene"], spec["seq_frames"], cfg)
    F = seq.frame_count()
    frames = [seq.render_depth(t) for t in range(F)]
    dev = torch.device("cuda", local_rank)
    d_frames = torch.stack([torch.from_numpy(f.view(np.int16)) for f in frames]).to(dev)
    phase = [(3 * (rank * S + s)) % F for s in range(S)]
    streams = [torch.cuda.Stream(device=dev) for _ in range(S)]

    def frame_ptr(s, t):
        return d_frames[(phase[s] + t) % F].data_ptr()

    def run_threads(fn):
        ths = [threading.Thread(target=fn, args=(s,)) for s in range(S)]
        for th in ths:
            th.start()
        for th in ths:
            th.join()

    def timed(fn_frame, objs):
        start = torch.cuda.Event(enable_timing=True)
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(S)]
        torch.cuda.synchronize()
        dist_barrier(world)
        start.record(torch.cuda.current_stream())
        for st in streams:
            st.wait_event(start)

        def loop(s):
            for t in range(1 + W, 1 + W + K):
                fn_frame(objs[s], s, t)
            ends[s].record(streams[s])

        run_threads(loop)
        torch.cuda.synchronize()
        return dist_max(max(start.elapsed_time(e) for e in ends), world)

    # device-resident pass
    ctxs = [pkg.Context(cfg, local_rank, streams[s].cuda_stream) for s in range(S)]
    run_threads(lambda s: [ctxs[s].process_frame_device(frame_ptr(s, t), t) for t in range(1 + W)])
    launches0 = sum(c.total_launches() for c in ctxs)
    with ClockSampler(local_rank) as clk:
        total_ms = timed(lambda c, s, t: c.process_frame_device(frame_ptr(s, t), t), ctxs)
    launches = sum(c.total_launches() for c in ctxs) - launches0
    surfels = [c.model_size() for c in ctxs]
    for c in ctxs:
        c.close()
    # end-to-end pass: host depth buffers through the C ABI
    pipes = [pkg.Pipeline(cfg, local_rank, streams[s].cuda_stream) for s in range(S)]
    run_threads(lambda s: [pipes[s].process_frame(frames[(phase[s] + t) % F], t)
                           for t in range(1 + W)])
    e2e_ms = timed(lambda p, s, t: p.process_frame(frames[(phase[s] + t) % F], t), pipes)
    for p in pipes:
        p.close()
    return dict(total_ms=total_ms, e2e_ms=e2e_ms, launches=launches, clocks=clk.summary(),
                surfels=surfels, bytes_in=frames[0].nbytes, pcg_grid=os.environ["DS_PCG_GRID"])


def roofline(ks, peak_gbs, config="cfg2"):
    rows = {}
    for name, v in ks.items():
        if v["launches"] and v["ms"] > 0:
            rows[name] = dict(launches=v["launches"], ms=v["ms"], bytes=v["bytes"],
                              gbs=v["bytes"] / (v["ms"] * 1e-3) / 1e9)
    dom = max(rows, key=lambda n: rows[n]["ms"]) if rows else None
    out = None
    traffic, traffic_src = None, None
    for name in ("r02_traffic.json", "r01_traffic.json"):  # newest ncu capture first
        try:  # ncu-measured DRAM bytes per launch of the same kernel (profiles/)
            t = json.load(open(os.path.join(REPO, "profiles", name)))
        except Exception:
            continue
        if dom in t and t.get("config", "cfg2") == config:  # captured on this workload only
            traffic, traffic_src = t[dom]["bytes_per_launch"], f"profiles/{name}: {t['source']}"
            break
    if dom:
        r = rows[dom]
        out = {"kernel": dom, "bound": "hbm", "achieved": round(r["gbs"], 1), "peak": peak_gbs,
               "unit": "GB/s", "frac": round(r["gbs"] / peak_gbs, 4), "traffic": traffic,
               "traffic_source": traffic_src,
               "mean_launch_us": round(1e3 * r["ms"] / r["launches"], 2),
               "algorithmic_bytes_per_launch": round(r["bytes"] / r["launches"])}
    per = {n: {"gbs": round(r["gbs"], 1), "frac": round(r["gbs"] / peak_gbs, 4),
               "ms_share": round(r["ms"] / sum(x["ms"] for x in rows.values()), 4),
               "mean_launch_us": round(1e3 * r["ms"] / r["launches"], 2)}
           for n, r in sorted(rows.items(), key=lambda kv: -kv[1]["ms"])}
    return out, per


def dist_barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def dist_max(v, world):
    """Max over ranks (the timing rule: the slowest rank defines the job time).
    Host-side gloo on a CPU tensor: the ranks' sequences are independent, so
    nothing on the data path is a collective and no NCCL communicator exists."""
    if world <= 1:
        return v
    import torch
    import torch.distributed as dist

    t = torch.tensor([v], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_fps(world, steps, max_total_ms):
    """Whole-job throughput: every rank processed `steps` frames of its own sequence."""
    return world * steps / (max_total_ms * 1e-3)


def dryrun(args, rank, world):
    """DS_BENCH_DRYRUN=1 (CPU tests only): the launcher, rendezvous, barrier and
    max-over-ranks timing of the N-rank path with a host sleep standing in for
    the per-frame work (rank r sleeps (1 + r) ms per step). Prints a line marked
    "dryrun" -- never a measurement."""
    dist_barrier(world)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        time.sleep(1e-3 * (1 + rank))
    ms = dist_max(1e3 * (time.perf_counter() - t0), world)
    dist_barrier(world)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"dryrun": True, "metric": "frames/s", "n_gpus": world,
                          "steps": args.steps, "value": aggregate_fps(world, args.steps, ms),
                          "max_rank_ms": ms}), flush=True)


def spawn_ranks(n):
    """`bench.py --gpus N` without a launcher: one process per GPU (RANK /
    LOCAL_RANK / WORLD_SIZE set as torchrun would), gloo rendezvous on
    127.0.0.1; rank 0 prints the JSON line. Returns the worst exit code."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n),
                   LOCAL_WORLD_SIZE=str(n), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + sys.argv[1:],
                                      env=env))
    return max(p.wait() for p in procs)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=94)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="cfg2", choices=["cfg2", "cfg1", "cfg3"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sequences", type=int, default=1,
                    help="independent cfg2 sequences per GPU (BASELINE config 5)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    args.warmup = max(args.warmup, 3)
    # one step = one frame of the config's sequence: warm-up + timed frames stay
    # within its length
    spec = CONFIGS[args.config]
    args.steps = max(1, min(args.steps, spec["seq_frames"] - 1 - args.warmup,
                            spec.get("max_steps", args.steps)))
    if args.impl == "reference":
        if rank == 0:
            from bench_reference import run_reference

            print(json.dumps(run_reference(args)), flush=True)
        return
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("gloo")  # barrier + max-over-ranks timing only
    if os.environ.get("DS_BENCH_DRYRUN") == "1":
        return dryrun(args, rank, world)
    if args.sequences > 1:
        r = run_multi(args, rank, world, local_rank)
        if world > 1:
            import torch.distributed as dist

            dist.barrier()
            dist.destroy_process_group()
        if rank == 0:
            S, K = args.sequences, args.steps
            line = {
                "metric": "frames/s", "value": round(world * S * K / (r["total_ms"] * 1e-3), 3),
                "unit": "frames/s", "n_gpus": world, "steps": K, "warmup": args.warmup,
                "ms_per_step": round(r["total_ms"] / K, 3), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None,
                "dtype": "f64+f32", "storage": "fp64 arithmetic; fp32 SoA surfels, fp64 nodes, fp32 JtJ blocks",
                "data": "synthetic",
                "config": {"workload": f"cfg5: {S} independent cfg2 sequences per GPU "
                                       f"(articulated_body 640x480, phase-shifted), 10 GN x 10 PCG",
                           "sequences_per_gpu": S, "pcg_ctas_per_context": int(r["pcg_grid"]),
                           "surfels_per_sequence_end": [min(r["surfels"]), max(r["surfels"])],
                           "l2": "inputs resident, no flush (S streams share L2)",
                           "parallelism": f"{S} streams x {world} GPUs, no collective"},
                "e2e": {"value": round(world * S * K / (r["e2e_ms"] * 1e-3), 3), "unit": "frames/s",
                        "h2d_bytes_per_step": S * r["bytes_in"], "d2h_bytes_per_step": S * 360},
                "gpu_launches": int(r["launches"]), "roofline": None, "clocks": r["clocks"],
            }
            print(json.dumps(line), flush=True)
        return
    r = run_b200(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()
    if rank != 0:
        return
    pk = peaks()
    K = r["K"]
    value = aggregate_fps(world, K, r["total_ms"])
    e2e = aggregate_fps(world, K, r["e2e_ms"])
    roof, per = roofline(r["kernels"], pk.get("hbm_gbs", 6650.0), args.config)
    st = r["stats"]
    solve_ms = float(np.mean([s["solve_ms"] for s in st]))
    gn_iters = float(np.mean([s["gn_iters"] for s in st]))
    line = {
        "metric": "frames/s", "value": round(value, 3), "unit": "frames/s", "n_gpus": world,
        "steps": K, "warmup": args.warmup, "ms_per_step": round(r["total_ms"] / K, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64+f32", "storage": "fp64 arithmetic; fp32 SoA surfels, fp64 nodes, fp32 JtJ blocks",
        "data": "synthetic",
        "config": {"workload": f"{args.config}: {r['spec']['scene']} {r['cfg']['width']}x"
                               f"{r['cfg']['height']}, {r['spec'].get('gn_iters', 10)} GN x 10 PCG "
                               f"per frame",
                   "surfels": st[-1]["surfel_count"], "nodes": st[-1]["node_count"],
                   "frames_per_rank": K, "l2": "flushed between steps (256 MiB write, untimed)",
                   "surfels_range": [min(s["surfel_count"] for s in st), max(s["surfel_count"] for s in st)],
                   "correspondences_mean": round(float(np.mean([s["correspondences"] for s in st]))),
                   "parallelism": f"independent sequences, 1 per GPU x {world}",
                   **({"initial_capacity": {k: r["spec"][k] for k in ("max_surfels", "max_nodes")
                                            if k in r["spec"]}}
                      if any(k in r["spec"] for k in ("max_surfels", "max_nodes")) else {})},
        "e2e": {"value": round(e2e, 3), "unit": "frames/s", "h2d_bytes_per_step": r["bytes_in"],
                "d2h_bytes_per_step": 360},
        "gpu_launches": int(r["launches"]),
        "reference_frames": {"frames": list(range(1, 1 + r["ref_frames"][0])),
                             "e2e_fps": round(r["ref_frames"][0] / (r["ref_frames"][1] * 1e-3), 3),
                             "note": "frames the --impl reference arm times (rank 0, phase 0)"},
        "solve_ms": round(solve_ms, 3), "gn_iters_per_frame": round(gn_iters, 2),
        "ms_per_gn_iter": round(solve_ms / max(gn_iters, 1e-9), 3),
        "roofline": roof, "kernels": per, "clocks": r["clocks"],
    }
    if args.config == "cfg3":
        line["cpu_baseline"] = {"value": None, "unit": "frames/s", "cores": 1, "kind": "port",
                                "sample": "n/a: the reference's dense 6N x 6N system at ~8k nodes "
                                          "needs ~18 GB (SURVEY 8(d))"}
    elif world > 1:  # the CPU sample runs at N = 1 only
        line["cpu_baseline"] = {"value": None, "unit": "frames/s", "cores": 0, "kind": "port",
                                "sample": "measured in the N = 1 run only"}
    elif not args.no_cpu_baseline:
        try:
            from bench_reference import cpu_baseline

            line["cpu_baseline"] = cpu_baseline(args, r["spec"], r["cfg"])
        except Exception as e:  # never fail the GPU line on the CPU sample
            line["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
