"""CPU reference timing for bench.py: `--impl reference` and the `cpu_baseline` leg.

The reference itself runs here: `oracle/_ref/libdynsurf_ref.so` is the
UNMODIFIED reference (/root/reference/proj/core/src) compiled out of tree
against the repo's shims for its absent dependencies (an Eigen subset, a
libpng stub; `make -C oracle ref`; its own 106 unit
tests pass on that build, tests/test_ref_oracle.py). It is driven through its
own `Pipeline::process_frame` (pipeline.cpp:74-142) frame by frame -- frame
maps, model maps + rigid ICP, the full Levenberg-Marquardt loop with a dense
6N x 6N system per GN iteration (solver.cpp:296-420), forward warp, fusion,
reinit checks. Nothing is extrapolated: every timed frame is one real
process_frame call, wall-clocked on the host. (Where oracle/_ref was not
built, the same timing runs through the oracle's restatement, kind "port".)

Threads. The reference is single-threaded (no threads / OpenMP anywhere).
  * config 1 runs exactly that: 1 core, the LDLT of the Eigen shim.
  * config 2's LM step is a dense LDLT of a ~9.2k x 9.2k matrix (648 MB) per
    attempt -- about 70 s on one core, ~12 min per frame. To finish in minutes,
    the reference arm hands that one step to LAPACK's Cholesky (scipy's
    OpenBLAS dpotrf/dpotrs on all host threads; dsysv if the Cholesky fails).
    Everything else stays single-threaded as in the reference. This can only
    make the reference arm faster than the shipped reference, i.e. the B200 /
    reference ratio it yields is conservative.

Input frames come from the host-only scene library (synth/), so this arm never
maps the product CUDA library.
"""
from __future__ import annotations

import ctypes as C
import os
import platform
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))

# timed frames per reference-arm run (cfg2: ~10-25 s per frame on the host)
MAX_TIMED = {"cfg1": 9, "cfg2": 3}


def host_cpu() -> dict:
    model = platform.processor() or ""
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"model": model, "nproc": os.cpu_count()}


_keep = []  # the ctypes callback must outlive its installation


def _lapack_callback():
    """A ctypes callback (n, a, b, x) -> 0 solving the dense LM step with
    LAPACK's Cholesky: see the module docstring."""
    from scipy.linalg import lapack, solve

    FN = C.CFUNCTYPE(C.c_int32, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_double),
                     C.POINTER(C.c_double))

    def fn(n, a, b, x):
        A = np.ctypeslib.as_array(a, shape=(n, n))
        B = np.ctypeslib.as_array(b, shape=(n,))
        X = np.ctypeslib.as_array(x, shape=(n,))
        M = np.array(A, order="C", copy=True)  # A is read again for the residual guard
        # symmetric: the row-major copy is its own column-major transpose
        c, info = lapack.dpotrf(M.T, lower=0, clean=0, overwrite_a=1)
        if info == 0:
            sol, info = lapack.dpotrs(c, B, lower=0)
        if info != 0:
            sol = solve(np.array(A, copy=True), B, assume_a="sym")
        X[:] = sol
        return 0

    cb = FN(fn)
    _keep.append(cb)
    return FN, cb


def _blas_threads() -> int:
    try:
        from threadpoolctl import threadpool_info

        return max((p.get("num_threads") or 1) for p in threadpool_info()) or 1
    except Exception:
        return os.cpu_count() or 1


def install_lapack_solver(O):
    """or_set_dense_solver(LAPACK Cholesky) on the oracle port."""
    FN, cb = _lapack_callback()
    L = O.lib()
    L.or_set_dense_solver.argtypes = [FN]
    L.or_set_dense_solver(cb)
    L.or_dense_solve_count.restype = C.c_int64
    return _blas_threads()


def uninstall_dense_solver(O):
    L = O.lib()
    L.or_set_dense_solver.argtypes = [C.c_void_p]
    L.or_set_dense_solver(None)


def time_oracle_frames(spec, cfg, first_timed: int, n_timed: int, lapack: bool):
    """Runs the oracle's process_frame on frames 0 .. first_timed+n_timed-1 of
    the config's synthetic sequence; frames >= first_timed are timed. Returns
    per-frame wall seconds and stats."""
    sys.path.insert(0, os.path.join(REPO, "tests"))
    import oracle_py as O
    import paper_1904_13073_b200 as pkg

    threads = install_lapack_solver(O) if lapack else 1
    try:
        ocfg = O.make_config(**{k: v for k, v in cfg.items() if k in O.DEFAULTS})
        seq = pkg.SyntheticSequence(spec["scene"], spec["seq_frames"], cfg)
        pipe = O.OraclePipeline(ocfg)  # faithful mode: fp64 state, as shipped
        O.lib().or_dense_solve_count.restype = C.c_int64
        solves0 = O.lib().or_dense_solve_count()
        secs, stats = [], []
        for t in range(first_timed + n_timed):
            d = seq.render_depth(t)
            t0 = time.perf_counter()
            st = pipe.process_frame(d, t)
            dt = time.perf_counter() - t0
            if t >= first_timed:
                secs.append(dt)
                stats.append(dict(frame=t, surfels=st.surfel_count, nodes=st.node_count,
                                  gn_iters=st.solver.iterations, solve_s=st.solve_ms * 1e-3,
                                  fusion_s=st.fusion_ms * 1e-3, rigid_s=st.rigid_ms * 1e-3))
        solves = O.lib().or_dense_solve_count() - solves0
    finally:
        if lapack:
            uninstall_dense_solver(O)
    return dict(secs=secs, stats=stats, threads=threads, dense_solves=int(solves))


def ref_available() -> bool:
    sys.path.insert(0, os.path.join(REPO, "tests"))
    import ref_py as R

    return R.available()


def time_ref_frames(spec, cfg, first_timed: int, n_timed: int, lapack: bool):
    """time_oracle_frames on the compiled reference (oracle/_ref): its own
    Pipeline::process_frame."""
    sys.path.insert(0, os.path.join(REPO, "tests"))
    import oracle_py as O
    import paper_1904_13073_b200 as pkg
    import ref_py as R

    # the dense LM step by LAPACK always (conservative: faster than the
    # reference's unblocked LDLT); lapack=False keeps it on one thread
    _, cb = _lapack_callback()
    R.set_dense_solver(cb)
    threads = _blas_threads() if lapack else 1
    limit = None
    if not lapack:  # one BLAS thread for the whole run (restored below)
        from threadpoolctl import threadpool_limits

        limit = threadpool_limits(1)
    try:
        ocfg = O.make_config(**{k: v for k, v in cfg.items() if k in O.DEFAULTS})
        seq = pkg.SyntheticSequence(spec["scene"], spec["seq_frames"], cfg)
        pipe = R.RefPipeline(ocfg)
        solves0 = R.dense_solve_count()
        secs, stats = [], []
        for t in range(first_timed + n_timed):
            d = seq.render_depth(t)
            t0 = time.perf_counter()
            st = pipe.process_frame(d, t)
            dt = time.perf_counter() - t0
            if t >= first_timed:
                secs.append(dt)
                stats.append(dict(frame=t, surfels=st["surfel_count"], nodes=st["node_count"],
                                  gn_iters=st["solver_iterations"],
                                  solve_s=st["ms"]["solve"] * 1e-3,
                                  fusion_s=st["ms"]["fusion"] * 1e-3,
                                  rigid_s=st["ms"]["rigid"] * 1e-3))
        solves = R.dense_solve_count() - solves0
        pipe.close()
    finally:
        R.set_dense_solver(None)
        if limit is not None:
            limit.restore_original_limits()
    return dict(secs=secs, stats=stats, threads=threads, dense_solves=int(solves), kind="reference",
                lapack_threads=threads)


def time_frames(spec, cfg, first_timed: int, n_timed: int, lapack: bool):
    """The compiled reference when oracle/_ref exists, else the oracle port."""
    if ref_available():
        return time_ref_frames(spec, cfg, first_timed, n_timed, lapack)
    r = time_oracle_frames(spec, cfg, first_timed, n_timed, lapack)
    r["kind"] = "port"
    return r


def describe(cfg_name, r, lapack):
    st = r["stats"]
    cpu = host_cpu()
    frames = f"frames {st[0]['frame']}-{st[-1]['frame']}" if len(st) > 1 else f"frame {st[0]['frame']}"
    if r.get("kind") == "reference":
        solver = (f"dense LM step by LAPACK Cholesky on {r['threads']} thread(s), the rest 1 thread"
                  " (faster than the reference's unblocked LDLT: a conservative baseline)")
    else:
        solver = (f"dense LM step by LAPACK Cholesky on {r['threads']} threads, the rest 1 thread"
                  if lapack else "restated Eigen LDLT, 1 thread")
    who = ("reference Pipeline::process_frame (oracle/_ref: the unmodified reference sources "
           "built against the repo's Eigen subset)" if r.get("kind") == "reference"
           else "CPU oracle process_frame (the reference restated)")
    return (f"{who} (full LM loop, {solver}) on {cfg_name} {frames}: "
            f"{len(st)} frames in {sum(r['secs']):.2f} s, surfels {st[0]['surfels']}-{st[-1]['surfels']}, "
            f"nodes {st[-1]['nodes']}, GN iterations {[s['gn_iters'] for s in st]}, "
            f"solve {sum(s['solve_s'] for s in st):.2f} s; host {cpu['model']} ({cpu['nproc']} threads)")


def cpu_baseline(args, spec, cfg):
    """bench.py's cpu_baseline leg: a bounded sample (~10-30 s of CPU work)."""
    if args.config == "cfg1":  # frames 1-5 after the init frame, 1 core
        r = time_frames(spec, cfg, 1, 5, lapack=False)
        cores, lapack = 1, False
    else:  # cfg2: the first tracked frame after the init frame
        r = time_frames(spec, cfg, 1, 1, lapack=True)
        cores, lapack = r["threads"], True
    v = len(r["secs"]) / sum(r["secs"])
    return {"value": round(v, 6), "unit": "frames/s", "cores": cores, "kind": r["kind"],
            "sample": describe(args.config, r, lapack)}


def run_reference(args):
    import bench

    spec = bench.CONFIGS[args.config]
    if args.config == "cfg3":
        return {"impl": "reference", "unavailable": "config 3 (~8k nodes): the reference's dense "
                "6N x 6N normal equations need ~18 GB and an O((6N)^3) LDLT per LM attempt"}
    cfg = bench.make_cfg(spec)
    lapack = args.config != "cfg1"
    # the first tracked frames of the sequence after the (untimed) init frame:
    # cfg1 all 9 of them; cfg2 the first 3 (~30-50 s each on the host). bench.py's
    # B200 arm reports the same frames ("reference_frames") next to its own
    # timed window, which sits later in the sequence on a larger model.
    first = 1
    n_timed = spec["seq_frames"] - 1 if args.config == "cfg1" else MAX_TIMED["cfg2"]
    r = time_frames(spec, cfg, first, n_timed, lapack=lapack)
    total = sum(r["secs"])
    v = len(r["secs"]) / total
    cores = r["threads"] if lapack else 1
    return {
        "impl": "reference", "metric": "frames/s", "value": round(v, 6), "unit": "frames/s",
        "n_gpus": args.gpus, "steps": len(r["secs"]), "warmup": first,
        "ms_per_step": round(1e3 * total / len(r["secs"]), 1), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "data": "synthetic",
        "config": {"workload": f"{args.config}: {spec['scene']} {spec['width']}x{spec['height']}, "
                               f"max {spec.get('gn_iters', 10)} GN per frame (reference LM loop, dense solve)",
                   "frames_timed": [s["frame"] for s in r["stats"]],
                   "device": f"host CPU ({host_cpu()['model']})"},
        "cpu_baseline": {"value": round(v, 6), "unit": "frames/s", "cores": cores, "kind": r["kind"],
                         "sample": describe(args.config, r, lapack)},
        "per_frame_s": [round(x, 3) for x in r["secs"]],
        "dense_solves": r["dense_solves"],
        "e2e": {"value": round(v, 6), "unit": "frames/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
