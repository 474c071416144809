"""The N>1 bench path on CPU: 2 ranks over gloo, barrier + max-over-ranks timing and
the weak-scaling aggregate (independent sequences, no collective on the data path)."""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench

    bench.dist_barrier(world)
    per_rank_ms = 100.0 + 50.0 * rank          # rank 1 is the slow one
    tmax = bench.dist_max(per_rank_ms, world)
    out[rank] = (tmax, bench.aggregate_fps(world, 10, tmax))
    dist.destroy_process_group()


def test_two_rank_gloo_timing_and_aggregate():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    assert out[0][0] == out[1][0] == 150.0
    # 2 ranks x 10 frames in 150 ms (slowest rank) = 133.3 frames/s
    assert abs(out[0][1] - 2 * 10 / 0.150) < 1e-9


def test_single_rank_is_identity():
    import bench

    assert bench.dist_max(3.5, 1) == 3.5
    assert bench.aggregate_fps(1, 50, 500.0) == 100.0


def test_bench_main_spawns_ranks_over_gloo():
    """`bench.py --gpus 2` with no launcher environment: main() spawns two rank
    processes itself, they rendezvous over gloo on 127.0.0.1 (no NCCL), time with
    a barrier + max over ranks, and rank 0 alone prints one JSON line with
    n_gpus = 2 (DS_BENCH_DRYRUN stands in a host sleep for the device work)."""
    import json
    import subprocess
    import sys

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items()
           if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    env["DS_BENCH_DRYRUN"] = "1"
    out = subprocess.run([sys.executable, os.path.join(repo, "bench.py"), "--gpus", "2",
                          "--steps", "20", "--warmup", "3"], env=env, capture_output=True,
                         text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["dryrun"] is True and d["n_gpus"] == 2 and d["steps"] == 20
    # the slow rank (2 ms per step) defines the job time
    assert d["max_rank_ms"] >= 20 * 2.0
    assert abs(d["value"] - 2 * 20 / (d["max_rank_ms"] * 1e-3)) < 1e-6
    assert "nccl" not in (out.stdout + out.stderr).lower()
