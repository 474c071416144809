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
