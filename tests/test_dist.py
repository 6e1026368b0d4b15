"""Multi-GPU path on CPU: bench.py's replica timing reduction (max over ranks)
and whole-job value with a world-size-2 gloo process group."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    elapsed = [0.5, 0.8][rank]          # per-rank device seconds for the same K steps
    m = bench.reduce_max(elapsed, dist, "cpu")
    v = bench.job_value(world, 100, m)
    dist.barrier()
    q.put((rank, m, v))
    dist.destroy_process_group()


def test_replica_timing_is_max_over_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(2))
    for rank, m, v in res:
        assert m == pytest.approx(0.8)
        assert v == pytest.approx(2 * 100 / 0.8)


def test_single_process_identity():
    import bench
    assert bench.reduce_max(1.25, None) == 1.25
    assert bench.job_value(1, 20, 0.5) == 40.0
