"""Multi-GPU path (replicas) on CPU: world-size-2 gloo process
group exercising the cross-rank timing reduction bench.py uses (max over ranks
of device time, sum of Krylov iterations) and the reference-arm rank rule."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1806_05896_b200 import replicas


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        r, w, lr = replicas.env_rank()
        # rank r timed 100 + 10 r ms and did 50 + r iterations
        ms, it = replicas.reduce_step_stats(100.0 + 10.0 * r, 50 + r, dist)
        q.put((r, w, lr, ms, it, replicas.aggregate_rate(ms, it), replicas.reference_runs_on(r)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_timing_reduction():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r, (rank, w, lr, ms, it, rate, ref) in enumerate(out):
        assert (rank, w, lr) == (r, world, r)
        assert ms == 110.0            # max over ranks
        assert it == 101.0            # 50 + 51
        assert rate == pytest.approx(101.0 / 0.110)
        assert ref == (r == 0)        # only rank 0 runs the reference arm


def test_single_process_reduction_is_identity():
    assert replicas.reduce_step_stats(12.5, 7) == (12.5, 7.0)
    assert replicas.aggregate_rate(500.0, 10) == 20.0
