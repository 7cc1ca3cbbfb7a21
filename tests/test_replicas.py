"""Multi-GPU path (replicas) on CPU: world-size-2 gloo process
groups exercising what bench.py does across ranks: the sweep partition (C2's
9 cells dealt round-robin over the ranks), the concurrent per-rank execution
and the record gather back to every rank in cell order, the cross-rank timing
reduction (max over ranks of device time, sum of Krylov iterations), the
reference-arm rank rule and the --gpus / WORLD_SIZE check."""
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


def _sweep_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n_cells = 9
        mine = replicas.partition(n_cells, rank, world)
        # each "cell" is solved by a host-side stand-in on its own thread:
        # the record carries the cell index, the rank and a result only that
        # cell produces, so the gather can be checked for order and ownership
        res = replicas.run_concurrent(lambda i: dict(cell=i, rank=rank, iters=10 + i, ms=5.0 * (i + 1)),
                                      mine)
        recs = replicas.gather_records(res, n_cells, dist)
        iters = sum(r["iters"] for r in res.values())
        ms = max((r["ms"] for r in res.values()), default=0.0)
        max_ms, all_iters = replicas.reduce_step_stats(ms, iters, dist)
        q.put((rank, mine, recs, max_ms, all_iters, replicas.waves(n_cells, world)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_sweep_partition_and_gather():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_sweep_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted((q.get(timeout=120) for _ in procs), key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, mine0, recs0, ms0, it0, wv), (r1, mine1, recs1, ms1, it1, _) = out
    assert mine0 == [0, 2, 4, 6, 8] and mine1 == [1, 3, 5, 7]  # round-robin, disjoint, complete
    assert wv == 5
    # every rank receives all 9 records, in cell order, each from its owner
    for recs in (recs0, recs1):
        assert [r["cell"] for r in recs] == list(range(9))
        assert [r["rank"] for r in recs] == [i % 2 for i in range(9)]
        assert [r["iters"] for r in recs] == [10 + i for i in range(9)]
    assert ms0 == ms1 == 45.0                      # slowest cell of either rank
    assert it0 == it1 == sum(10 + i for i in range(9))


def test_partition_edge_cases():
    # 9 cells over 8 GPUs: rank 0 runs two (two waves), the others one
    parts = [replicas.partition(9, r, 8) for r in range(8)]
    assert parts[0] == [0, 8] and all(len(p) == 1 for p in parts[1:])
    assert sorted(i for p in parts for i in p) == list(range(9))
    assert replicas.waves(9, 8) == 2 and replicas.waves(9, 1) == 9 // 1
    # more ranks than cells: idle ranks get nothing
    assert replicas.partition(3, 5, 8) == []
    with pytest.raises(ValueError):
        replicas.partition(9, 2, 2)
    # a record from no rank / from two ranks is an error
    with pytest.raises(RuntimeError):
        replicas.gather_records({0: 1}, 2)


def test_ensure_world(monkeypatch):
    monkeypatch.setenv("WORLD_SIZE", "2")
    replicas.ensure_world(2, [])  # matching torchrun world: runs in-process
    with pytest.raises(SystemExit):
        replicas.ensure_world(4, [])  # mismatch fails loudly
    monkeypatch.delenv("WORLD_SIZE")
    replicas.ensure_world(1, [])  # single GPU without torchrun: in-process


def test_single_process_reduction_is_identity():
    assert replicas.reduce_step_stats(12.5, 7) == (12.5, 7.0)
    assert replicas.aggregate_rate(500.0, 10) == 20.0
