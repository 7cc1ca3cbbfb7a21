"""Multi-GPU execution model: replicas only.

The hot path does not shard inside one IPM solve (a per-colour-pass halo
exchange would be needed); the natural unit is an independent solve, as in the
reference's run_sweep thread pool (bench.cpp:296-382). Two modes:

* sweep partition: the cells of a sweep (C2: 9 (alpha, beta) cells) are dealt
  round-robin over the ranks (``partition``; 9 cells over 8 GPUs = 2 waves on
  rank 0), each rank runs its cells concurrently on its GPU (one context and
  host thread per cell, ``run_concurrent``), and the per-cell records are
  gathered to every rank in cell order (``gather_records``);
* replicas: every rank solves its own copy of the workload (C5; weak scaling).

No collective touches the data path. The cross-rank operations are the
record gather and the timing reduction: the step time is the maximum over ranks
of the device-measured time, the work is the sum of the ranks' Krylov
iterations. ``ensure_world`` makes ``bench.py --gpus N`` either run under a
matching torchrun world or relaunch itself under one.
"""
from __future__ import annotations

import os
import subprocess
import sys
import threading
from typing import Callable, List, Sequence


def env_rank():
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def partition(n_items: int, rank: int, world: int) -> List[int]:
    """Indices of the items rank `rank` runs: item i goes to rank i mod world."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"partition: bad rank {rank} of world {world}")
    return list(range(rank, n_items, world))


def waves(n_items: int, world: int) -> int:
    """Rounds of concurrent solves the slowest rank runs (ceil(n / world))."""
    return -(-n_items // world)


def run_concurrent(fn: Callable[[int], object], indices: Sequence[int]) -> dict:
    """fn(i) for every index on its own host thread (each cell owns its
    context/stream, so the solves overlap on the device); {i: fn(i)}. The first
    exception is re-raised on the calling thread."""
    res, err = {}, []

    def body(i):
        try:
            res[i] = fn(i)
        except BaseException as e:  # re-raised below
            err.append(e)

    th = [threading.Thread(target=body, args=(i,)) for i in indices]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if err:
        raise err[0]
    return res


def gather_records(local: dict, n_items: int, dist=None) -> list:
    """Merge every rank's {index: record} into one list in index order (on
    every rank). Records are small picklable summaries, never field data."""
    if dist is not None and dist.is_available() and dist.is_initialized() \
            and dist.get_world_size() > 1:
        parts = [None] * dist.get_world_size()
        dist.all_gather_object(parts, dict(local))
    else:
        parts = [dict(local)]
    merged = {}
    for p in parts:
        for k, v in p.items():
            if k in merged:
                raise RuntimeError(f"gather_records: item {k} ran on two ranks")
            merged[k] = v
    missing = [i for i in range(n_items) if i not in merged]
    if missing:
        raise RuntimeError(f"gather_records: items {missing} ran on no rank")
    return [merged[i] for i in range(n_items)]


def reduce_step_stats(total_ms: float, iters: float, dist=None, device="cpu"):
    """(max over ranks of total_ms, sum over ranks of iters). Works with the
    nccl (device tensors) and gloo (host tensors) backends."""
    import torch

    ms = torch.tensor([float(total_ms)], dtype=torch.float64, device=device)
    it = torch.tensor([float(iters)], dtype=torch.float64, device=device)
    if dist is not None and dist.is_available() and dist.is_initialized() \
            and dist.get_world_size() > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        dist.all_reduce(it, op=dist.ReduceOp.SUM)
    return float(ms[0]), float(it[0])


def aggregate_rate(max_ms: float, all_iters: float) -> float:
    """Whole-job throughput (iterations per second) of the replicas."""
    return all_iters / (max_ms / 1e3)


def reference_runs_on(rank: int) -> bool:
    """`bench.py --impl reference` under torchrun: rank 0 alone times the CPU
    reference; the other ranks exit without work."""
    return rank == 0


def ensure_world(gpus: int, argv: Sequence[str], port: int = 29533) -> None:
    """Make the process world match ``--gpus``.

    Under torchrun WORLD_SIZE must equal `gpus` (raises otherwise). Without a
    torchrun environment and gpus > 1, re-executes this script under
    ``torch.distributed.run --nproc-per-node gpus`` on 127.0.0.1 and exits
    with its status; gpus == 1 runs in-process."""
    world = os.environ.get("WORLD_SIZE")
    if world is not None:
        if int(world) != gpus:
            raise SystemExit(f"bench: --gpus {gpus} but WORLD_SIZE={world}")
        return
    if gpus <= 1:
        return
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           *argv]
    raise SystemExit(subprocess.call(cmd))
