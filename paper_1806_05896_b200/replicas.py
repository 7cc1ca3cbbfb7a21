"""Multi-GPU execution model: replicas only.

The hot path does not shard inside one IPM solve (a per-colour-pass halo
exchange would be needed); the natural unit is an independent solve, as in the
reference's run_sweep thread pool (bench.cpp:296-382). With N ranks each rank
runs its own full replica of the 9-cell sweep on its GPU (weak scaling); no
collective touches the data path. The only cross-rank operation is the timing
reduction: the step time is the maximum over ranks of the device-measured time,
the work is the sum of the ranks' Krylov iterations.
"""
from __future__ import annotations

import os


def env_rank():
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


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
