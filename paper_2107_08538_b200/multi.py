"""One process per GPU: rank plumbing for the job-mix bench (no data-path
collective — jobs are independent and shard by placement).

Each rank runs its own seeded mix on its own device (`rank_mix`); the only
collective is the max over ranks of the device-timed step (`max_over_ranks`),
so the whole-job value is (jobs on all ranks) / (slowest rank's time).
"""

from __future__ import annotations

import os


def dist_env() -> tuple[int, int, int]:
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def rank_mix(mix: str, jobs_per_rank: int, rank: int, base_seed: int = 1):
    """Rank r's share of the weak-scaled workload: its own seeded mix with
    seed base_seed + r (disjoint synthetic inputs per rank)."""
    from .catalog import gen_mix

    return gen_mix(mix, jobs_per_rank, seed=base_seed + rank)


def max_over_ranks(values: list[float], dist=None, device=None) -> list[float]:
    """Element-wise max over ranks (device-timed step times)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return list(values)
    import torch

    t = torch.tensor(values, dtype=torch.float64, device=device if device is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t.tolist()]


def whole_job_rate(jobs_per_rank: int, world: int, ms_per_step: float) -> float:
    """jobs/s of the whole job: every rank's jobs over the slowest rank's time."""
    return jobs_per_rank * world / (ms_per_step / 1000.0)
