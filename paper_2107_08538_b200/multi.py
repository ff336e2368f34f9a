"""Fleet plumbing for the job-mix bench: ONE decision authority over N GPUs.

The reference builds one Scheduler over every DeviceState
(gs/sim_engine.py:224-229): mgb-warps is a global argmin over the devices'
ledgers (gs/schedulers.py:155-171) and SA hands each job to the lowest free
device (:173-178).  So the fleet is driven by one process: rank 0 opens the
placement engine with one ledger per GPU and runs the executor over all N
devices (jobs run on per-device streams; their staged inputs move over
NVLink peer copies when a job lands on another GPU).  Jobs are independent,
so there is no collective on the data path.

Under torchrun (one process per GPU, as the bench contract launches it) the
other ranks hold their GPU's context and only join the barriers and the
max-over-ranks of the step time (they report 0 ms: the driving rank's device
clock covers the whole fleet because the executor synchronizes every device
before it returns).
"""

from __future__ import annotations

import os


def dist_env() -> tuple[int, int, int]:
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def fleet_plan(gpus: int, world: int, rank: int) -> tuple[bool, list[int]]:
    """(does this rank drive the fleet, the CUDA devices it drives).

    world == 1: this process drives GPUs 0..gpus-1 itself.  world > 1: one
    rank per GPU (world must equal gpus); rank 0 drives all of them."""
    if gpus < 1:
        raise ValueError("need at least one GPU")
    if world > 1 and world != gpus:
        raise ValueError(f"torchrun world size {world} != --gpus {gpus}")
    if rank != 0:
        return False, []
    return True, list(range(gpus))


def fleet_mix(mix: str, jobs_per_gpu: int, gpus: int, base_seed: int = 1):
    """The fleet's workload: one seeded mix of jobs_per_gpu * gpus jobs
    (weak scaling: per-GPU work fixed as N grows), placed by one authority."""
    from .catalog import gen_mix

    return gen_mix(mix, jobs_per_gpu * gpus, seed=base_seed)


def max_over_ranks(values: list[float], dist=None, device=None) -> list[float]:
    """Element-wise max over ranks (device-timed step times)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return list(values)
    import torch

    t = torch.tensor(values, dtype=torch.float64, device=device if device is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t.tolist()]


def rate(completed_per_step: float, ms_per_step: float) -> float:
    """Whole-fleet jobs/s: jobs COMPLETED per step over the (max-over-ranks)
    step time (gs/metrics.py:49-59 counts completed jobs only)."""
    return completed_per_step / (ms_per_step / 1000.0) if ms_per_step > 0 else 0.0
