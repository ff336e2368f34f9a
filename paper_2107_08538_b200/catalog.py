"""Rodinia-class job catalog and seeded job mixes (BASELINE cfg 1).

The reference's catalog (gpushare/data/catalog.json) describes each job by
footprint and duration only; here each template is an executable job with a
small and a large size class (the reference's 1-4 GiB / 4-13 GiB classes,
catalog.json:3).  `gen_mix` follows gpushare/workload_gen.py:177-214: larges
rounded up, picks drawn from random.Random(f"{seed}|{mix}|{n}"), then
shuffled, job ids j00..jNN.
"""

from __future__ import annotations

import math
import random
from dataclasses import dataclass

from .workloads import Job

# kind -> (small kwargs, large kwargs)
RODINIA = {
    "bfs": (dict(n=16_000_000), dict(n=48_000_000)),
    "hotspot": (dict(n=8192, iters=40), dict(n=16384, iters=40)),
    "srad": (dict(n=8192, iters=10), dict(n=16384, iters=10)),
    "kmeans": (dict(n=4_000_000, m=34, iters=5), dict(n=8_000_000, m=34, iters=10)),
    "backprop": (dict(n=16_000_000, m=16, iters=2), dict(n=32_000_000, m=16, iters=2)),
    "needle": (dict(n=8192), dict(n=16384)),
    "lud": (dict(n=4096), dict(n=6144)),
}

# the 8-job CPU-runnable mix of cfg 0 (2x bfs, hotspot, srad, kmeans, repeated)
CFG0 = [("bfs", dict(n=1_000_000)), ("bfs", dict(n=1_000_000)), ("hotspot", dict(n=1024, iters=20)),
        ("srad", dict(n=2048, iters=5)), ("kmeans", dict(n=494_020, m=34, iters=5))]


@dataclass(frozen=True)
class MixJob:
    job_id: str
    template: str
    job_class: str
    job: Job


def parse_mix(mix: str) -> tuple[int, int]:
    rl, rs = (int(x) for x in mix.split(":"))
    if rl < 0 or rs < 0 or rl + rs == 0:
        raise ValueError(f"bad mix {mix!r}")
    return rl, rs


def gen_mix(mix: str = "3:1", n: int = 32, seed: int = 1, kinds: tuple[str, ...] = tuple(RODINIA)) -> list[MixJob]:
    """Seeded job mix, larges:smalls (workload_gen.py:177-214 selection)."""
    rl, rs = parse_mix(mix)
    n_large = math.ceil(rl / (rl + rs) * n)
    n_small = n - n_large
    rng = random.Random(f"{seed}|{mix}|{n}")
    picks = [(rng.choice(kinds), "small") for _ in range(n_small)]
    picks += [(rng.choice(kinds), "large") for _ in range(n_large)]
    rng.shuffle(picks)
    width = max(2, len(str(n - 1)))
    out = []
    for i, (kind, cls) in enumerate(picks):
        kw = RODINIA[kind][0 if cls == "small" else 1]
        out.append(MixJob(f"j{i:0{width}d}", f"{kind}_{cls}", cls,
                          Job(kind, seed=seed * 1000 + i, **kw)))
    return out


def cfg0_mix(seed: int = 1) -> list[MixJob]:
    """BASELINE cfg 0: 8 jobs (2x bfs, hotspot, srad, kmeans, repeated to 8)."""
    out = []
    for i in range(8):
        kind, kw = CFG0[i % len(CFG0)]
        out.append(MixJob(f"j{i:02d}", kind, "small", Job(kind, seed=seed * 1000 + i, **kw)))
    return out


def host_footprint(job: Job) -> int:
    """The probe's mem_bytes computed on the host alone (same rule as
    gs_job_probe: buffers rounded to 2 MiB + the 8 MiB task heap) — used by
    the CPU reference arm, which must not touch the GPU engine."""
    g = 2 << 20
    n, m = job.n, job.m
    sizes = {
        "bfs": [(n + 1) * 4, n * 24, n * 4, n * 4, n * 4, 16, (n // 32 + 1) * 4],
        "hotspot": [n * n * 4] * 3,
        "srad": [n * n * 4] * 3 + [16],
        "kmeans": [n * m * 4, n * 4, 5 * m * 4, 5 * m * 8, 40],
        "backprop": [(n + 1) * 4, m * (n + 1) * 4, m * (n + 1) * 4, 320, 148 * 8 * 16 * 8],
        "needle": [(n + 1) * (n + 1) * 4] * 2 + [(n // 32 + 1) * 4],
        "lud": [n * n * 4],
    }[job.kind]
    return (8 << 20) + sum((s + g - 1) // g * g for s in sizes)


def algorithmic_work(job: Job) -> tuple[float, str]:
    """(work, unit) per job run — SURVEY.md §8d's per-unit figures times the
    units a run processes: bytes for HBM-bound kernels, flops for lud."""
    n, it, m = job.n, max(job.iters, 1), job.m
    if job.kind == "hotspot":
        return 12.0 * n * n * it, "B"
    if job.kind == "srad":
        return 24.0 * n * n * it, "B"
    if job.kind == "bfs":
        return 4.0 * 6 * n + 13.0 * n, "B"
    if job.kind == "kmeans":
        return (4.0 * n * m + 4.0 * n) * it, "B"
    if job.kind == "backprop":
        return 16.0 * (n + 1) * (m + 1) * it, "B"
    if job.kind == "needle":
        return 8.0 * (n + 1) * (n + 1), "B"
    if job.kind == "lud":
        return 2.0 / 3.0 * n ** 3, "FLOP"
    return 0.0, "B"
