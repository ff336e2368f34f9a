"""Synthetic probe streams for the placement-decision sweep (BASELINE cfg 4).

10^3..10^6 probes with threads in {64,128,256,512,1024}, thread blocks in
[1, 296] (2 waves of 148 SMs), memory in [1, 24] GiB, regs in {0, 32, 64}
and smem in {0, 8K, 16K} (SURVEY.md §8d cfg 4), seeded with numpy's PCG64
so the same (n, seed) gives the same stream on every box.  Probe i carries
task handle i (uid ``p{i}``).
"""

from __future__ import annotations

import numpy as np

from ._native import PROBE_DTYPE

GIB = 1 << 30
THREADS = np.array([64, 128, 256, 512, 1024], dtype=np.int64)
REGS = np.array([0, 32, 64], dtype=np.int64)
SMEM = np.array([0, 8192, 16384], dtype=np.int64)


def gen_probes(n: int, seed: int = 0, mem_gib: tuple[int, int] = (1, 24),
               max_tbs: int = 296) -> np.ndarray:
    rng = np.random.default_rng(seed)
    threads = THREADS[rng.integers(0, len(THREADS), n)]
    tbs = rng.integers(1, max_tbs + 1, n)
    mem = rng.integers(mem_gib[0], mem_gib[1] + 1, n) * GIB
    regs = REGS[rng.integers(0, len(REGS), n)]
    smem = SMEM[rng.integers(0, len(SMEM), n)]
    wpb = -(-threads // 32)
    p = np.zeros(n, dtype=PROBE_DTYPE)
    p["mem_bytes"] = mem
    p["heap_limit_bytes"] = 8 << 20
    p["total_warps"] = tbs * wpb
    p["est_duration_ms"] = 1.0
    p["thread_blocks"] = tbs
    p["warps_per_block"] = wpb
    p["threads_per_block"] = threads
    p["regs_per_thread"] = regs
    p["smem_per_block"] = smem
    p["handle"] = np.arange(n)
    p["job"] = -1
    p["level"] = 2  # GS_PROBE_FRESH: every probe names a new task handle
    return p
