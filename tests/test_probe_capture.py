"""Probe capture: libgs's gs_request_from_launches
aggregates recorded launches and buffers exactly like the reference's
compute_resource_request (gs/task_builder.py:258-290), restated in
gpushare.task_builder (both pinned to the reference's own outputs in
test_probe_golden.py).  Host arithmetic: runs on CPU."""

import random

import pytest

from paper_2107_08538_b200 import _native as nat
from paper_2107_08538_b200 import workloads as W
from paper_2107_08538_b200.gpushare.task_builder import LaunchShape, compute_resource_request


@pytest.mark.parametrize("seed", range(20))
def test_matches_compute_resource_request(seed):
    rng = random.Random(seed)
    n = rng.randint(1, 8)
    launches = []
    for _ in range(n):
        # ties in tbs * ceil(threads / 32) are common: the FIRST maximum wins
        launches.append((rng.choice([1, 2, 80, 96, 148, 296]), rng.choice([32, 64, 100, 128, 256, 1024]),
                         rng.choice([0, 32, 64, 128]), rng.choice([0, 8192, 16384, 49152]),
                         rng.choice([0.0, 0.5, 1.25])))
    buffers = [rng.randint(0, 1 << 34) for _ in range(rng.randint(0, 5))]
    heap = rng.choice([8 << 20, 0, 64 << 20])
    got = W.request_from_launches(launches, buffers, heap)
    want = compute_resource_request({f"b{i}": b for i, b in enumerate(buffers)},
                                    [LaunchShape("k", *l) for l in launches], heap_limit_bytes=heap)
    assert (got.mem_bytes, got.heap_limit_bytes, got.thread_blocks, got.warps_per_block, got.total_warps,
            got.threads_per_block, got.regs_per_thread, got.smem_per_block) == (
        want.mem_bytes, want.heap_limit_bytes, want.thread_blocks, want.warps_per_block, want.total_warps,
        want.threads_per_block, want.regs_per_thread, want.smem_per_block)
    assert got.est_duration_ms == pytest.approx(want.est_duration_ms)


def test_no_launch_is_a_config_error():
    with pytest.raises(nat.NativeError):
        W.request_from_launches([], [1 << 20])
