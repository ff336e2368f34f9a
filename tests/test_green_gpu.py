"""Green-context SM partitions for co-located jobs (gs_exec_set_sm_parts):
the partitions tile the device's SMs, jobs run on them with grids sized to
the partition, and their outputs stay bit-exact with the CPU oracle."""

import pytest

from oracle import kernels as K

pytestmark = pytest.mark.gpu

W = pytest.importorskip("paper_2107_08538_b200.workloads")


@pytest.fixture
def parts():
    yield
    W.set_sm_parts(0)


@pytest.mark.parametrize("p", [2, 4])
def test_partitions_tile_the_device(p):
    import torch

    sms = W.sm_parts_layout(p)
    assert len(sms) == p
    assert sum(sms) == torch.cuda.get_device_properties(0).multi_processor_count
    assert min(sms) >= 8 and max(sms) - min(sms) <= 32


def test_jobs_on_partitions_match_oracle(parts):
    W.set_sm_parts(2)
    jobs = [W.Job("hotspot", n=512, iters=6, seed=3), W.Job("bfs", n=200_000, seed=4),
            W.Job("needle", n=512, seed=5), W.Job("kmeans", n=50_000, m=34, iters=3, seed=6),
            W.Job("srad", n=512, iters=4, seed=7), W.Job("lud", n=256, seed=8)]
    res = W.run_jobs(jobs, policy="mgb-warps", workers=4)
    assert res.completed == len(jobs) and res.oom == 0
    layout = set(W.sm_parts_layout(2))
    for j, r in zip(jobs, res.records):
        assert r["sm_share"] in layout
        if j.kind in ("bfs", "hotspot", "srad", "kmeans", "needle"):
            want = K.run(j.kind, n=j.n, iters=j.iters, m=j.m, seed=j.seed)
            assert r["checksum"] == K.digest(j.kind, want), j.kind


def test_whole_device_when_off():
    W.set_sm_parts(0)
    res = W.run_jobs([W.Job("hotspot", n=256, iters=2, seed=1)], policy="mgb-warps", workers=1)
    assert res.completed == 1 and res.records[0]["sm_share"] == 0
