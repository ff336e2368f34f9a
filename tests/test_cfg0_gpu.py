"""BASELINE cfg 0 (the 8-job mix on 2 devices, the reference's CPU-runnable
case) through the executor: two ledgers on the one GPU, every output equal
to the CPU oracle's, every placement equal to the reference scheduler's."""

import pytest

from oracle import kernels as K
from oracle import oracle as O

pytestmark = pytest.mark.gpu

W = pytest.importorskip("paper_2107_08538_b200.workloads")
C = pytest.importorskip("paper_2107_08538_b200.catalog")


@pytest.mark.parametrize("policy", ["mgb-warps", "mgb-sm", "sa"])
def test_cfg0_on_two_devices(policy):
    jobs = [m.job for m in C.cfg0_mix(1)]
    W.stage(jobs, [0], W.MODE_DEVICE)
    try:
        res = W.run_jobs(jobs, policy=policy, devices=[0, 0], workers=4, ledger_bytes=W.ledger_capacity(0) // 2)
        xlog = W.exec_log()
    finally:
        W.unstage()
    assert res.completed == len(jobs) and res.oom == 0
    for j, r in zip(jobs, res.records):
        want = K.run(j.kind, n=j.n, iters=j.iters, m=j.m, seed=j.seed)
        assert r["checksum"] == K.digest(j.kind, want), j.kind
    n_dec, bad = O.replay_exec_log(xlog)
    assert n_dec >= len(jobs) and not bad
