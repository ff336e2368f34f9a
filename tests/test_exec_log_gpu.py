"""Live placements vs the reference Scheduler semantics (pytest -m gpu).

SURVEY §7.3 (1): every decision the executor's single decision authority
makes while real jobs run (submits, releases, FIFO re-drives, in the order it
serialized them: gs_exec_log) is replayed through the golden-pinned C oracle
of schedulers.py:89-123 / device_model.py:192-209 and must agree decision for
decision — the placements the bench actually makes, not only recorded
streams.
"""

import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

W = pytest.importorskip("paper_2107_08538_b200.workloads")

MIX = [W.Job("bfs", n=300_000, seed=1), W.Job("hotspot", n=1024, iters=20, seed=2),
       W.Job("srad", n=1024, iters=5, seed=3), W.Job("kmeans", n=200_000, m=34, iters=3, seed=4),
       W.Job("backprop", n=200_000, m=16, iters=1, seed=5), W.Job("needle", n=1024, seed=6),
       W.Job("lud", n=1024, seed=7), W.Job("bfs", n=500_000, seed=8)] * 2


def _check(res, n_jobs):
    log = W.exec_log()
    kinds = [e.kind for e in log.events]
    assert kinds.count(W.EV_SUBMIT) == n_jobs
    checked, bad = O.replay_exec_log(log)
    assert not bad, bad[:5]
    assert checked >= 2 * n_jobs
    return log


@pytest.mark.parametrize("policy", ["mgb-warps", "mgb-sm", "sa", "cg:3"])
def test_live_placements_match_oracle(policy):
    res = W.run_jobs(MIX, policy=policy, workers=6)
    assert res.completed + res.oom == len(MIX)
    _check(res, len(MIX))


@pytest.mark.parametrize("policy", ["mgb-warps", "mgb-sm"])
def test_live_placements_with_deferrals_match_oracle(policy):
    """A ledger that holds only ~2 jobs: most submits DEFER and are admitted
    by re-drives; the whole admission order must match the oracle's."""
    tight = max(W.probe(j).mem_bytes for j in MIX) * 2
    res = W.run_jobs(MIX, policy=policy, workers=8, ledger_bytes=tight)
    assert res.completed == len(MIX) and res.oom == 0
    log = _check(res, len(MIX))
    assert sum(1 for e in log.events if e.kind == W.EV_SUBMIT and e.outcome == 1) > 0  # deferrals happened
    assert sum(1 for e in log.events if e.kind == W.EV_DRAIN and e.outcome == 0) > 0   # and were re-driven


def test_live_placements_two_ledgers_and_arrivals_match_oracle():
    cap = W.ledger_capacity(0) // 4
    # a batch of four at t = 0 (co-resident: mgb-warps spreads them over both
    # ledgers), then one arrival every 3 ms
    arrivals = [0.0 if i < 4 else 3.0 * i for i in range(len(MIX))]
    res = W.run_jobs(MIX, policy="mgb-warps", devices=[0, 0], workers=8, ledger_bytes=cap, arrivals_ms=arrivals)
    assert res.completed == len(MIX)
    log = _check(res, len(MIX))
    assert len(log.specs) == 2
    assert {e.device for e in log.events if e.kind == W.EV_SUBMIT and e.outcome == 0} == {0, 1}
