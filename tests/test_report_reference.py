"""Run outputs read by the reference's own tools (CPU).

A B200 run's report (report.sim_report, with the placement log's decision
rows) is loaded into the UNMODIFIED reference SimReport and fed to the
reference's compute_metrics and CompareResult.to_csv (gs/metrics.py:62-138):
the reference must read it, produce the same metric row as
report.metrics_row, the same CSV bytes as report.compare_csv, and
SimReport.to_json must equal report.to_json byte for byte.  Skipped where
the reference tree is absent (the GPU box).
"""

import os
import sys
from types import SimpleNamespace

import pytest

from paper_2107_08538_b200 import catalog as C
from paper_2107_08538_b200 import report as Rp

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present")


@pytest.fixture(scope="module")
def ref():
    sys.path.insert(0, REF)
    try:
        import gpushare.metrics as M
        import gpushare.sim_engine as SE
    finally:
        sys.path.remove(REF)
    return SimpleNamespace(M=M, SE=SE)


class _Res:
    def __init__(self, records, makespan):
        self.records = records
        self.makespan_ms = makespan
        self.completed = sum(r["state"] == "done" for r in records)
        self.crashed = len(records) - self.completed


def _rec(state, end, wait, compute, kind="bfs", device=0):
    return {"state": state, "kind": kind, "device": device, "pull_ms": 1.0, "admit_ms": 1.0 + wait, "end_ms": end,
            "turnaround_ms": end, "wait_ms": wait, "compute_ms": compute}


def _log(mix):
    """A placement log shaped like workloads.exec_log(): submits, a deferral
    re-driven after a release."""
    def ev(kind, h, dev, out, mem=0, free=0, warps=0, t=0.0):
        return SimpleNamespace(kind=kind, handle=h, device=dev, outcome=out, freed=0, free_mem_after=free,
                               in_use_warps_after=warps, t_ms=t, probe=SimpleNamespace(mem_bytes=mem))
    return SimpleNamespace(events=[
        ev(0, 0, 0, 0, mem=5 << 30, free=100 << 30, warps=2368, t=0.1),
        ev(0, 1, -1, 1, mem=200 << 30, t=0.2),
        ev(0, 2, 1, 0, mem=3 << 30, free=150 << 30, warps=592, t=0.3),
        ev(1, 0, 0, 0, t=50.0),
        ev(3, 1, 0, 0, free=1 << 30, warps=2368, t=50.1),
        ev(0, 3, 0, 2, mem=900 << 30, t=51.0),
    ], specs=[], policy=3, cg_ratio=6)


def _reports(seed=0):
    mix = C.gen_mix("3:1", 4, seed=2)
    devs = [{"name": "b200", "sm_count": 148, "mem_bytes": 180 << 30}] * 2
    ours = _Res([_rec("done", 100.0, 0.0, 50.0), _rec("done", 300.0, 49.0, 90.0, "hotspot"),
                 _rec("done", 120.0, 0.0, 70.0, "srad", 1), _rec("rejected", 51.0, 0.0, 0.0)], 300.0)
    sa = _Res([_rec("done", 200.0, 0.0, 40.0), _rec("done", 500.0, 150.0, 80.0, "hotspot"),
               _rec("done", 350.0, 200.0, 60.0, "srad", 1), _rec("rejected", 51.0, 0.0, 0.0)], 500.0)
    r1 = Rp.sim_report(ours, mix, "mgb-warps", 8, devs, seed=seed, solo_ms=[40.0, 80.0, 60.0, 1.0],
                       workload_name="std3:1x4", decision_rows=Rp.decisions(_log(mix), mix, "mgb-warps"))
    r0 = Rp.sim_report(sa, mix, "sa", 8, devs, seed=seed, solo_ms=[40.0, 80.0, 60.0, 1.0],
                       workload_name="std3:1x4")
    return r0, r1


def _to_ref(ref, rep):
    d = dict(rep)
    d.setdefault("decisions", None)
    return ref.SE.SimReport(**d)


def test_reference_reads_our_report_and_agrees_on_metrics(ref):
    base, rep = _reports()
    m_ref = ref.M.compute_metrics(_to_ref(ref, rep), _to_ref(ref, base))
    m = Rp.metrics_row(rep, base)
    for k_ref, k in (("throughput_jps", "throughput"), ("norm_throughput", "norm_throughput"),
                     ("avg_turnaround_ms", "avg_turnaround_ms"), ("avg_wait_ms", "avg_wait_ms"),
                     ("speedup", "speedup"), ("crash_pct", "crash_pct"), ("slowdown_pct", "slowdown_pct"),
                     ("completed", "completed"), ("crashed", "crashed"), ("makespan_ms", "makespan_ms")):
        assert getattr(m_ref, k_ref) == m[k], k


def test_report_json_is_byte_identical_to_simreport(ref):
    _, rep = _reports()
    assert "decisions" in rep and len(rep["decisions"]) == 5
    assert set(rep["decisions"][0]) == {"time_ms", "job_id", "task", "policy", "outcome", "device", "mem_bytes",
                                        "free_mem_after", "in_use_warps_after"}
    assert [d["outcome"] for d in rep["decisions"]] == ["assign", "defer", "assign", "assign", "reject"]
    assert Rp.to_json(rep) == _to_ref(ref, rep).to_json()


def test_compare_csv_is_byte_identical(ref):
    rows = []
    for wl in ("std3:1x4",):
        for policy in ("mgb-warps", "sa"):
            group = []
            for seed in (0, 1):
                base, rep = _reports(seed)
                r = rep if policy == "mgb-warps" else base
                group.append(Rp.compare_row(wl, Rp.metrics_row(r, base)))
            rows.extend(group)
            rows.extend(Rp.aggregate_rows(group))
    # the same rows through the reference's own _row / _aggregate / to_csv
    ref_rows = []
    for policy in ("mgb-warps", "sa"):
        group = []
        for seed in (0, 1):
            base, rep = _reports(seed)
            r = rep if policy == "mgb-warps" else base
            group.append(ref.M._row(ref.M.compute_metrics(_to_ref(ref, r), _to_ref(ref, base), "std3:1x4")))
        ref_rows.extend(group)
        ref_rows.append(ref.M._aggregate(group, "mean", __import__("statistics").fmean))
        ref_rows.append(ref.M._aggregate(group, "stddev", __import__("statistics").pstdev))
    assert Rp.compare_csv(rows) == ref.M.CompareResult(ref_rows).to_csv()
