"""Reference-compatible run records (CPU): SimReport keys and metric formulas."""

import json

from paper_2107_08538_b200 import catalog as C
from paper_2107_08538_b200 import report as Rp


class _Res:
    def __init__(self, records, makespan):
        self.records = records
        self.makespan_ms = makespan
        self.completed = sum(r["state"] == "done" for r in records)
        self.crashed = len(records) - self.completed


def _rec(state, end, wait, compute, kind="bfs"):
    return {"state": state, "kind": kind, "device": 0, "pull_ms": 0.0, "admit_ms": wait, "end_ms": end,
            "turnaround_ms": end, "wait_ms": wait, "compute_ms": compute}


def test_sim_report_has_reference_keys_and_metrics():
    mix = C.gen_mix("3:1", 4, seed=2)
    res = _Res([_rec("done", 100.0, 0.0, 50.0), _rec("done", 300.0, 20.0, 90.0), _rec("oom", 10.0, 0.0, 0.0),
                _rec("done", 200.0, 5.0, 60.0)], 300.0)
    rep = Rp.sim_report(res, mix, "mgb-warps", 8, [{"name": "b200", "sm_count": 148, "mem_bytes": 1}],
                        solo_ms=[40.0, 90.0, 1.0, 50.0])
    # SimReport.to_dict keys (sim_engine.py:99-115)
    assert set(rep) == {"policy", "seed", "workers", "devices", "jobs", "kernels", "crashes", "makespan_ms",
                        "completed", "crashed", "workload_digest", "workload_name"}
    assert set(rep["jobs"][0]) == {"job_id", "template", "class", "state", "pull_ms", "end_ms", "turnaround_ms",
                                   "wait_ms"}
    assert rep["completed"] == 3 and rep["crashed"] == 1 and len(rep["crashes"]) == 1
    m = Rp.metrics_row(rep)
    assert abs(m["throughput"] - 3 / 0.3) < 1e-9            # completed / makespan_s (metrics.py:49-59)
    assert abs(m["avg_turnaround_ms"] - 200.0) < 1e-9
    assert abs(m["slowdown_pct"] - (25.0 + 0.0 + 20.0) / 3) < 1e-9  # (actual/solo - 1) * 100
    assert abs(m["crash_pct"] - 25.0) < 1e-9
    assert json.loads(Rp.to_json(rep)) == rep
    assert Rp.to_json(rep).endswith("}\n")


def test_workload_digest_is_stable_and_seed_sensitive():
    a, b = C.gen_mix("3:1", 8, seed=1), C.gen_mix("3:1", 8, seed=2)
    assert Rp.workload_digest(a) == Rp.workload_digest(C.gen_mix("3:1", 8, seed=1))
    assert Rp.workload_digest(a) != Rp.workload_digest(b)
    assert len(Rp.workload_jsonl(a).splitlines()) == 8
