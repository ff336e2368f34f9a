"""Reference-compatible records of real runs.

`sim_report` turns an executor run (workloads.run_jobs) into the reference's
SimReport dictionary (gpushare/sim_engine.py:83-119, rows of :597-629): the
same keys, so the reference's own tools (metrics.compute_metrics, the
compare grid) read a B200 run exactly like a simulated one; `to_json`
matches SimReport.to_json byte for byte (sorted keys, indent 2).
`workload_jsonl` / `workload_digest` mirror Workload.to_jsonl / .digest
(workload_gen.py:51-67) with the executable job spec in place of a trace.
`metrics_row` restates metrics.compute_metrics (metrics.py:49-98).
"""

from __future__ import annotations

import hashlib
import json
import statistics


def workload_jsonl(mix) -> str:
    """One sorted-key JSON object per job (Workload.to_jsonl layout)."""
    lines = []
    for m in mix:
        j = m.job
        spec = json.dumps({"kind": j.kind, "n": j.n, "m": j.m, "iters": j.iters, "seed": j.seed}, sort_keys=True)
        lines.append(json.dumps({"job_id": m.job_id, "class": m.job_class, "template": m.template,
                                 "inline_trace": spec}, sort_keys=True))
    return "\n".join(lines) + "\n"


def workload_digest(mix) -> str:
    return hashlib.sha256(workload_jsonl(mix).encode()).hexdigest()


def sim_report(result, mix, policy: str, workers: int, devices: list[dict], seed: int = 0,
               solo_ms: list[float] | None = None, workload_name: str = "") -> dict:
    """SimReport.to_dict() of a wall-clock run.  Kernel rows carry the job's
    device time (CUDA events) as actual_ms and its isolated time as solo_ms
    when `solo_ms` is given (per-kernel slowdown, metrics.py:75-79)."""
    jobs, kernels, crashes = [], [], []
    for i, (m, r) in enumerate(zip(mix, result.records)):
        state = "done" if r["state"] == "done" else "crashed"
        jobs.append({"job_id": m.job_id, "template": m.template, "class": m.job_class, "state": state,
                     "pull_ms": r["pull_ms"], "end_ms": r["end_ms"], "turnaround_ms": r["turnaround_ms"],
                     "wait_ms": r["wait_ms"]})
        if state == "done":
            kernels.append({"job_id": m.job_id, "task": f"{m.job_id}.t0.0", "kernel": r["kind"],
                            "device": r["device"], "start_ms": r["admit_ms"], "end_ms": r["end_ms"],
                            "solo_ms": solo_ms[i] if solo_ms else r["compute_ms"], "actual_ms": r["compute_ms"]})
        else:
            crashes.append({"job_id": m.job_id, "time_ms": r["end_ms"], "reason": r["state"],
                            "device": r["device"]})
    return {
        "policy": policy, "seed": seed, "workers": workers, "devices": devices, "jobs": jobs,
        "kernels": kernels, "crashes": crashes, "makespan_ms": result.makespan_ms,
        "completed": result.completed, "crashed": result.crashed,
        "workload_digest": workload_digest(mix), "workload_name": workload_name,
    }


def to_json(report: dict) -> str:
    return json.dumps(report, sort_keys=True, indent=2) + "\n"


def _raw(rep: dict) -> tuple[float, float, float]:
    done = [j for j in rep["jobs"] if j["state"] == "done"]
    s = rep["makespan_ms"] / 1000.0
    return ((rep["completed"] / s) if s > 0 else 0.0,
            statistics.fmean(j["turnaround_ms"] for j in done) if done else 0.0,
            statistics.fmean(j["wait_ms"] for j in done) if done else 0.0)


def metrics_row(rep: dict, baseline: dict | None = None) -> dict:
    """compute_metrics (metrics.py:62-98) on report dictionaries."""
    base = baseline or rep
    if rep["workload_digest"] and base["workload_digest"] and rep["workload_digest"] != base["workload_digest"]:
        raise ValueError("baseline report is from a different workload")
    tput, tat, wait = _raw(rep)
    btput, btat, _ = _raw(base)
    n = len(rep["jobs"])
    slow = [(k["actual_ms"] / k["solo_ms"] - 1.0) * 100.0 for k in rep["kernels"] if k["solo_ms"] > 0]
    return {"policy": rep["policy"], "workers": rep["workers"], "seed": rep["seed"], "n_jobs": n,
            "completed": rep["completed"], "crashed": rep["crashed"], "makespan_ms": rep["makespan_ms"],
            "throughput": tput, "norm_throughput": tput / btput if btput > 0 else 0.0,
            "avg_turnaround_ms": tat, "avg_wait_ms": wait, "speedup": btat / tat if tat > 0 else 0.0,
            "crash_pct": rep["crashed"] / n * 100.0 if n else 0.0,
            "slowdown_pct": statistics.fmean(slow) if slow else 0.0}
