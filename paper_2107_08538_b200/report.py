"""Reference-compatible records of real runs.

`sim_report` turns an executor run (workloads.run_jobs) into the reference's
SimReport dictionary (gpushare/sim_engine.py:83-119, rows of :597-629): the
same keys, so the reference's own tools (metrics.compute_metrics, the
compare grid) read a B200 run exactly like a simulated one; `to_json`
matches SimReport.to_json byte for byte (sorted keys, indent 2).
`workload_jsonl` / `workload_digest` mirror Workload.to_jsonl / .digest
(workload_gen.py:51-67) with the executable job spec in place of a trace.
`metrics_row` restates metrics.compute_metrics (metrics.py:49-98);
`decisions` turns the executor's placement log (workloads.exec_log) into the
SimReport.decisions rows (Scheduler._log, schedulers.py:203-218); and
`compare_csv` writes the compare grid's CSV (metrics.py:124-138, :175-200)
byte for byte.
"""

from __future__ import annotations

import csv
import hashlib
import io
import json
import statistics

OUTCOMES = {0: "assign", 1: "defer", 2: "reject"}  # schedulers.py:11-13
CSV_COLUMNS = ["workload", "policy", "workers", "seed", "throughput", "norm_throughput",
               "avg_turnaround_ms", "speedup", "crash_pct", "slowdown_pct", "makespan_ms"]  # metrics.py:24-27


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


def decisions(log, mix, policy: str) -> list[dict]:
    """SimReport.decisions rows of an executor run: one per submit and per
    tried re-drive entry, in the decision authority's order, with the
    reference's 9 keys (schedulers.py:203-218).  Task uids follow
    sim_engine.py:168 (`{job}.t0.0`: a catalog job is one task) or
    sim_engine.py:296 (`{job}.claim` for the job-granular sa / cg claims)."""
    claim = policy == "sa" or policy.startswith("cg")
    rows = []
    for e in log.events:
        if e.kind not in (0, 3) or e.outcome not in OUTCOMES:
            continue
        jid = mix[e.handle].job_id
        has = e.outcome == 0
        rows.append({"time_ms": e.t_ms, "job_id": jid, "task": f"{jid}.claim" if claim else f"{jid}.t0.0",
                     "policy": policy, "outcome": OUTCOMES[e.outcome], "device": e.device if has else None,
                     "mem_bytes": e.probe.mem_bytes if e.kind == 0 else _submitted_mem(log, e.handle),
                     "free_mem_after": e.free_mem_after if has else None,
                     "in_use_warps_after": e.in_use_warps_after if has else None})
    return rows


def _submitted_mem(log, handle: int) -> int:
    for e in log.events:
        if e.kind == 0 and e.handle == handle:
            return e.probe.mem_bytes
    return 0


def sim_report(result, mix, policy: str, workers: int, devices: list[dict], seed: int = 0,
               solo_ms: list[float] | None = None, workload_name: str = "",
               decision_rows: list[dict] | None = None) -> dict:
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
    rep = {
        "policy": policy, "seed": seed, "workers": workers, "devices": devices, "jobs": jobs,
        "kernels": kernels, "crashes": crashes, "makespan_ms": result.makespan_ms,
        "completed": result.completed, "crashed": result.crashed,
        "workload_digest": workload_digest(mix), "workload_name": workload_name,
    }
    if decision_rows is not None:  # SimReport.to_dict adds it only when collected (sim_engine.py:114-115)
        rep["decisions"] = decision_rows
    return rep


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


def compare_row(workload: str, m: dict) -> dict:
    """metrics._row (metrics.py:175-188) of a metrics_row result."""
    return {"workload": workload, "policy": m["policy"], "workers": m["workers"], "seed": m["seed"],
            "throughput": m["throughput"], "norm_throughput": m["norm_throughput"],
            "avg_turnaround_ms": m["avg_turnaround_ms"], "speedup": m["speedup"], "crash_pct": m["crash_pct"],
            "slowdown_pct": m["slowdown_pct"], "makespan_ms": m["makespan_ms"]}


def aggregate_rows(group: list[dict]) -> list[dict]:
    """The mean and stddev rows compare appends after each seed group
    (metrics.py:165-167, :191-200)."""
    out = []
    for label, fn in (("mean", statistics.fmean), ("stddev", statistics.pstdev)):
        row = dict(group[0])
        row["seed"] = label
        for col in CSV_COLUMNS:
            if col in ("workload", "policy", "workers", "seed"):
                continue
            row[col] = float(fn([r[col] for r in group]))
        out.append(row)
    return out


def compare_csv(rows: list[dict]) -> str:
    """CompareResult.to_csv (metrics.py:124-138): *_ms columns %.3f, other
    floats %.6g."""
    buf = io.StringIO()
    w = csv.DictWriter(buf, fieldnames=CSV_COLUMNS, lineterminator="\n")
    w.writeheader()
    for row in rows:
        out = {}
        for col in CSV_COLUMNS:
            v = row[col]
            if isinstance(v, float):
                out[col] = f"{v:.3f}" if col.endswith("_ms") else f"{v:.6g}"
            else:
                out[col] = v
        w.writerow(out)
    return buf.getvalue()
