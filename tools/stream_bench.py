"""BASELINE cfg 2 and cfg 3 on one B200 (the bench line is cfg 1).

    python tools/stream_bench.py --config 2 [--jobs 32] [--seed 1]
    python tools/stream_bench.py --config 3 [--jobs 128] [--seed 1] [--load 0.7]

cfg 2  Darknet YOLOv3-tiny + ResNet-50 inference mix (random init, batch
       32-64, large images: 7-33 GB per job) whose co-running footprint exceeds
       the device: run under mgb-warps (memory-safe), cg:8 (no memory
       check) and sa; reports jobs/s, mean turnaround and OOMs per policy.
cfg 3  a 128-job stream mixing cfg 1's Rodinia jobs with cfg 2's Darknet
       jobs, Poisson arrivals (seeded) at the offered load `--load` of one
       GPU's solo service rate; reports jobs/s, mean turnaround and the
       per-kernel slowdown against each job run alone
       ((co-located / solo device time - 1) * 100, metrics.py:75-79).
Inputs are synthesized on the device by each job (unstaged), so every
job's time includes its input generation.  Each policy runs `--reps` times
and the last run is reported: the first run of a policy grows the
stream-ordered device pool to that policy's co-running footprint (physical
mapping of up to ~170 GB), a one-off cost a serving process pays once.
One JSON line per policy.
"""

from __future__ import annotations

import argparse
import json
import os
import random
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2107_08538_b200 import catalog as C  # noqa: E402
from paper_2107_08538_b200.catalog import CFG2_BATCHES, CFG2_RESNET, CFG2_SIZES, darknet_mix  # noqa: E402
from paper_2107_08538_b200 import workloads as W  # noqa: E402

GIB = 1 << 30


def summarize(res, solo=None) -> dict:
    done = [r for r in res.records if r["state"] == "done"]
    d = {
        "jobs_per_s": round(res.completed / (res.makespan_ms / 1000.0), 4) if res.makespan_ms else 0.0,
        "makespan_ms": round(res.makespan_ms, 1),
        "mean_turnaround_ms": round(statistics.fmean(r["turnaround_ms"] for r in done), 1) if done else None,
        "mean_wait_ms": round(statistics.fmean(r["wait_ms"] for r in done), 1) if done else None,
        "completed": res.completed, "oom": res.oom, "crashed": res.crashed,
    }
    if solo:
        sl = [(r["compute_ms"] / solo[i] - 1.0) * 100.0 for i, r in enumerate(res.records)
              if r["state"] == "done" and solo[i] > 0]
        d["kernel_slowdown_pct_mean"] = round(statistics.fmean(sl), 2) if sl else None
        d["kernel_slowdown_pct_median"] = round(statistics.median(sl), 2) if sl else None
    return d


def cfg2(args):
    jobs = darknet_mix(args.jobs, args.seed, CFG2_SIZES, CFG2_BATCHES, CFG2_RESNET)
    foot = sum(C.host_footprint(j) for j in jobs)
    for policy in ("mgb-warps", "cg:8", "sa"):
        for _ in range(args.reps):  # the last run is reported (device pool warm)
            res = W.run_jobs(jobs, policy=policy, workers=args.workers)
        line = {"config": "cfg2 darknet yolov3-tiny + resnet-50 mix", "policy": policy, "jobs": len(jobs),
                "sum_footprint_gib": round(foot / GIB, 1), **summarize(res)}
        print(json.dumps(line), flush=True)
        if args.dump:
            with open(args.dump, "a") as f:
                f.write(json.dumps({"policy": policy, "summary": line,
                                    "jobs": [{"kind": j.kind, "n": j.n, "m": j.m, **r}
                                             for j, r in zip(jobs, res.records)]}) + "\n")


def cfg3(args):
    rod = [m.job for m in C.gen_mix("3:1", args.jobs // 2, seed=args.seed)]
    dk = darknet_mix(args.jobs - len(rod), args.seed + 1)
    rng = random.Random(f"{args.seed}|cfg3|{args.jobs}")
    jobs = rod + dk
    rng.shuffle(jobs)
    # isolated device time of every job (the slowdown baseline) and the
    # solo service rate the offered load is measured against
    solo = []
    for j in jobs:
        _, rec = W.run_solo(j)
        solo.append(rec.compute_ms)
    W.run_solo(jobs[0])
    mean_service_ms = statistics.fmean(solo)
    lam = args.load / mean_service_ms  # jobs per ms
    t, arrivals = 0.0, []
    for _ in jobs:
        t += rng.expovariate(lam)
        arrivals.append(t)
    for policy in ("mgb-warps", "sa"):
        for _ in range(args.reps):
            res = W.run_jobs(jobs, policy=policy, workers=args.workers, arrivals_ms=arrivals)
        line = {"config": "cfg3 poisson rodinia+darknet stream", "policy": policy, "jobs": len(jobs),
                "offered_load": args.load, "mean_solo_ms": round(mean_service_ms, 2),
                "arrival_span_ms": round(arrivals[-1], 1), **summarize(res, solo)}
        print(json.dumps(line), flush=True)
        if args.by_kind:
            print(json.dumps({"policy": policy, "by_kind": by_kind(jobs, res, solo)}), flush=True)
        if args.dump:
            with open(args.dump, "a") as f:
                f.write(json.dumps({"policy": policy, "load": args.load, "summary": line,
                                    "jobs": [{"kind": j.kind, "n": j.n, "m": j.m, "solo_ms": s, **r}
                                             for j, r, s in zip(jobs, res.records, solo)]}) + "\n")


def by_kind(jobs, res, solo) -> dict:
    """Per job kind: count, mean turnaround and mean kernel slowdown."""
    out = {}
    for j, r, s in zip(jobs, res.records, solo):
        if r["state"] != "done":
            continue
        d = out.setdefault(j.kind, {"n": 0, "tat": 0.0, "slow": 0.0, "solo": 0.0})
        d["n"] += 1
        d["tat"] += r["turnaround_ms"]
        d["slow"] += (r["compute_ms"] / s - 1.0) * 100.0 if s > 0 else 0.0
        d["solo"] += s
    return {k: {"n": d["n"], "tat_ms": round(d["tat"] / d["n"], 1), "slowdown_pct": round(d["slow"] / d["n"], 1),
                "solo_ms": round(d["solo"] / d["n"], 2)} for k, d in out.items()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, choices=[2, 3], required=True)
    ap.add_argument("--jobs", type=int, default=None)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--workers", type=int, default=8)
    ap.add_argument("--load", type=float, default=0.7)
    ap.add_argument("--dump", default=None, help="cfg 3: append every run's per-job records (JSON lines) here")
    ap.add_argument("--by-kind", action="store_true", help="cfg 3: also print per-kind turnaround / slowdown")
    ap.add_argument("--reps", type=int, default=2,
                    help="runs per policy; the last is reported, so the device pool has grown to the "
                         "policy's co-running footprint (the bench's warm-up rule)")
    args = ap.parse_args()
    if args.jobs is None:
        args.jobs = 32 if args.config == 2 else 128
    (cfg2 if args.config == 2 else cfg3)(args)


if __name__ == "__main__":
    main()
