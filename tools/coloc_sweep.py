"""Co-location trade-off on the cfg 1 mix (one GPU, inputs staged in HBM):
jobs/s and per-kernel slowdown vs solo for SM partitions x workers.

    python tools/coloc_sweep.py [--configs 0x8,2x8,4x8,0x4,0x2] [--reps 2]

Config PxW: P green-context SM partitions (0 = whole-device streams), W
workers.  One JSON line per config, plus sa.  Slowdown = (co-located
kernel device time / solo - 1) * 100 (metrics.py:75-79)."""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2107_08538_b200 import catalog as C  # noqa: E402
from paper_2107_08538_b200 import workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="0x8,2x8,4x8,0x4,0x2")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--jobs", type=int, default=32)
    ap.add_argument("--policy", default="mgb-warps")
    ap.add_argument("--capture", action="store_true", help="executor capture mode (task-graph probes + replay)")
    args = ap.parse_args()
    mix = C.gen_mix("3:1", args.jobs, seed=1)
    jobs = [m.job for m in mix]
    W.stage(jobs, [0], W.MODE_DEVICE)
    cap = W.ledger_capacity(0)
    solo = {}
    for m in mix:
        if m.template not in solo:
            W.run_solo(m.job)
            solo[m.template] = min(W.run_solo(m.job)[1].compute_ms for _ in range(2))
    runs = [(p, w, args.policy) for p, w in (tuple(int(x) for x in c.split("x")) for c in args.configs.split(","))]
    runs.append((0, 8, "sa"))
    W.set_capture(args.capture)
    for parts, workers, policy in runs:
        W.set_sm_parts(parts)
        W.run_jobs(jobs, policy=policy, workers=workers, ledger_bytes=cap)
        ms, sl, ta = [], [], []
        for _ in range(args.reps):
            res = W.run_jobs(jobs, policy=policy, workers=workers, ledger_bytes=cap)
            ms.append(res.makespan_ms)
            ta += [r["turnaround_ms"] for r in res.records if r["state"] == "done"]
            sl += [(r["compute_ms"] / solo[mix[i].template] - 1) * 100 for i, r in enumerate(res.records)
                   if r["state"] == "done"]
        mk = statistics.fmean(ms)
        print(json.dumps({"capture": args.capture, "parts": parts, "workers": workers, "policy": policy, "makespan_ms": round(mk, 1),
                          "jobs_per_s": round(len(jobs) / (mk / 1000), 2),
                          "mean_turnaround_ms": round(statistics.fmean(ta), 1),
                          "slowdown_mean_pct": round(statistics.fmean(sl), 1),
                          "slowdown_median_pct": round(statistics.median(sl), 1),
                          "layout": W.sm_parts_layout(parts) if parts > 1 else None}), flush=True)
    W.set_sm_parts(0)
    W.unstage()


if __name__ == "__main__":
    main()
