"""BASELINE cfg 2 (Darknet mix, footprints > HBM) per policy and worker count.

    python tools/cfg2_sweep.py [--workers 2,4,8] [--policies mgb-warps,sa] [--reps 2]

One JSON line per (policy, workers, rep): jobs/s, OOMs, mean turnaround.
Each configuration runs once untimed first (bench.py's cfg2_block protocol).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main() -> int:
    import torch

    from paper_2107_08538_b200 import catalog as C
    from paper_2107_08538_b200 import workloads as W

    ap = argparse.ArgumentParser()
    ap.add_argument("--workers", default="2,4,8")
    ap.add_argument("--policies", default="mgb-warps,sa")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--jobs", type=int, default=32)
    ap.add_argument("--seed", type=int, default=7)
    a = ap.parse_args()
    jobs = C.darknet_mix(a.jobs, a.seed, C.CFG2_SIZES, C.CFG2_BATCHES, C.CFG2_RESNET)
    for policy in a.policies.split(","):
        for w in [int(x) for x in a.workers.split(",")]:
            W.run_jobs(jobs, policy=policy, devices=[0], workers=w)
            for rep in range(a.reps):
                torch.cuda.synchronize(0)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                res = W.run_jobs(jobs, policy=policy, devices=[0], workers=w)
                e1.record()
                torch.cuda.synchronize(0)
                ms = e0.elapsed_time(e1)
                done = [r for r in res.records if r["state"] == "done"]
                print(json.dumps({"policy": policy, "workers": w, "rep": rep,
                                  "jobs_per_s": round(res.completed / (ms / 1e3), 3), "ms": round(ms, 1),
                                  "oom": res.oom,
                                  "mean_turnaround_ms": round(statistics.fmean(r["turnaround_ms"] for r in done), 1),
                                  "mean_compute_ms": round(statistics.fmean(r["compute_ms"] for r in done), 1)}),
                      flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
