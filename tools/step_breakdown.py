"""Where a cfg 1 step's time goes (one GPU, inputs staged in HBM, as bench.py).

    python tools/step_breakdown.py [--workers 2] [--policies mgb-warps,sa] [--reps 2]

Per policy: makespan, the jobs' summed device time split into setup (copies
and memsets before the first kernel), kernels and tail (output digest and
read-back), host time outside the stream (allocation, decisions, waits),
and the kernel time per kind.  One JSON line per (policy, rep).
"""

from __future__ import annotations

import argparse
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main() -> int:
    from paper_2107_08538_b200 import catalog as C
    from paper_2107_08538_b200 import workloads as W

    ap = argparse.ArgumentParser()
    ap.add_argument("--workers", type=int, default=2)
    ap.add_argument("--policies", default="mgb-warps,sa")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--seed", type=int, default=1)
    a = ap.parse_args()
    jobs = [m.job for m in C.gen_mix("3:1", 32, seed=a.seed)]
    W.stage(jobs, [0], W.MODE_DEVICE)
    cap = W.ledger_capacity(0)
    try:
        for policy in a.policies.split(","):
            W.run_jobs(jobs, policy=policy, workers=a.workers, ledger_bytes=cap)
            for rep in range(a.reps):
                res = W.run_jobs(jobs, policy=policy, workers=a.workers, ledger_bytes=cap)
                recs = res.records
                per_kind = collections.Counter()
                for r, j in zip(recs, jobs):
                    per_kind[j.kind] += r["compute_ms"]
                busy = sum(r["end_ms"] - r["admit_ms"] for r in recs)
                dev = {k: round(sum(r[k] for r in recs), 1) for k in ("gen_ms", "compute_ms", "tail_ms")}
                print(json.dumps({
                    "policy": policy, "workers": a.workers, "rep": rep, "makespan_ms": round(res.makespan_ms, 1),
                    "jobs_per_s": round(res.completed / (res.makespan_ms / 1e3), 2),
                    "sum_admit_to_end_ms": round(busy, 1), **{"sum_" + k: v for k, v in dev.items()},
                    "host_outside_stream_ms": round(busy - sum(dev.values()), 1),
                    "decision_ms": round(res.decision_ms, 1),
                    "kernel_ms_by_kind": {k: round(v, 1) for k, v in sorted(per_kind.items())}}), flush=True)
    finally:
        W.unstage()
    return 0


if __name__ == "__main__":
    sys.exit(main())
