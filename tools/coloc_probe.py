"""Co-location diagnostic: N copies of one job under sa and cg:k, reporting
makespan and per-job device time, to see how a kind shares the GPU.

    python tools/coloc_probe.py yolo 1280 32 [copies]
    python tools/coloc_probe.py resnet 896 32
"""

import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2107_08538_b200 import workloads as W  # noqa: E402

kind, n, m = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
copies = int(sys.argv[4]) if len(sys.argv) > 4 else 4
jobs = [W.Job(kind, n=n, m=m, iters=1, seed=100 + i) for i in range(copies)]
W.run_solo(jobs[0])
for policy in ["sa", "cg:2", f"cg:{copies}"]:
    for rep in range(2):
        res = W.run_jobs(jobs, policy=policy, workers=copies)
    comp = [r["compute_ms"] for r in res.records]
    print(f"{kind} n={n} m={m} x{copies} {policy:6s}: makespan {res.makespan_ms:8.1f} ms  "
          f"compute mean {statistics.fmean(comp):8.1f} max {max(comp):8.1f}  oom {res.oom}", flush=True)
    if os.environ.get("VERBOSE"):
        for r in res.records:
            print(f"    pull {r['pull_ms']:8.1f} admit {r['admit_ms']:8.1f} end {r['end_ms']:8.1f} "
                  f"compute {r['compute_ms']:7.2f}", flush=True)
