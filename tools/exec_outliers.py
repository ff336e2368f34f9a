"""Repeat the cfg-1 mix step and print the per-job phase records of any step
slower than 1.3x the median (diagnoses intermittent executor stalls).

    python tools/exec_outliers.py [policy] [reps]
"""

import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2107_08538_b200 import catalog as C  # noqa: E402
from paper_2107_08538_b200 import workloads as W  # noqa: E402

policy = sys.argv[1] if len(sys.argv) > 1 else "mgb-warps"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 12
mix = C.gen_mix("3:1", 32, seed=1)
jobs = [m.job for m in mix]
W.stage(jobs, [0], W.MODE_DEVICE)
runs = []
for rep in range(reps):
    t = time.perf_counter()
    res = W.run_jobs(jobs, policy=policy, workers=8)
    wall = (time.perf_counter() - t) * 1e3
    runs.append(res)
    print(f"rep {rep}: makespan {res.makespan_ms:.1f} ms, call wall {wall:.1f} ms", flush=True)
med = statistics.median(r.makespan_ms for r in runs)
for i, res in enumerate(runs):
    if res.makespan_ms < 1.3 * med:
        continue
    print(f"== rep {i} makespan {res.makespan_ms:.1f} (median {med:.1f})")
    for m, r in sorted(zip(mix, res.records), key=lambda x: x[1]["admit_ms"]):
        print(f"  {m.template:16s} admit {r['admit_ms']:7.1f} end {r['end_ms']:7.1f} setup {r['setup_ms']:6.1f} "
              f"gen {r['gen_ms']:6.1f} comp {r['compute_ms']:7.2f} tail {r['tail_ms']:6.1f}")
