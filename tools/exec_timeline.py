"""Executor timeline of one cfg-1 mix run: per job pull / admit / end and
device time, to see where a step's wall time goes.

    GS_RING=0|1 python tools/exec_timeline.py [policy] [jobs] [workers]
"""

import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2107_08538_b200 import catalog as C  # noqa: E402
from paper_2107_08538_b200 import workloads as W  # noqa: E402

policy = sys.argv[1] if len(sys.argv) > 1 else "mgb-warps"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 32
workers = int(sys.argv[3]) if len(sys.argv) > 3 else 8
mix = C.gen_mix("3:1", n, seed=1)
jobs = [m.job for m in mix]
W.stage(jobs, [0], W.MODE_DEVICE)
for rep in range(2):
    t = time.time()
    res = W.run_jobs(jobs, policy=policy, workers=workers)
    print(f"run {rep} {policy} ring={os.environ.get('GS_RING', '0') == '1'}: makespan {res.makespan_ms:.1f} ms "
          f"wall {time.time() - t:.2f} s decision_ms {res.decision_ms:.1f} launches {res.decision_launches}",
          flush=True)
for m, r in zip(mix, res.records):
    print(f"  {m.template:16s} dev {r['device']} pull {r['pull_ms']:9.1f} admit {r['admit_ms']:9.1f} "
          f"end {r['end_ms']:9.1f} compute {r['compute_ms']:8.2f} state {r['state']}")
