"""e2e mix makespan vs worker count (inputs in pinned host memory, H2D/D2H
inside the run):  python tools/e2e_probe.py [workers ...]"""

import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2107_08538_b200 import catalog as C  # noqa: E402
from paper_2107_08538_b200 import workloads as W  # noqa: E402

mix = C.gen_mix("3:1", 32, seed=1)
jobs = [m.job for m in mix]
W.stage(jobs, [0], W.MODE_E2E)
for w in [int(a) for a in sys.argv[1:]] or [8]:
    for rep in range(2):
        t = time.time()
        res = W.run_jobs(jobs, policy="mgb-warps", workers=w, mode=W.MODE_E2E)
    h2d = sum(r["h2d_bytes"] for r in res.records)
    d2h = sum(r["d2h_bytes"] for r in res.records)
    print(f"workers {w}: makespan {res.makespan_ms:.1f} ms ({32 / res.makespan_ms * 1e3:.1f} jobs/s) "
          f"h2d {h2d / 1e9:.1f} GB d2h {d2h / 1e9:.1f} GB -> {h2d / res.makespan_ms / 1e6:.1f} GB/s in", flush=True)
