"""Run one job solo and time it: python tools/debug_job.py kind n [iters] [m]."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2107_08538_b200 import workloads as W  # noqa: E402

kind, n = sys.argv[1], int(sys.argv[2])
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 1
m = int(sys.argv[4]) if len(sys.argv) > 4 else 0
t = time.time()
out, rec = W.run_solo(W.Job(kind, n=n, iters=iters, m=m))
print(kind, n, "wall", round(time.time() - t, 3), "compute_ms", round(rec.compute_ms, 3), "kernels", rec.n_kernels,
      "checksum", rec.checksum, flush=True)
