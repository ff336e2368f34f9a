"""Solo device time of one job, best of R runs: python tools/kernel_time.py kind n [iters] [m] [R]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2107_08538_b200 import catalog as C  # noqa: E402
from paper_2107_08538_b200 import workloads as W  # noqa: E402

kind, n = sys.argv[1], int(sys.argv[2])
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 1
m = int(sys.argv[4]) if len(sys.argv) > 4 else 0
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 5
job = W.Job(kind, n=n, iters=iters, m=m, seed=1001)
W.run_solo(job)
ms = [W.run_solo(job)[1].compute_ms for _ in range(reps)]
work, unit = C.algorithmic_work(job)
best = min(ms)
extra = f" {work / (best * 1e-3) / 1e9:.1f} GB/s" if unit == "B" else ""
print(f"{kind} n={n} iters={iters} m={m}: best {best:.3f} ms (runs {', '.join(f'{x:.3f}' for x in ms)}){extra}",
      flush=True)
