"""Solo device time of every catalog job (small and large class), with the
achieved fraction of the roofline — quick kernel health check on the box.

    python tools/solo_times.py [kind ...]
"""

import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2107_08538_b200 import catalog as C  # noqa: E402
from paper_2107_08538_b200 import workloads as W  # noqa: E402

PEAK = {"B": 6451.2e9, "FLOP": 74.4e12, "TC_FLOP": 1652.5e12}


def main():
    kinds = sys.argv[1:] or list(C.RODINIA) + list(C.DARKNET)
    for kind in kinds:
        classes = C.RODINIA.get(kind) or C.DARKNET.get(kind)
        for cls, kw in zip(("small", "large"), classes):
            job = W.Job(kind, seed=7, **kw)
            t = time.time()
            W.run_solo(job)  # warm-up (allocations, module load)
            w0 = time.time() - t
            _, rec = W.run_solo(job)
            work, unit = C.algorithmic_work(job)
            rate = work / (rec.compute_ms * 1e-3)
            print(json.dumps({"kind": kind, "class": cls, "job": kw, "compute_ms": round(rec.compute_ms, 3),
                              "launches": rec.n_kernels, "first_wall_s": round(w0, 2),
                              "achieved": round(rate / (1e9 if unit == "B" else 1e12), 1),
                              "unit": "GB/s" if unit == "B" else "TFLOP/s",
                              "frac": round(rate / PEAK[unit], 4)}), flush=True)


if __name__ == "__main__":
    main()
