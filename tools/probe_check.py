"""Print every catalog job's probe and its reference occupancy on an empty
B200 (occupancy_limit_per_sm x 148 must cover thread_blocks, else mgb-sm
REJECTs the job).

    python tools/probe_check.py
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2107_08538_b200 import catalog as C  # noqa: E402
from paper_2107_08538_b200 import workloads as W  # noqa: E402
from paper_2107_08538_b200.gpushare import ResourceRequest, device_spec, occupancy_limit_per_sm  # noqa: E402

spec = device_spec("b200")
jobs = [W.Job(k, seed=1, **kw) for k, cl in {**C.RODINIA, **C.DARKNET}.items() for kw in cl]
jobs += [W.Job("lud", n=1024), W.Job("needle", n=1024), W.Job("srad", n=1024, iters=5)]
for j in jobs:
    p = W.probe(j)
    r = ResourceRequest(p.mem_bytes, p.heap_limit_bytes, p.thread_blocks, p.warps_per_block, p.total_warps,
                        p.threads_per_block, p.regs_per_thread, p.smem_per_block, 0.0)
    occ = occupancy_limit_per_sm(spec, r)
    cap = occ * spec.sm_count
    print(f"{j.kind:8s} n={j.n:<9d} tbs={p.thread_blocks:4d} thr={p.threads_per_block:4d} regs={p.regs_per_thread:3d} "
          f"smem={p.smem_per_block:6d} occ/SM={occ:2d} cap={cap:5d} {'OK' if cap >= p.thread_blocks else 'REJECT'}")
