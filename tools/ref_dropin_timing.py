"""The reference's own Python Scheduler on the same synchronous stream as
tools/sched_timing.py's drop-in loops (submit; release the oldest when > 32
resident or requests are queued; on_release), timed per probe on this
host's CPU.  Needs /root/reference (run here, not on the GPU box).

    python tools/ref_dropin_timing.py
"""

import json
import os
import sys
import time

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from gpushare.device_model import DeviceSpec, DeviceState  # noqa: E402
from gpushare.schedulers import Scheduler, ScheduleRequest, parse_policy  # noqa: E402
from gpushare.task_builder import ResourceRequest  # noqa: E402

from paper_2107_08538_b200.sweep import gen_probes  # noqa: E402


def run(policy: str, n: int) -> dict:
    GIB, KIB = 1 << 30, 1 << 10  # the b200 preset of the drop-in
    spec = DeviceSpec("b200", sm_count=148, mem_bytes=180 * GIB, smem_per_sm_bytes=228 * KIB)
    devs = [DeviceState(spec, i) for i in range(8)]
    sched = Scheduler(devs, parse_policy(policy))
    probes = gen_probes(n, seed=3)
    reqs = [ScheduleRequest("j", f"p{i}", ResourceRequest(int(p["mem_bytes"]), 0, int(p["thread_blocks"]),
                                                          int(p["warps_per_block"]), int(p["total_warps"]),
                                                          int(p["threads_per_block"]), int(p["regs_per_thread"]),
                                                          int(p["smem_per_block"]), 1.0), "task", 0.0)
            for i, p in enumerate(probes)]
    fifo, t_sub, n_sub = [], 0.0, 0
    t = time.perf_counter()
    for r in reqs:
        a = time.perf_counter()
        d = sched.submit(r, 0.0)
        t_sub += time.perf_counter() - a
        n_sub += 1
        if d.outcome == "assign":
            fifo.append((d.device, r.task_uid))
        if len(fifo) > 32 or sched.pending:
            if fifo:
                dv, u = fifo.pop(0)
                devs[dv].release_task(u)
            for q, dv in sched.on_release(0.0):
                fifo.append((dv, q.task_uid))
    loop = (time.perf_counter() - t) / n * 1e6
    return {"what": "reference_python_sync_per_probe_us", "policy": policy, "n": n, "loop_us": round(loop, 2),
            "submit_us": round(t_sub / n_sub * 1e6, 2), "host": os.uname().nodename, "cores": 1}


if __name__ == "__main__":
    for pol in ("mgb-warps", "mgb-sm"):
        print(json.dumps(run(pol, 2000)), flush=True)
