"""Placement-engine timing (cfg 4): sync-call latency and sweep throughput.

    python tools/sched_timing.py [--quick]

Prints one JSON object per measurement.  GPU numbers are CUDA-event kernel
times (sweeps) or wall-clock per synchronous drop-in call; the CPU number is
the C oracle (a restatement of the reference algorithm) on one core.
"""

import ctypes
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import oracle as O  # noqa: E402
from paper_2107_08538_b200 import _native as nat  # noqa: E402
from paper_2107_08538_b200.gpushare import (  # noqa: E402
    DeviceState,
    ResourceRequest,
    ScheduleRequest,
    Scheduler,
    device_spec,
    parse_policy,
)
from paper_2107_08538_b200.sweep import gen_probes  # noqa: E402


def sweep_gpu(spec, policy, probes):
    devs = [DeviceState(spec, i) for i in range(8)]
    sched = Scheduler(devs, parse_policy(policy))
    cap = 2 * len(probes) + 16
    ev = np.zeros((cap, 3), dtype=np.int32)
    ne, ms = ctypes.c_int64(), ctypes.c_float()
    nat.check(nat.lib().gs_sweep(sched._ptr, probes.ctypes.data, len(probes), 32, ev.ctypes.data, cap,
                                 ctypes.byref(ne), ctypes.byref(ms)))
    return ev[: ne.value], ms.value


def sweep_cpu(spec, policy, probes):
    devs = [O.OracleDevice(spec, i) for i in range(8)]
    s = O.OracleScheduler(devs, 2 if policy == "mgb-sm" else 3, 6, True)
    t = time.perf_counter()
    ev = s.sweep(probes, 32)
    return ev, (time.perf_counter() - t) * 1e3


def sync_latency(spec, policy, n):
    devs = [DeviceState(spec, i) for i in range(8)]
    sched = Scheduler(devs, parse_policy(policy))
    probes = gen_probes(n, seed=3)
    reqs = [ScheduleRequest("j", f"p{i}", ResourceRequest(int(p["mem_bytes"]), 0, int(p["thread_blocks"]),
                                                          int(p["warps_per_block"]), int(p["total_warps"]),
                                                          int(p["threads_per_block"]), int(p["regs_per_thread"]),
                                                          int(p["smem_per_block"]), 1.0), "task", 0.0)
            for i, p in enumerate(probes)]
    fifo = []
    t = time.perf_counter()
    for r in reqs:
        d = sched.submit(r, 0.0)
        if d.outcome == "assign":
            fifo.append((d.device, r.task_uid))
        if len(fifo) > 32 or sched.pending:
            if fifo:
                dv, u = fifo.pop(0)
                devs[dv].release_task(u)
            for q, dv in sched.on_release(0.0):
                fifo.append((dv, q.task_uid))
    return (time.perf_counter() - t) / n * 1e6


def main():
    quick = "--quick" in sys.argv
    spec = device_spec("b200")
    sizes = [10**3, 10**4, 10**5] if quick else [10**3, 10**4, 10**5, 10**6]
    for policy in ("mgb-warps", "mgb-sm"):
        sweep_gpu(spec, policy, gen_probes(1000, 0))  # warm-up
        for n in sizes:
            probes = gen_probes(n, seed=7)
            ev, ms = sweep_gpu(spec, policy, probes)
            rec = {"what": "sweep", "policy": policy, "n": n, "gpu_ms": round(ms, 3),
                   "gpu_ns_per_probe": round(ms * 1e6 / n, 1), "events": int(len(ev))}
            if n <= (10**5 if policy == "mgb-sm" else 10**6):
                oev, cms = sweep_cpu(spec, policy, probes)
                rec.update(cpu_oracle_ms=round(cms, 3), cpu_ns_per_probe=round(cms * 1e6 / n, 1),
                           bit_exact=bool(np.array_equal(ev, oev)))
            print(json.dumps(rec), flush=True)
        us = sync_latency(spec, policy, 2000)
        print(json.dumps({"what": "sync_dropin_per_probe_us", "policy": policy, "us": round(us, 2)}), flush=True)


if __name__ == "__main__" and "--ring" not in sys.argv:
    main()


def ring_latency(policy="mgb-warps", n=3000):
    spec = device_spec("b200")
    devs = [DeviceState(spec, i) for i in range(8)]
    sched = Scheduler(devs, parse_policy(policy))
    sched.start_ring(max_pending=n + 1, max_handles=n + 1, max_jobs=8)
    probes = gen_probes(n, seed=3)
    reqs = [ScheduleRequest("j", f"p{i}", ResourceRequest(int(p["mem_bytes"]), 0, int(p["thread_blocks"]),
                                                          int(p["warps_per_block"]), int(p["total_warps"]),
                                                          int(p["threads_per_block"]), int(p["regs_per_thread"]),
                                                          int(p["smem_per_block"]), 1.0), "task", 0.0)
            for i, p in enumerate(probes)]
    fifo = []
    t = time.perf_counter()
    for r in reqs:
        d = sched.submit(r, 0.0)
        if d.outcome == "assign":
            fifo.append((d.device, r.task_uid))
        if len(fifo) > 32 or sched.pending:
            if fifo:
                dv, u = fifo.pop(0)
                devs[dv].release_task(u)
            for q, dv in sched.on_release(0.0):
                fifo.append((dv, q.task_uid))
    us = (time.perf_counter() - t) / n * 1e6
    sched.stop_ring()
    return us


if __name__ == "__main__" and "--ring" in sys.argv:
    for pol in ("mgb-warps", "mgb-sm"):
        print(json.dumps({"what": "sync_dropin_ring_per_probe_us", "policy": pol, "us": round(ring_latency(pol), 2)}))
