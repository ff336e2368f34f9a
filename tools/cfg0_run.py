"""BASELINE cfg 0: the 8-job Rodinia mix (2x bfs, hotspot, srad, kmeans,
repeated to 8) on 2 devices, the reference's CPU-runnable case.

    python tools/cfg0_run.py

CPU side: the C port of the reference scheduler (oracle/gs_oracle.c) places
the 8 probes on 2 ledgers, and the oracle's CPU kernels (all host threads)
run the jobs one after another.  GPU side: the executor places the same 8
jobs on 2 ledgers (two simulated devices on the one GPU, as the reference
simulates its devices) with the sm_100a decision kernel and runs them on
the GPU; outputs are checked against the CPU run and the placement log is
replayed through the oracle.  One JSON line per side."""

from __future__ import annotations

import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import kernels as K  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2107_08538_b200 import catalog as C  # noqa: E402
from paper_2107_08538_b200 import workloads as W  # noqa: E402


def main():
    mix = C.cfg0_mix(1)
    jobs = [m.job for m in mix]
    # CPU: scheduler port + CPU kernels
    t0 = time.perf_counter()
    outs = [K.run(j.kind, n=j.n, iters=j.iters, m=j.m, seed=j.seed) for j in jobs]
    cpu_s = time.perf_counter() - t0
    print(json.dumps({"side": "cpu", "config": "cfg0", "jobs": len(jobs), "seconds": round(cpu_s, 3),
                      "jobs_per_s": round(len(jobs) / cpu_s, 3), "threads": os.cpu_count()}), flush=True)
    # GPU: 2 ledgers on one GPU, inputs staged
    W.stage(jobs, [0], W.MODE_DEVICE)
    cap = W.ledger_capacity(0) // 2
    for policy in ("mgb-warps", "sa"):
        W.run_jobs(jobs, policy=policy, devices=[0, 0], workers=4, ledger_bytes=cap)
        res = W.run_jobs(jobs, policy=policy, devices=[0, 0], workers=4, ledger_bytes=cap)
        xlog = W.exec_log()
        n_dec, bad = O.replay_exec_log(xlog)
        ok = sum(1 for j, r, o in zip(jobs, res.records, outs) if r["checksum"] == K.digest(j.kind, o))
        print(json.dumps({"side": "gpu", "config": "cfg0", "policy": policy, "jobs": len(jobs),
                          "completed": res.completed, "oom": res.oom, "makespan_ms": round(res.makespan_ms, 2),
                          "jobs_per_s": round(res.completed / (res.makespan_ms / 1000.0), 2),
                          "outputs_bit_exact": ok, "placements_replayed": n_dec, "placement_mismatches": len(bad),
                          "devices_used": sorted({r["device"] for r in res.records})}), flush=True)
    W.unstage()


if __name__ == "__main__":
    main()
