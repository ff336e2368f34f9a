"""Job-mix throughput on B200 under the GPU placement engine.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step runs BASELINE cfg 1's job mix (32 Rodinia-class jobs, 3:1
large:small, synthetic seeded inputs) end to end: every job's probe is
placed by the sm_100a decision kernel (mgb-warps, Alg. 3), jobs run
concurrently on per-job streams with stream-ordered allocations, releases
re-drive the FIFO.  One process per GPU; under torchrun each rank runs its
own mix on its own device (jobs are independent: placement shards them, no
collective on the data path) -> scaling "weak".

value   jobs/s with inputs resident in HBM when the timed region starts
e2e     jobs/s through the same API with inputs in pinned host memory:
        H2D of every input and D2H of every output inside the timed region
sa      the one-job-per-GPU baseline (policy sa) on the same mix and device

--impl reference times the reference's path on the host CPU: the C port of
the reference scheduler (oracle/gs_oracle.c, schedulers.py semantics) plus
the CPU restatements of the kernels (oracle/kernels_cpu.c, all host
threads) on a bounded sample of the same mix.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "job-mix jobs/s + mean turnaround at 1/2/4/8 B200 vs one-job-per-GPU; OOMs"
UNIT = "jobs/s"


_T0 = time.time()


def log(msg: str) -> None:
    """Progress on stderr (the JSON line stays the only stdout output)."""
    print(f"[bench +{time.time() - _T0:7.1f}s] {msg}", file=sys.stderr, flush=True)


def peaks() -> dict:
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "_fallback": True}


FP32_TFLOPS_NOMINAL = 148 * 128 * 2 * 1.965e9 / 1e12  # 74.4: 148 SMs x 128 FMA lanes


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = f"/tmp/gs_clocks_{os.getpid()}.csv"

    def __enter__(self):
        if os.environ.get("GS_BENCH_NO_CLOCKS"):  # diagnostics only: the bench line then says "unsampled"
            return self
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self) -> dict:
        try:
            rows = [r.split(",") for r in open(self.path).read().strip().splitlines()]
        except OSError:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in rows if len(r) >= 9]
        mx = [float(r[2]) for r in rows if len(r) >= 9]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows if len(r) >= 9 for i in range(4)
                          if r[5 + i].strip().lower() == "active"})
        loaded = sorted(sm)[len(sm) // 2:] if sm else []
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(sm)}


def run_steps(W, jobs, policy, device, workers, mode, steps, warmup, torch, dist=None):
    """W warm-up + K timed steps; device-timed with CUDA events; the K steps
    are bracketed by a barrier across ranks (and a device synchronize) on
    both sides.  The ledger capacity is queried once (a slow driver query)
    before the steps."""
    cap = W.ledger_capacity(device)
    for w in range(warmup):
        r = W.run_jobs(jobs, policy=policy, devices=[device], workers=workers, mode=mode, ledger_bytes=cap)
        log(f"warmup {w} {policy} mode={mode}: {r.makespan_ms:.1f} ms, {r.completed} done, {r.oom} oom")
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    times, results = [], []
    # the interpreter's cyclic GC is host noise, not executor work: collect
    # before the timed steps and keep it off while they run
    gc.collect()
    gc.disable()
    for _ in range(steps):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        res = W.run_jobs(jobs, policy=policy, devices=[device], workers=workers, mode=mode, ledger_bytes=cap)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
        results.append(res)
        log(f"step {policy} mode={mode}: {times[-1]:.1f} ms (executor makespan {res.makespan_ms:.1f}), "
            f"{res.completed} done, {res.oom} oom")
    gc.enable()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    return times, results


def summarize(results, times):
    done = [r for res in results for r in res.records if r["state"] == "done"]
    return {
        "ms_per_step": statistics.fmean(times),
        "mean_turnaround_ms": statistics.fmean(r["turnaround_ms"] for r in done) if done else 0.0,
        "mean_wait_ms": statistics.fmean(r["wait_ms"] for r in done) if done else 0.0,
        "completed": sum(res.completed for res in results),
        "oom": sum(res.oom for res in results),
        "crashed": sum(res.crashed for res in results),
        "kernel_launches": sum(res.kernel_launches for res in results),
        "decision_launches": sum(res.decision_launches for res in results),
        "decision_ms": sum(res.decision_ms for res in results),
    }


def kernel_rooflines(W, C, jobs, device, pk):
    """Every distinct job of the mix alone on the device (CUDA events on the
    job's stream around its kernels).  Returns (per-kind roofline of the
    kind's largest job: algorithmic work / kernel time vs the measured peak,
    per-template solo ms)."""
    solo_ms, first = {}, {}
    for mj in jobs:
        if mj.template in solo_ms:
            continue
        log(f"solo {mj.template} n={mj.job.n}")
        W.run_solo(mj.job, device)  # warm-up
        solo_ms[mj.template] = min(W.run_solo(mj.job, device)[1].compute_ms for _ in range(2))
        j = mj.job
        if j.kind not in first or j.n * max(j.m, 1) > first[j.kind][0].n * max(first[j.kind][0].m, 1):
            first[j.kind] = (j, mj.template)
    out = {}
    hbm = pk["hbm_gbs"]
    for kind, (job, tpl) in first.items():
        ms = solo_ms[tpl]
        work, unit = C.algorithmic_work(job)
        _, rec = W.run_solo(job, device)
        if unit == "B":
            ach = work / (ms * 1e-3) / 1e9
            out[kind] = {"bound": "hbm", "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
                         "frac": round(ach / hbm, 4), "ms": round(ms, 3), "launches": rec.n_kernels,
                         "job": {"n": job.n, "iters": job.iters, "m": job.m}}
        elif unit == "TC_FLOP":
            ach = work / (ms * 1e-3) / 1e12
            pkt = pk["bf16_tflops"]
            out[kind] = {"bound": "tensor", "achieved": round(ach, 1), "peak": pkt, "unit": "TFLOP/s",
                         "frac": round(ach / pkt, 4), "ms": round(ms, 3), "launches": rec.n_kernels,
                         "job": {"n": job.n, "batch": job.m}}
        else:
            ach = work / (ms * 1e-3) / 1e12
            out[kind] = {"bound": "fp32", "achieved": round(ach, 2), "peak": round(FP32_TFLOPS_NOMINAL, 1),
                         "unit": "TFLOP/s", "frac": round(ach / FP32_TFLOPS_NOMINAL, 4), "ms": round(ms, 3),
                         "launches": rec.n_kernels, "job": {"n": job.n}}
    return out, solo_ms


def traffic_from_profiles(kind: str):
    """ncu DRAM bytes of one launch of the kind's main kernel (profiles/traffic.json)."""
    try:
        with open(os.path.join(REPO, "profiles", "traffic.json")) as f:
            return json.load(f).get(kind)
    except (OSError, ValueError):
        return None


def pcie_h2d_gbps(torch) -> float:
    """Measured pinned host -> device copy bandwidth (the e2e ceiling)."""
    n = 1 << 28  # 1 GiB of float32
    h = torch.empty(n, dtype=torch.float32, pin_memory=True)
    d = torch.empty(n, dtype=torch.float32, device="cuda")
    best = 1e9
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        d.copy_(h, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del h, d
    return 4.0 * n / (best * 1e-3) / 1e9


def cpu_sample(jobs, budget_s: float):
    """The oracle's CPU kernels on all host threads over a bounded sample of
    the mix (jobs in mix order until the time budget is spent)."""
    from oracle import kernels as K

    t0 = time.perf_counter()
    n = 0
    names = []
    for mj in jobs:
        j = mj.job
        K.run(j.kind, n=j.n, iters=j.iters, m=j.m, seed=j.seed)
        n += 1
        names.append(mj.template)
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    return n / dt, n, names, dt


def reference_arm(args, jobs):
    """--impl reference: the reference's path on host cores (C port)."""
    from oracle import oracle as O
    from paper_2107_08538_b200 import _native as nat
    from paper_2107_08538_b200.catalog import host_footprint
    from paper_2107_08538_b200.gpushare import device_spec

    threads = os.cpu_count() or 1
    values = []
    sample_desc = ""
    spec = device_spec("b200")
    for step in range(args.warmup + args.steps):
        # placement of the whole mix on the CPU scheduler port (B200
        # ledgers), then the kernels of a bounded sample on all threads
        t0 = time.perf_counter()
        devs = [O.OracleDevice(spec, i) for i in range(max(1, args.gpus))]
        sched = O.OracleScheduler(devs, 3, 6, True)
        for i, mj in enumerate(jobs):
            pr = nat.GsProbe(host_footprint(mj.job), 8 << 20, 296 * 8, 0.0, 296, 8, 256, 0, 0, i, i, 0)
            sched.submit(pr)
        rate, n, names, dt = cpu_sample(jobs[step % len(jobs):] + jobs[:step % len(jobs)], args.cpu_budget)
        total = time.perf_counter() - t0
        if step >= args.warmup:
            values.append(n / total)
            sample_desc = f"{n} of {len(jobs)} mix jobs per step ({', '.join(names)}) + placement of all {len(jobs)}"
    v = statistics.fmean(values)
    line = {
        "metric": METRIC, "value": round(v, 4), "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(1000.0 / v, 1) if v else None, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32/i32", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": f"cfg1: {len(jobs)}-job Rodinia mix {args.mix} (bounded CPU sample)",
                   "policy": "mgb-warps (C port of schedulers.py)", "cpu_threads": threads},
        "cpu_baseline": {"value": round(v, 4), "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample_desc},
        "e2e": {"value": round(v, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--policy", default="mgb-warps")
    ap.add_argument("--mix", default="3:1")
    ap.add_argument("--jobs", type=int, default=32)
    ap.add_argument("--workers", type=int, default=8)
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-sa", action="store_true")
    args = ap.parse_args()
    from paper_2107_08538_b200 import catalog as C
    from paper_2107_08538_b200.multi import dist_env, max_over_ranks, rank_mix, whole_job_rate

    rank, world, local = dist_env()

    if args.impl == "reference":
        if rank != 0:
            return 0
        reference_arm(args, C.gen_mix(args.mix, args.jobs, seed=1))
        return 0

    import torch

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2107_08538_b200 import workloads as W

    pk = peaks()
    mix = rank_mix(args.mix, args.jobs, rank)
    jobs = [m.job for m in mix]
    device = local

    # ---- device mode: inputs staged in HBM before the timed region ----
    log(f"staging {len(jobs)} jobs (device mode)")
    W.stage(jobs, [device], W.MODE_DEVICE)
    if dist:
        dist.barrier()
    with Clocks(device) as clk:
        times, results = run_steps(W, jobs, args.policy, device, args.workers, W.MODE_DEVICE, args.steps,
                                   args.warmup, torch, dist)
    ours = summarize(results, times)
    sa = None
    if not args.skip_sa:
        st, sr = run_steps(W, jobs, "sa", device, args.workers, W.MODE_DEVICE, args.steps, 1, torch, dist)
        sa = summarize(sr, st)
    W.unstage()
    kern, solo_ms = kernel_rooflines(W, C, mix, device, pk)

    # ---- e2e mode: pinned host inputs, H2D + D2H inside the timed region ----
    e2e = sa_e2e = None
    if not args.skip_e2e:
        log("staging (e2e mode: pinned host inputs)")
        W.stage(jobs, [device], W.MODE_E2E)
        et, er = run_steps(W, jobs, args.policy, device, args.workers, W.MODE_E2E, args.steps, 1, torch, dist)
        e2e = summarize(er, et)
        e2e["h2d"] = sum(r["h2d_bytes"] for r in er[-1].records)
        e2e["d2h"] = sum(r["d2h_bytes"] for r in er[-1].records)
        if not args.skip_sa:
            st2, sr2 = run_steps(W, jobs, "sa", device, args.workers, W.MODE_E2E, args.steps, 1, torch, dist)
            sa_e2e = summarize(sr2, st2)
        W.unstage()

    # ---- max over ranks ----
    ms_step = ours["ms_per_step"]
    e2e_ms = e2e["ms_per_step"] if e2e else None
    ms_step, e2e_max, sa_max, sa_e2e_max = max_over_ranks(
        [ms_step, e2e_ms or 0.0, sa["ms_per_step"] if sa else 0.0, sa_e2e["ms_per_step"] if sa_e2e else 0.0],
        dist, device="cuda")
    e2e_ms = e2e_max or None
    if sa:
        sa["ms_per_step"] = sa_max
    if sa_e2e:
        sa_e2e["ms_per_step"] = sa_e2e_max
    n_total = len(jobs) * world
    value = whole_job_rate(len(jobs), world, ms_step)

    # dominant kernel: the kind with the largest share of device time in the mix
    # dominant kind: the largest share of the mix's solo device time
    share = {}
    for mj in mix:
        share[mj.job.kind] = share.get(mj.job.kind, 0.0) + solo_ms[mj.template]
    dom = max(share, key=share.get)
    kd = kern[dom]
    tr = traffic_from_profiles(dom) or {}
    roof = {"kernel": dom, "bound": kd["bound"], "achieved": kd["achieved"], "peak": kd["peak"],
            "unit": kd["unit"], "frac": kd["frac"], "traffic": tr.get("dram_bytes_per_launch"),
            "traffic_kernel": tr.get("kernel"), "algorithmic_bytes_per_launch": tr.get("algorithmic_bytes_per_launch"),
            "share_of_mix_solo_device_time": round(share[dom] / sum(share.values()), 3),
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)" if kd["bound"] == "hbm"
            else "nominal FP32 (148 SMs x 128 FMA x 1.965 GHz)"}
    # aggregate HBM roofline fraction of the whole mix
    mix_bytes = sum(C.algorithmic_work(j)[0] for j in jobs if C.algorithmic_work(j)[1] == "B")
    mix_frac = mix_bytes / (ms_step / 1000.0) / 1e9 / pk["hbm_gbs"]

    line = {
        "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 2), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32/i32", "data": "synthetic (seeded hash inputs)",
        "config": {"workload": f"cfg1: {args.jobs}-job Rodinia mix {args.mix} per GPU "
                               "(bfs/hotspot/srad/kmeans/backprop/needle/lud)",
                   "policy": args.policy, "workers_per_gpu": args.workers,
                   "inputs": "staged in HBM, larger than L2 (no flush needed)", "parallelism": f"placement x{world}"},
        "mean_turnaround_ms": round(ours["mean_turnaround_ms"], 2),
        "mean_wait_ms": round(ours["mean_wait_ms"], 2),
        "oom": ours["oom"], "crashed": ours["crashed"],
        "gpu_launches": ours["kernel_launches"] + ours["decision_launches"],
        "decision_launches": ours["decision_launches"],
        "decision_ms_per_step": round(ours["decision_ms"] / args.steps, 3),
        "roofline": roof,
        "mix_hbm_frac": round(mix_frac, 4),
        "kernels": kern,
    }
    if sa:
        sa_value = n_total / (sa["ms_per_step"] / 1000.0)
        line["sa"] = {"value": round(sa_value, 4), "ms_per_step": round(sa["ms_per_step"], 2),
                      "mean_turnaround_ms": round(sa["mean_turnaround_ms"], 2), "oom": sa["oom"]}
        line["speedup_vs_sa"] = round(value / sa_value, 3)
        line["turnaround_speedup_vs_sa"] = round(sa["mean_turnaround_ms"] / max(ours["mean_turnaround_ms"], 1e-9), 3)
    if e2e:
        pcie = pcie_h2d_gbps(torch)
        h2d_rate = e2e["h2d"] / (e2e_ms / 1000.0) / 1e9
        line["e2e"] = {"value": round(n_total / (e2e_ms / 1000.0), 4), "unit": UNIT,
                       "h2d_bytes_per_step": e2e["h2d"], "d2h_bytes_per_step": e2e["d2h"],
                       "mean_turnaround_ms": round(e2e["mean_turnaround_ms"], 2), "oom": e2e["oom"],
                       "pcie_h2d_achieved_GBps": round(h2d_rate, 1), "pcie_h2d_peak_GBps": round(pcie, 1),
                       "pcie_h2d_frac": round(h2d_rate / pcie, 3)}
        if sa_e2e:
            sv = n_total / (sa_e2e["ms_per_step"] / 1000.0)
            line["e2e"]["sa_value"] = round(sv, 4)
            line["e2e"]["speedup_vs_sa"] = round(line["e2e"]["value"] / sv, 3)
    line["clocks"] = clk.summary()
    if rank == 0:
        rate, n, names, dt = cpu_sample(mix, args.cpu_budget)
        line["cpu_baseline"] = {"value": round(rate, 4), "unit": UNIT, "cores": os.cpu_count() or 1,
                                "kind": "port",
                                "sample": f"{n} mix jobs ({', '.join(names)}) on the CPU restatements, "
                                          f"{dt:.1f} s, OpenMP all host threads"}
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
