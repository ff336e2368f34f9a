"""Record golden event streams from the reference placement path.

Run in the build container (the reference is importable only here):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the UNMODIFIED reference package read-only from
/root/reference/pkg/src, wraps its DeviceState / Scheduler in recording
subclasses, and drives them through the reference's own SimEngine
(gpushare/sim_engine.py: the hot path's caller) and through the cfg 4
placement sweep.  Every top-level call into the hot path is written out
with its inputs, its outputs (decisions, plans, freed bytes, log rows,
errors) and post-call ledger snapshots of every device:

    [free_mem, in_use_warps, rr_cursor, version, crc32(sm arrays)]

tests/replay.py replays these streams through the GPU drop-in (pytest -m
gpu) and through the C oracle (CPU suite), demanding exact equality.
"""

from __future__ import annotations

import gzip
import json
import os
import random
import sys
import zlib

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REF)
sys.path.insert(0, os.path.join(REF, "..", "tests"))
sys.path.insert(0, REPO)

import gpushare.device_model as DM  # noqa: E402
import gpushare.schedulers as S  # noqa: E402
import gpushare.sim_engine as SE  # noqa: E402
from gpushare.errors import ContractViolation  # noqa: E402
from gpushare.metrics import run_workload  # noqa: E402
from gpushare.task_builder import ResourceRequest  # noqa: E402
from gpushare.workload_gen import builtin_catalog, gen_workload, standard_workload  # noqa: E402

import randprog as rp  # noqa: E402  (reference test fixtures)

from paper_2107_08538_b200.sweep import gen_probes  # noqa: E402


def crc(dev) -> int:
    buf = b"".join(np.asarray(a, dtype="<i4").tobytes()
                   for a in (dev.sm_warps, dev.sm_tbs, dev.sm_regs, dev.sm_smem))
    return zlib.crc32(buf)


def snap(dev) -> list:
    return [dev.free_mem, dev.in_use_warps, dev.rr_cursor, dev.version, crc(dev)]


def res_list(r) -> list:
    return [r.mem_bytes, r.heap_limit_bytes, r.thread_blocks, r.warps_per_block, r.total_warps,
            r.threads_per_block, r.regs_per_thread, r.smem_per_block, r.est_duration_ms]


class Recorder:
    def __init__(self):
        self.events: list[dict] = []
        self.devs: list = []
        self.depth = 0

    def ev(self, **kw):
        kw["post"] = [snap(d) for d in self.devs]
        self.events.append(kw)

    def kid(self, dev) -> int:
        return self.devs.index(dev)


REC: Recorder | None = None


class RDev(DM.DeviceState):
    def __post_init__(self):
        super().__post_init__()
        REC.devs.append(self)
        s = self.spec
        REC.events.append({"e": "dev", "spec": [s.name, s.sm_count, s.mem_bytes, s.max_warps_per_sm,
                                                s.max_tbs_per_sm, s.regs_per_sm, s.smem_per_sm_bytes],
                           "index": self.index})

    def _top(self):
        return REC.depth == 0

    def release_task(self, task_uid):
        top = self._top()
        try:
            out = super().release_task(task_uid)
        except ContractViolation as e:
            if top:
                REC.ev(e="release", d=REC.kid(self), uid=task_uid, err=str(e))
            raise
        if top:
            REC.ev(e="release", d=REC.kid(self), uid=task_uid, out=out)
        return out

    def allocate_raw(self, task_uid, nbytes):
        top = self._top()
        out = super().allocate_raw(task_uid, nbytes)
        if top:
            REC.ev(e="alloc_raw", d=REC.kid(self), uid=task_uid, n=nbytes, out=out)
        return out

    def check_conservation(self):
        top = self._top()
        try:
            super().check_conservation()
        except ContractViolation as e:
            if top:
                REC.ev(e="check", d=REC.kid(self), err=str(e))
            raise
        if top:
            REC.ev(e="check", d=REC.kid(self), err=None)

    def try_place_blocks(self, res):
        top = self._top()
        plan = super().try_place_blocks(res)
        if top:
            REC.ev(e="try_place", d=REC.kid(self), res=res_list(res),
                   out=None if plan is None else [list(plan.blocks_per_sm), plan.final_cursor,
                                                  plan.version])
        return plan


class RSched(S.Scheduler):
    def __post_init__(self):
        super().__post_init__()
        REC.events.append({"e": "sched", "devs": [REC.kid(d) for d in self.devices],
                           "policy": self.policy.kind, "cg": self.policy.cg_ratio,
                           "skip": self.skip_ahead, "log": self.log is not None})

    def submit(self, req, now):
        n0 = len(self.log) if self.log is not None else 0
        REC.depth += 1
        try:
            d = super().submit(req, now)
        finally:
            REC.depth -= 1
        REC.ev(e="submit", req=[req.job_id, req.task_uid, res_list(req.resources), req.level,
                                req.submitted_ms], now=now, out=[d.outcome, d.device],
               log=self.log[n0:] if self.log is not None else None)
        return d

    def on_release(self, now):
        n0 = len(self.log) if self.log is not None else 0
        REC.depth += 1
        try:
            adm = super().on_release(now)
        finally:
            REC.depth -= 1
        REC.ev(e="on_release", now=now, out=[[r.task_uid, d] for r, d in adm],
               pending=[r.task_uid for r in self.pending],
               log=self.log[n0:] if self.log is not None else None)
        return adm

    def job_ended(self, job_id):
        REC.depth += 1
        try:
            super().job_ended(job_id)
        finally:
            REC.depth -= 1
        REC.ev(e="job_ended", job=job_id)


def record(fn) -> list[dict]:
    global REC
    REC = Recorder()
    orig = (SE.DeviceState, SE.Scheduler)
    SE.DeviceState, SE.Scheduler = RDev, RSched
    try:
        fn()
    finally:
        SE.DeviceState, SE.Scheduler = orig
    return REC.events


def write(name: str, runs: list[dict]) -> None:
    path = os.path.join(HERE, name)
    with gzip.open(path, "wt", compresslevel=9) as f:
        for run in runs:
            f.write(json.dumps(run, sort_keys=True) + "\n")
    n_ev = sum(len(r["events"]) for r in runs)
    print(f"{name}: {len(runs)} runs, {n_ev} events, {os.path.getsize(path)} bytes")


# -- corpora -------------------------------------------------------------------

def sim_runs() -> list[dict]:
    """The reference SimEngine driving the hot path."""
    runs = []

    def add(label, fn):
        runs.append({"label": label, "events": record(fn)})

    # safety corpus slice (acceptance criteria 3/4, test_sim_engine.py:271-280)
    for seed in range(120):
        jobs, devices, workers = rp.gen_mini_workload(seed)
        for policy in ("mgb-sm", "mgb-warps"):
            cfg = SE.SimConfig(S.parse_policy(policy), devices, workers, seed=seed,
                               check_invariants=True, collect_decision_log=True)
            add(f"mini{seed}-{policy}", lambda jobs=jobs, cfg=cfg: SE.run_sim(jobs, cfg))
    # strict FIFO (skip_ahead=False)
    for seed in range(120, 150):
        jobs, devices, workers = rp.gen_mini_workload(seed)
        for policy in ("mgb-sm", "mgb-warps"):
            cfg = SE.SimConfig(S.parse_policy(policy), devices, workers, seed=seed,
                               skip_ahead=False, collect_decision_log=True)
            add(f"strict{seed}-{policy}", lambda jobs=jobs, cfg=cfg: SE.run_sim(jobs, cfg))
    # criterion 10 workload on 2 x p100, all four policies
    p100 = [DM.device_spec("p100")] * 2
    wl = standard_workload("w3", 2)
    for policy in ("sa", "cg:3", "mgb-sm", "mgb-warps"):
        add(f"w3-p100-{policy}", lambda policy=policy: run_workload(
            wl, policy, p100, 10, 2, collect_decision_log=True))
    # cg crashes with OOM (criterion 5 setting)
    wl5 = gen_workload("3:1", 16, 3)
    add("cg6-oom", lambda: run_workload(wl5, "cg:6", p100, 6, 3, collect_decision_log=True))
    # 4 x v100, 16 workers (criterion 7 setting)
    v100 = [DM.device_spec("v100")] * 4
    wl7 = standard_workload("w7", 1)
    for policy in ("mgb-sm", "mgb-warps"):
        add(f"w7-v100-{policy}", lambda policy=policy: run_workload(
            wl7, policy, v100, 16, 1, collect_decision_log=True))
    # the B200 preset at 8 devices, 32-job std 3:1 mix
    b200 = DM.DeviceSpec("b200", sm_count=148, mem_bytes=180 * DM.GIB, smem_per_sm_bytes=228 * DM.KIB)
    wl32 = gen_workload("3:1", 32, 1)
    for policy in ("sa", "cg:6", "mgb-sm", "mgb-warps"):
        add(f"std32-b200x8-{policy}", lambda policy=policy: run_workload(
            wl32, policy, [b200] * 8, 64, 1, collect_decision_log=True, check_invariants=True))
    # neural catalog on 2 x b200 with small memory to force deferrals
    small = DM.DeviceSpec("b200s", sm_count=148, mem_bytes=3 * DM.GIB, smem_per_sm_bytes=228 * DM.KIB)
    wln = gen_workload("1:1", 16, 2, builtin_catalog("neural"))
    for policy in ("mgb-sm", "mgb-warps"):
        add(f"neural-b200s-{policy}", lambda policy=policy: run_workload(
            wln, policy, [small] * 2, 12, 2, collect_decision_log=True, check_invariants=True))
    return runs


SWEEPS = [
    # (label, fleet spec args, n_devices, n probes, seed, policy, max_resident)
    ("b200x8-warps-1k", "b200", 8, 1000, 1, "mgb-warps", 32),
    ("b200x8-sm-1k", "b200", 8, 1000, 1, "mgb-sm", 32),
    ("b200x8-warps-10k", "b200", 8, 10000, 2, "mgb-warps", 32),
    ("b200x8-sm-10k", "b200", 8, 10000, 2, "mgb-sm", 32),
    ("b200x2-sm-3k", "b200", 2, 3000, 3, "mgb-sm", 32),
    ("b200x2-warps-3k", "b200", 2, 3000, 3, "mgb-warps", 32),
    ("p100x2-sm-2k", "p100", 2, 2000, 4, "mgb-sm", 8),
    ("p100x2-warps-2k", "p100", 2, 2000, 4, "mgb-warps", 8),
]


def fleet_spec(name: str) -> DM.DeviceSpec:
    if name == "b200":
        return DM.DeviceSpec("b200", sm_count=148, mem_bytes=180 * DM.GIB, smem_per_sm_bytes=228 * DM.KIB)
    return DM.device_spec(name)


def sweep_reference(spec, n_dev, probes, policy, max_resident) -> np.ndarray:
    """The cfg 4 driver over the reference Scheduler (mirrors gs_sweep)."""
    devices = [DM.DeviceState(spec, i) for i in range(n_dev)]
    sched = S.Scheduler(devices, S.parse_policy(policy))
    fifo: list = []
    head = 0
    events = []
    for i, p in enumerate(probes):
        res = ResourceRequest(int(p["mem_bytes"]), int(p["heap_limit_bytes"]), int(p["thread_blocks"]),
                              int(p["warps_per_block"]), int(p["total_warps"]),
                              int(p["threads_per_block"]), int(p["regs_per_thread"]),
                              int(p["smem_per_block"]), float(p["est_duration_ms"]))
        uid = i
        d = sched.submit(S.ScheduleRequest("j", uid, res, "task", 0.0), 0.0)
        kind = {"assign": 0, "defer": 1, "reject": 2}[d.outcome]
        events.append((kind, i, d.device if d.device is not None else -1))
        if d.outcome == "assign":
            fifo.append((d.device, uid))
        if len(fifo) - head > max_resident or sched.pending:
            if len(fifo) > head:
                dev, u = fifo[head]
                head += 1
                devices[dev].release_task(u)
            for req, dev in sched.on_release(0.0):
                events.append((3, req.task_uid, dev))
                fifo.append((dev, req.task_uid))
    return np.asarray(events, dtype=np.int32).reshape(-1, 3), devices


def sweep_runs() -> dict:
    out = {}
    for label, fname, n_dev, n, seed, policy, max_res in SWEEPS:
        spec = fleet_spec(fname)
        probes = gen_probes(n, seed)
        ev, devices = sweep_reference(spec, n_dev, probes, policy, max_res)
        out[label] = ev
        out[label + ".meta"] = np.array([n_dev, n, seed, max_res, 0 if policy == "mgb-warps" else 1,
                                         spec.sm_count, spec.mem_bytes, spec.max_warps_per_sm,
                                         spec.max_tbs_per_sm, spec.regs_per_sm, spec.smem_per_sm_bytes],
                                        dtype=np.int64)
        out[label + ".final"] = np.array([snap(d) for d in devices], dtype=np.int64)
        print(f"sweep {label}: {len(ev)} events")
    return out


def main() -> None:
    random.seed(0)
    write("sim_streams.jsonl.gz", sim_runs())
    sw = sweep_runs()
    np.savez_compressed(os.path.join(HERE, "sweeps.npz"), **sw)
    print("sweeps.npz", os.path.getsize(os.path.join(HERE, "sweeps.npz")), "bytes")


if __name__ == "__main__":
    main()
