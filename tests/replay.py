"""Golden event-stream replay (parity harness).

The streams in tests/golden/ were recorded from the reference placement
path driven by the reference's own SimEngine (tests/golden/make_golden.py).
`replay_run` pushes one recorded run through a backend and demands, event by
event, identical decisions, plans, freed bytes, errors, decision-log rows,
pending queues and post-call ledger snapshots of every device.

Backends:
  DropinBackend  the product: paper_2107_08538_b200.gpushare on the GPU
  OracleBackend  the C restatement in oracle/ (CPU; checker only)
"""

from __future__ import annotations

import gzip
import json
import os
import zlib
from collections import deque

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
POLICY_CODES = {"sa": 0, "cg": 1, "mgb-sm": 2, "mgb-warps": 3}


def load_sim_runs(limit: int | None = None):
    with gzip.open(os.path.join(GOLDEN, "sim_streams.jsonl.gz"), "rt") as f:
        for i, line in enumerate(f):
            if limit is not None and i >= limit:
                return
            yield json.loads(line)


def load_sweeps() -> dict:
    return dict(np.load(os.path.join(GOLDEN, "sweeps.npz")))


def sm_crc(arrays) -> int:
    return zlib.crc32(b"".join(np.asarray(a, dtype="<i4").tobytes() for a in arrays))


def conservation_message(kind, sm, index, free, held, cap, in_use, warps_sum, arrays) -> str:
    """The reference's messages (device_model.py:224-245)."""
    if kind == 1:
        return f"device {index}: free {free} + held {held} != capacity {cap}"
    if kind == 2:
        return f"device {index}: warp ledger {in_use} != sum of residents {warps_sum}"
    arr, what = {3: (arrays[1], "blocks"), 4: (arrays[0], "warps"),
                 5: (arrays[2], "regs"), 6: (arrays[3], "smem")}[kind]
    return f"device {index} sm {sm}: {int(arr[sm])} {what}"


class _Res:
    __slots__ = ("mem_bytes", "heap_limit_bytes", "thread_blocks", "warps_per_block",
                 "total_warps", "threads_per_block", "regs_per_thread", "smem_per_block",
                 "est_duration_ms")

    def __init__(self, vals):
        for k, v in zip(self.__slots__, vals):
            setattr(self, k, v)


# -- backends -----------------------------------------------------------------


class DropinBackend:
    """Drives the product's public drop-in API (GPU)."""

    def __init__(self, ring: bool = False):
        from paper_2107_08538_b200 import gpushare as G

        self.G = G
        self.devs = []
        self.sched = None
        self.log = None
        self.ring = ring

    def dev(self, spec, index):
        self.devs.append(self.G.DeviceState(self.G.DeviceSpec(*spec), index))

    def make_sched(self, devs, policy, cg, skip, log):
        self.log = [] if log else None
        pol = self.G.PolicyConfig(policy, cg)
        self.sched = self.G.Scheduler([self.devs[k] for k in devs], pol, skip_ahead=skip, log=self.log)
        if self.ring:
            self.sched.start_ring()

    def close(self):
        if self.ring and self.sched is not None:
            self.sched.stop_ring()

    def submit(self, job, uid, res, level, t, now):
        n0 = len(self.log) if self.log is not None else 0
        req = self.G.ScheduleRequest(job, uid, self.G.ResourceRequest(*res), level, t)
        d = self.sched.submit(req, now)
        return [d.outcome, d.device], (self.log[n0:] if self.log is not None else None)

    def on_release(self, now):
        n0 = len(self.log) if self.log is not None else 0
        adm = self.sched.on_release(now)
        return ([[r.task_uid, d] for r, d in adm], [r.task_uid for r in self.sched.pending],
                self.log[n0:] if self.log is not None else None)

    def job_ended(self, job):
        self.sched.job_ended(job)

    def release(self, k, uid):
        try:
            return self.devs[k].release_task(uid), None
        except self.G.ContractViolation as e:
            return None, str(e)

    def alloc_raw(self, k, uid, n):
        return self.devs[k].allocate_raw(uid, n)

    def check(self, k):
        try:
            self.devs[k].check_conservation()
            return None
        except self.G.ContractViolation as e:
            return str(e)

    def try_place(self, k, res):
        plan = self.devs[k].try_place_blocks(_Res(res))
        return None if plan is None else [list(plan.blocks_per_sm), plan.final_cursor, plan.version]

    def snapshot(self, k):
        d = self.devs[k]
        return [d.free_mem, d.in_use_warps, d.rr_cursor, d.version,
                sm_crc((d.sm_warps, d.sm_tbs, d.sm_regs, d.sm_smem))]


class OracleBackend:
    """Drives the C oracle with the reference's bookkeeping (CPU)."""

    def __init__(self):
        import ctypes

        from oracle import oracle as O

        self.O = O
        self.ct = ctypes
        self.devs = []
        self.sched = None
        self.uids: dict = {}
        self.jobs: dict = {}
        self.pending = deque()
        self.log = None
        self.policy = None

    def _h(self, uid):
        return self.uids.setdefault(uid, len(self.uids))

    def _j(self, job):
        return self.jobs.setdefault(job, len(self.jobs))

    def dev(self, spec, index):
        from paper_2107_08538_b200.gpushare.device_model import DeviceSpec

        self.devs.append(self.O.OracleDevice(DeviceSpec(*spec), index))

    def make_sched(self, devs, policy, cg, skip, log):
        self.log = [] if log else None
        self.policy = (policy, cg)
        self.sched = self.O.OracleScheduler([self.devs[k] for k in devs], POLICY_CODES[policy], cg, skip)

    def _row(self, now, job, uid, mem, outcome, dev, free_after, warps_after):
        label = f"cg:{self.policy[1]}" if self.policy[0] == "cg" else self.policy[0]
        return {"time_ms": now, "job_id": job, "task": uid, "policy": label, "outcome": outcome,
                "device": dev, "mem_bytes": mem,
                "free_mem_after": free_after if dev is not None else None,
                "in_use_warps_after": warps_after if dev is not None else None}

    def submit(self, job, uid, res, level, t, now):
        names = {0: "assign", 1: "defer", 2: "reject"}
        probe = self.O.probe_struct(_Res(res), self._h(uid), self._j(job), 1 if level == "job" else 0)
        d = self.sched.submit(probe)
        outcome = names[d.outcome]
        dev = d.device if d.outcome == 0 else None
        if d.outcome == 1:
            self.pending.append((job, uid, res[0]))
        rows = None
        if self.log is not None:
            rows = [self._row(now, job, uid, res[0], outcome, dev, d.free_mem_after, d.in_use_warps_after)]
        return [outcome, dev], rows

    def on_release(self, now):
        names = {0: "assign", 1: "defer", 2: "reject"}
        entries = list(self.pending)
        out = self.sched.on_release()
        adm, gone, rows = [], set(), []
        for r in out:
            job, uid, mem = entries[int(r["pending_index"])]
            oc = int(r["outcome"])
            dev = int(r["device"]) if oc == 0 else None
            if oc == 0:
                adm.append([uid, dev])
                gone.add(int(r["pending_index"]))
            rows.append(self._row(now, job, uid, mem, names[oc], dev, int(r["free_mem_after"]),
                                  int(r["in_use_warps_after"])))
        self.pending = deque(e for i, e in enumerate(entries) if i not in gone)
        return adm, [e[1] for e in self.pending], (rows if self.log is not None else None)

    def job_ended(self, job):
        if job in self.jobs:
            self.O.lib().o_job_ended(self.sched.ptr, self.jobs[job])

    def release(self, k, uid):
        L = self.O.lib()
        d = self.devs[k]
        h = self.uids.get(uid)
        freed = self.ct.c_int64()
        if h is None or L.o_release(d.ptr, h, self.ct.byref(freed)) != 0:
            return None, f"release of unknown task {uid!r} on device {d.index}"
        return freed.value, None

    def alloc_raw(self, k, uid, n):
        return self.O.lib().o_alloc_raw(self.devs[k].ptr, self._h(uid), n) == 0

    def check(self, k):
        d = self.devs[k]
        sm, held, warps = self.ct.c_int32(), self.ct.c_int64(), self.ct.c_int64()
        kind = self.O.lib().o_check(d.ptr, self.ct.byref(sm), self.ct.byref(held), self.ct.byref(warps))
        if kind == 0:
            return None
        free, in_use, _, _ = d.ledger()
        return conservation_message(kind, sm.value, d.index, free, held.value, d.spec.mem_bytes,
                                    in_use, warps.value, d.arrays)

    def try_place(self, k, res):
        d = self.devs[k]
        n = int(d.spec.sm_count)
        blocks = np.zeros(n, dtype=np.int32)
        cur, ver = self.ct.c_int32(), self.ct.c_int64()
        rc = self.O.lib().o_try_place(d.ptr, self.ct.byref(self.O.probe_struct(_Res(res))), blocks.ctypes.data,
                                      self.ct.byref(cur), self.ct.byref(ver))
        return None if rc else [blocks.tolist(), cur.value, ver.value]

    def snapshot(self, k):
        return self.devs[k].snapshot()


# -- replay -------------------------------------------------------------------


def replay_run(backend, run: dict) -> int:
    """Replay one recorded run; returns the number of events checked."""
    label = run["label"]
    for i, ev in enumerate(run["events"]):
        kind = ev["e"]
        where = f"{label} event {i} ({kind})"
        if kind == "dev":
            backend.dev(ev["spec"], ev["index"])
            continue
        if kind == "sched":
            backend.make_sched(ev["devs"], ev["policy"], ev["cg"], ev["skip"], ev["log"])
            continue
        if kind == "submit":
            job, uid, res, level, t = ev["req"]
            out, rows = backend.submit(job, uid, res, level, t, ev["now"])
            assert out == ev["out"], f"{where}: decision {out} != reference {ev['out']}"
            assert rows == ev["log"], f"{where}: log {rows} != {ev['log']}"
        elif kind == "on_release":
            adm, pend, rows = backend.on_release(ev["now"])
            assert adm == ev["out"], f"{where}: admitted {adm} != {ev['out']}"
            assert pend == ev["pending"], f"{where}: pending {pend} != {ev['pending']}"
            assert rows == ev["log"], f"{where}: log mismatch"
        elif kind == "job_ended":
            backend.job_ended(ev["job"])
        elif kind == "release":
            out, err = backend.release(ev["d"], ev["uid"])
            assert err == ev.get("err"), f"{where}: error {err!r} != {ev.get('err')!r}"
            assert out == ev.get("out"), f"{where}: freed {out} != {ev.get('out')}"
        elif kind == "alloc_raw":
            out = backend.alloc_raw(ev["d"], ev["uid"], ev["n"])
            assert out == ev["out"], f"{where}: allocate_raw {out} != {ev['out']}"
        elif kind == "check":
            err = backend.check(ev["d"])
            assert err == ev["err"], f"{where}: check {err!r} != {ev['err']!r}"
        elif kind == "try_place":
            out = backend.try_place(ev["d"], ev["res"])
            assert out == ev["out"], f"{where}: plan {out} != {ev['out']}"
        else:
            raise AssertionError(f"{where}: unknown event")
        post = [backend.snapshot(k) for k in range(len(ev["post"]))]
        assert post == ev["post"], f"{where}: ledgers {post} != {ev['post']}"
    return len(run["events"])
