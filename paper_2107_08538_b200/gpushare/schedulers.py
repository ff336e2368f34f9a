"""Admission policies on the GPU (drop-in for gpushare/schedulers.py).

Scheduler keeps the reference's constructor and methods —
Scheduler(devices, policy, skip_ahead=True, log=None), submit(req, now),
on_release(now), job_ended(job_id), the `pending` deque and the decision
log — while every decision is made by libgs's sm_100a decision kernel
against the shared ledgers:

  mgb-sm     Alg. 2, first device (index order) passing memory + per-SM
             placement                               schedulers.py:137-153
  mgb-warps  Alg. 3, memory-feasible device with the fewest in-use warps,
             ties to the lower index                 schedulers.py:155-171
  sa         one job per device (the metric's baseline)    :173-178
  cg         round robin up to cg_ratio jobs per device    :180-189

The FIFO queue itself lives in HBM next to the decision kernel; `pending`
is its Python mirror (reference tests read it, tests/test_schedulers.py:81).
"""

from __future__ import annotations

import ctypes
from collections import deque
from dataclasses import dataclass

import numpy as np

from .. import _native as nat
from .device_model import DeviceState, handle_table, pack_probe
from .errors import ConfigError, ContractViolation

ASSIGN = "assign"
DEFER = "defer"
REJECT = "reject"

_OUTCOME = {nat.GS_ASSIGN: ASSIGN, nat.GS_DEFER: DEFER, nat.GS_REJECTED: REJECT}


@dataclass(frozen=True)
class PolicyConfig:
    kind: str  # sa | cg | mgb-sm | mgb-warps
    cg_ratio: int = 6

    @property
    def task_level(self) -> bool:
        return self.kind in ("mgb-sm", "mgb-warps")

    @property
    def label(self) -> str:
        return f"cg:{self.cg_ratio}" if self.kind == "cg" else self.kind


def parse_policy(text: str) -> PolicyConfig:
    """schedulers.py:40-53."""
    if text in ("sa", "mgb-sm", "mgb-warps"):
        return PolicyConfig(text)
    if text == "cg" or text.startswith("cg:"):
        ratio = 6
        if ":" in text:
            try:
                ratio = int(text.split(":", 1)[1])
            except ValueError:
                raise ConfigError(f"bad cg ratio in {text!r}") from None
        if ratio < 1:
            raise ConfigError("cg ratio must be >= 1")
        return PolicyConfig("cg", ratio)
    raise ConfigError(f"unknown scheduling policy {text!r}")


@dataclass(frozen=True)
class ScheduleRequest:
    job_id: str
    task_uid: str
    resources: object  # ResourceRequest
    level: str  # "task" or "job"
    submitted_ms: float


@dataclass(frozen=True)
class Decision:
    outcome: str
    device: int | None = None


def _destroy_sched(lib, ptr) -> None:
    lib.gs_sched_destroy(ptr)


class Scheduler:
    """schedulers.py:71-218 with the decisions made on the GPU."""

    def __init__(self, devices: list[DeviceState], policy: PolicyConfig,
                 skip_ahead: bool = True, log: list[dict] | None = None):
        self.devices = devices
        self.policy = policy
        self.skip_ahead = skip_ahead
        self.log = log
        self.pending: deque = deque()
        if not devices:
            raise ConfigError("a scheduler needs at least one device")
        eng = nat.engine()
        self._lib = eng.lib
        self._handles = handle_table()
        self._jobs: dict[str, int] = {}
        self._job_names: list[str] = []
        arr = (ctypes.c_void_p * len(devices))(*[d._ptr.value for d in devices])
        ptr = ctypes.c_void_p()
        code = nat.POLICY_CODES.get(policy.kind)
        if code is None:
            raise ConfigError(f"unknown scheduling policy {policy.kind!r}")
        rc = self._lib.gs_sched_create(eng.ptr, arr, len(devices), code, int(policy.cg_ratio),
                                       1 if skip_ahead else 0, ctypes.byref(ptr))
        if rc == nat.GS_ERR_CONFIG:
            raise ConfigError(nat.last_error())
        nat.check(rc)
        self._ptr = ptr
        self._dec = nat.GsDecision()
        import weakref

        self._finalizer = weakref.finalize(self, _destroy_sched, self._lib, ptr)

    # -- persistent decision kernel ---------------------------------------------

    def start_ring(self, max_pending: int = 4096, max_handles: int = 4096, max_jobs: int = 4096) -> None:
        """Serve this scheduler's calls from a resident decision warp over a
        pinned host-mapped command ring (include/gs.h gs_sched_ring_start).
        While it runs, ledgers must only change through the API."""
        nat.check(self._lib.gs_sched_ring_start(self._ptr, max_pending, max_handles, max_jobs))

    def stop_ring(self) -> None:
        nat.check(self._lib.gs_sched_ring_stop(self._ptr))

    # -- job-granular state mirrors ------------------------------------------

    def _job_state(self):
        n = len(self.devices)
        owner = np.zeros(n, dtype=np.int32)
        counts = np.zeros(n, dtype=np.int32)
        cur = ctypes.c_int32()
        self._lib.gs_sched_job_state(self._ptr, owner.ctypes.data, counts.ctypes.data,
                                     ctypes.byref(cur))
        return owner, counts, cur.value

    @property
    def sa_owner(self) -> dict[int, str]:
        owner, _, _ = self._job_state()
        return {i: self._job_names[j] for i, j in enumerate(owner) if j >= 0}

    @property
    def cg_counts(self) -> list[int]:
        return [int(c) for c in self._job_state()[1]]

    @property
    def cg_cursor(self) -> int:
        return self._job_state()[2]

    def _job(self, job_id: str) -> int:
        j = self._jobs.get(job_id)
        if j is None:
            j = self._jobs[job_id] = len(self._job_names)
            self._job_names.append(job_id)
        return j

    # -- admission -------------------------------------------------------------

    def submit(self, req: ScheduleRequest, now: float) -> Decision:
        """Decide a fresh request; Defer queues it (schedulers.py:89-95)."""
        uid = req.task_uid
        h = self._handles.get(uid)
        level = 1 if req.level == "job" else 0
        if not any(uid in d._resident for d in self.devices):
            level |= 2  # GS_PROBE_FRESH: no residency row to accumulate into
        probe = pack_probe(req.resources, h, self._job(req.job_id), level)
        dec = self._dec
        rc = self._lib.gs_submit(self._ptr, ctypes.byref(probe), ctypes.byref(dec))
        if rc < 0:
            self._handles.settle(uid)
            nat.check(rc)
        outcome = _OUTCOME[dec.outcome]
        device = dec.device if outcome == ASSIGN else None
        if outcome == ASSIGN and self.policy.task_level:
            self.devices[device]._mark_resident(uid, h)
        elif outcome == DEFER:
            self.pending.append(req)
            self._handles.incref(uid)
        self._handles.settle(uid)
        decision = Decision(outcome, device)
        if self.log is not None:
            self._log(now, req, decision, dec.free_mem_after, dec.in_use_warps_after)
        return decision

    def on_release(self, now: float) -> list[tuple[ScheduleRequest, int]]:
        """Re-evaluate deferred requests in FIFO order (schedulers.py:97-113)."""
        entries = list(self.pending)
        n = len(entries)
        if n != self._lib.gs_pending_count(self._ptr):
            raise ContractViolation("pending queue was modified outside the scheduler")
        out = np.zeros(max(n, 1), dtype=nat.DECISION_DTYPE)
        tried, admitted_n = ctypes.c_int32(), ctypes.c_int32()
        nat.check(self._lib.gs_on_release(self._ptr, out.ctypes.data, n, ctypes.byref(tried),
                                          ctypes.byref(admitted_n)))
        rows = out[: tried.value]
        admitted: list[tuple[ScheduleRequest, int]] = []
        gone = set()
        logging = self.log is not None
        task_level = self.policy.task_level
        for k in range(tried.value):
            oc = int(rows["outcome"][k])
            if oc != nat.GS_ASSIGN and not logging:
                continue
            idx = int(rows["pending_index"][k])
            req = entries[idx]
            if oc == nat.GS_ASSIGN:
                dev = int(rows["device"][k])
                if task_level:
                    self.devices[dev]._mark_resident(req.task_uid, self._handles.get(req.task_uid))
                self._handles.decref(req.task_uid)
                gone.add(idx)
                admitted.append((req, dev))
                if logging:
                    self._log(now, req, Decision(ASSIGN, dev), int(rows["free_mem_after"][k]),
                              int(rows["in_use_warps_after"][k]))
            else:
                self._log(now, req, Decision(_OUTCOME[oc]), 0, 0)
        if gone:
            self.pending.clear()
            self.pending.extend(e for i, e in enumerate(entries) if i not in gone)
        return admitted

    def job_ended(self, job_id: str) -> None:
        """Release job-granular claims (schedulers.py:115-123)."""
        j = self._jobs.get(job_id)
        if j is None:
            return
        nat.check(self._lib.gs_job_ended(self._ptr, j))

    # -- logging ---------------------------------------------------------------

    def _log(self, now: float, req: ScheduleRequest, decision: Decision,
             free_after: int, warps_after: int) -> None:
        """Decision-log row (schedulers.py:203-218), same 9 keys."""
        has = decision.device is not None
        self.log.append({
            "time_ms": now,
            "job_id": req.job_id,
            "task": req.task_uid,
            "policy": self.policy.label,
            "outcome": decision.outcome,
            "device": decision.device,
            "mem_bytes": req.resources.mem_bytes,
            "free_mem_after": free_after if has else None,
            "in_use_warps_after": warps_after if has else None,
        })
