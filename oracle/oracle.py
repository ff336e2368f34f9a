"""ctypes wrapper of the C oracle (libgs_oracle.so) — test infrastructure.

Exposes OracleDevice / OracleScheduler with the same call shapes the replay
harness (tests/replay.py) drives on the product's drop-in classes.  Parity
of this oracle with the reference is pinned by tests/test_oracle_golden.py
against event streams recorded from the reference itself.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import zlib
from ctypes import POINTER, c_int32, c_int64, c_void_p

import numpy as np

from paper_2107_08538_b200 import _native as nat  # structs only (no libgs load)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libgs_oracle.so")


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE, "libgs_oracle.so"], check=True)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = ctypes.CDLL(LIB)
        sig = {
            "o_dev_new": (c_void_p, [POINTER(nat.GsSpec), c_int32]),
            "o_dev_free": (None, [c_void_p]),
            "o_ledger": (None, [c_void_p, POINTER(c_int64)]),
            "o_set_ledger": (None, [c_void_p, POINTER(c_int64)]),
            "o_sm_array": (c_void_p, [c_void_p, c_int32]),
            "o_is_resident": (c_int32, [c_void_p, c_int32]),
            "o_occupancy_limit_per_sm": (c_int64, [POINTER(nat.GsSpec), POINTER(nat.GsProbe)]),
            "o_try_place": (c_int32, [c_void_p, POINTER(nat.GsProbe), c_void_p, POINTER(c_int32),
                                      POINTER(c_int64)]),
            "o_commit": (c_int32, [c_void_p, c_int32, POINTER(nat.GsProbe), c_void_p, c_int32, c_int64]),
            "o_reserve": (c_int32, [c_void_p, c_int64]),
            "o_assign": (None, [c_void_p, c_int32, c_int64]),
            "o_add_warps": (None, [c_void_p, c_int32, c_int64]),
            "o_alloc_raw": (c_int32, [c_void_p, c_int32, c_int64]),
            "o_release": (c_int32, [c_void_p, c_int32, POINTER(c_int64)]),
            "o_check": (c_int32, [c_void_p, POINTER(c_int32), POINTER(c_int64), POINTER(c_int64)]),
            "o_sched_new": (c_void_p, [c_void_p, c_int32, c_int32, c_int32, c_int32]),
            "o_sched_free": (None, [c_void_p]),
            "o_pending_count": (c_int32, [c_void_p]),
            "o_submit": (c_int32, [c_void_p, POINTER(nat.GsProbe), POINTER(nat.GsDecision)]),
            "o_on_release": (c_int32, [c_void_p, c_void_p, c_int32, POINTER(c_int32), POINTER(c_int32)]),
            "o_job_ended": (None, [c_void_p, c_int32]),
            "o_job_state": (None, [c_void_p, c_void_p, c_void_p, POINTER(c_int32)]),
            "o_sweep": (c_int32, [c_void_p, c_void_p, c_int32, c_int32, c_void_p, c_int64,
                                  POINTER(c_int64)]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def spec_struct(spec) -> nat.GsSpec:
    return nat.GsSpec(int(spec.sm_count), int(spec.mem_bytes), int(spec.max_warps_per_sm),
                      int(spec.max_tbs_per_sm), int(spec.regs_per_sm), int(spec.smem_per_sm_bytes))


def probe_struct(res, handle=0, job=-1, level=0) -> nat.GsProbe:
    return nat.GsProbe(int(res.mem_bytes), int(res.heap_limit_bytes), int(res.total_warps),
                       float(res.est_duration_ms), int(res.thread_blocks), int(res.warps_per_block),
                       int(res.threads_per_block), int(res.regs_per_thread), int(res.smem_per_block),
                       handle, job, level)


def sm_crc(arrays) -> int:
    """crc32 over sm_warps|sm_tbs|sm_regs|sm_smem as little-endian int32."""
    buf = b"".join(np.asarray(a, dtype="<i4").tobytes() for a in arrays)
    return zlib.crc32(buf)


class OracleDevice:
    def __init__(self, spec, index=0):
        self.spec = spec
        self.index = index
        self.L = lib()
        self.ptr = self.L.o_dev_new(ctypes.byref(spec_struct(spec)), index)
        n = int(spec.sm_count)
        self.arrays = [np.ctypeslib.as_array((ctypes.c_int32 * n).from_address(self.L.o_sm_array(self.ptr, w)))
                       for w in range(4)]

    def __del__(self):
        try:
            self.L.o_dev_free(self.ptr)
        except Exception:
            pass

    def ledger(self):
        out = (c_int64 * 4)()
        self.L.o_ledger(self.ptr, out)
        return list(out)

    def snapshot(self):
        free, warps, version, cursor = self.ledger()
        return [free, warps, cursor, version, sm_crc(self.arrays)]


class OracleScheduler:
    def __init__(self, devices, policy_code, cg_ratio, skip_ahead):
        self.L = lib()
        self.devices = devices
        arr = (c_void_p * len(devices))(*[d.ptr for d in devices])
        self.ptr = self.L.o_sched_new(arr, len(devices), policy_code, cg_ratio, 1 if skip_ahead else 0)

    def __del__(self):
        try:
            self.L.o_sched_free(self.ptr)
        except Exception:
            pass

    def submit(self, probe):
        out = nat.GsDecision()
        self.L.o_submit(self.ptr, ctypes.byref(probe), ctypes.byref(out))
        return out

    def on_release(self):
        n = self.L.o_pending_count(self.ptr)
        out = np.zeros(max(n, 1), dtype=nat.DECISION_DTYPE)
        tried, adm = c_int32(), c_int32()
        self.L.o_on_release(self.ptr, out.ctypes.data, n, ctypes.byref(tried), ctypes.byref(adm))
        return out[: tried.value]

    def sweep(self, probes: np.ndarray, max_resident: int):
        n = len(probes)
        cap = 2 * n + 16
        ev = np.zeros((cap, 3), dtype=np.int32)
        ne = c_int64()
        self.L.o_sweep(self.ptr, probes.ctypes.data, n, max_resident, ev.ctypes.data, cap, ctypes.byref(ne))
        return ev[: ne.value]


class _Spec:
    def __init__(self, s):
        for f in ("sm_count", "mem_bytes", "max_warps_per_sm", "max_tbs_per_sm", "regs_per_sm",
                  "smem_per_sm_bytes"):
            setattr(self, f, int(getattr(s, f)))


def replay_exec_log(log) -> tuple[int, list[str]]:
    """Replay an executor placement log (workloads.exec_log()) through the
    oracle Scheduler (the golden-pinned C restatement of schedulers.py:89-123
    and device_model.py:192-209) and compare every decision: submits
    (outcome, device), releases (status, freed bytes) and each re-drive's
    tried list (handle, outcome, device) in FIFO order.  Returns (decisions
    checked, mismatch descriptions)."""
    devs = [OracleDevice(_Spec(s), i) for i, s in enumerate(log.specs)]
    sched = OracleScheduler(devs, log.policy, log.cg_ratio, True)
    L = lib()
    evs = log.events
    checked, bad = 0, []
    i = 0
    while i < len(evs):
        e = evs[i]
        if e.kind == 0:  # submit
            d = sched.submit(e.probe)
            got = (e.outcome, e.device if e.outcome == 0 else -1)
            want = (d.outcome, d.device if d.outcome == 0 else -1)
            checked += 1
            if got != want:
                bad.append(f"event {i} submit h{e.handle}: gpu {got} oracle {want}")
            i += 1
            continue
        if e.kind in (1, 2):
            if e.kind == 1:
                freed = c_int64()
                st = L.o_release(devs[e.device].ptr, e.handle, ctypes.byref(freed))
                checked += 1
                if (st, freed.value) != (e.outcome, e.freed):
                    bad.append(f"event {i} release h{e.handle}: gpu {(e.outcome, e.freed)} oracle {(st, freed.value)}")
            else:
                L.o_job_ended(sched.ptr, e.handle)
            drained = sched.on_release()
            j = i + 1
            got = []
            while j < len(evs) and evs[j].kind == 3:
                got.append((evs[j].handle, evs[j].outcome, evs[j].device if evs[j].outcome == 0 else -1))
                j += 1
            want = [(int(r["handle"]), int(r["outcome"]), int(r["device"]) if r["outcome"] == 0 else -1)
                    for r in drained]
            checked += len(want)
            if got != want:
                bad.append(f"event {i} re-drive after h{e.handle}: gpu {got} oracle {want}")
            i = j
            continue
        bad.append(f"event {i}: unexpected kind {e.kind}")
        i += 1
    return checked, bad
