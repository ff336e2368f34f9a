"""Device ledgers backed by libgs (drop-in for gpushare/device_model.py).

DeviceState keeps the reference's attribute surface (free_mem, in_use_warps,
rr_cursor, version, sm_warps/sm_tbs/sm_regs/sm_smem, resident) but the bytes
live in pinned host-mapped memory owned by libgs: the decision kernels stage
exactly these bytes, and host reads/writes (including the tests' deliberate
corruption, reference tests/test_device_model.py:159-170) hit the same
memory.  Every mutation — placement planning, commits, reservations,
releases, conservation audits — runs on the GPU (csrc/gs_sched.cu).
"""

from __future__ import annotations

import ctypes
import weakref
from collections.abc import Mapping
from dataclasses import dataclass

import numpy as np

from .. import _native as nat
from .errors import ConfigError, ContractViolation

KIB = 1024
MIB = 1024 * KIB
GIB = 1024 * MIB


@dataclass(frozen=True)
class DeviceSpec:
    """device_model.py:22-30 (identical fields and defaults)."""

    name: str
    sm_count: int
    mem_bytes: int
    max_warps_per_sm: int = 64
    max_tbs_per_sm: int = 32
    regs_per_sm: int = 65536
    smem_per_sm_bytes: int = 96 * KIB


PRESETS = {
    "p100": DeviceSpec("p100", sm_count=56, mem_bytes=16 * GIB, smem_per_sm_bytes=64 * KIB),
    "v100": DeviceSpec("v100", sm_count=80, mem_bytes=16 * GIB, smem_per_sm_bytes=96 * KIB),
    # 148 SMs, 2048 threads/SM, 32 TBs/SM, 64K regs,
    # 228 KiB smem per SM, 180 GB HBM3e (BASELINE cfg 2).
    "b200": DeviceSpec("b200", sm_count=148, mem_bytes=180 * GIB, smem_per_sm_bytes=228 * KIB),
}


def device_spec(name: str) -> DeviceSpec:
    try:
        return PRESETS[name]
    except KeyError:
        raise ConfigError(f"unknown device preset {name!r}") from None


def occupancy_limit_per_sm(spec: DeviceSpec, res) -> int:
    """Max blocks of this shape one empty SM hosts (device_model.py:48-58)."""
    limits = [spec.max_tbs_per_sm]
    if res.warps_per_block > 0:
        limits.append(spec.max_warps_per_sm // res.warps_per_block)
    regs_per_block = res.regs_per_thread * res.threads_per_block
    if regs_per_block > 0:
        limits.append(spec.regs_per_sm // regs_per_block)
    if res.smem_per_block > 0:
        limits.append(spec.smem_per_sm_bytes // res.smem_per_block)
    return max(0, min(limits))


@dataclass(frozen=True)
class PlacementPlan:
    """Pure result of try_place_blocks (device_model.py:61-66)."""

    blocks_per_sm: tuple[int, ...]
    final_cursor: int
    version: int


@dataclass
class _Residency:
    """Snapshot of one resident task's row (device_model.py:69-77)."""

    task_uid: str
    mem_bytes: int = 0
    warps: int = 0
    blocks_per_sm: list[int] | None = None
    regs_per_block: int = 0
    smem_per_block: int = 0
    warps_per_block: int = 0


_I32 = (-(2**31), 2**31 - 1)
_I64 = (-(2**63), 2**63 - 1)


def _i32(name: str, v) -> int:
    v = int(v)
    if not _I32[0] <= v <= _I32[1]:
        raise ConfigError(f"{name}={v} does not fit the 64-byte probe record (int32)")
    return v


def _i64(name: str, v) -> int:
    v = int(v)
    if not _I64[0] <= v <= _I64[1]:
        raise ConfigError(f"{name}={v} does not fit int64")
    return v


def pack_probe(res, handle: int = 0, job: int = -1, level: int = 0) -> nat.GsProbe:
    """ResourceRequest -> 64 B gs_probe (duck-typed: reference objects work)."""
    return nat.GsProbe(
        _i64("mem_bytes", res.mem_bytes), _i64("heap_limit_bytes", res.heap_limit_bytes),
        _i64("total_warps", res.total_warps), float(res.est_duration_ms),
        _i32("thread_blocks", res.thread_blocks), _i32("warps_per_block", res.warps_per_block),
        _i32("threads_per_block", res.threads_per_block),
        _i32("regs_per_thread", res.regs_per_thread), _i32("smem_per_block", res.smem_per_block),
        handle, job, level)


class HandleTable:
    """Interns task uids to int32 residency handles.

    A handle stays live while some device holds a residency row for the uid
    or a pending request names it; it is recycled afterwards.
    """

    def __init__(self, eng: nat.Engine):
        self.eng = eng
        self.h: dict[str, int] = {}
        self.ref: dict[str, int] = {}
        self.free: list[int] = []
        self.next = 0

    def get(self, uid: str) -> int:
        h = self.h.get(uid)
        if h is None:
            if self.free:
                h = self.free.pop()
            else:
                h = self.next
                self.next += 1
                self.eng.reserve_handles(self.next)
            self.h[uid] = h
            self.ref[uid] = 0
        return h

    def incref(self, uid: str) -> None:
        self.ref[uid] += 1

    def decref(self, uid: str) -> None:
        self.ref[uid] -= 1
        self.settle(uid)

    def settle(self, uid: str) -> None:
        if self.ref.get(uid) == 0:
            del self.ref[uid]
            self.free.append(self.h.pop(uid))


_tables: dict[int, HandleTable] = {}


def handle_table() -> HandleTable:
    eng = nat.engine()
    t = _tables.get(id(eng))
    if t is None:
        t = _tables[id(eng)] = HandleTable(eng)
    return t


class _ResidentView(Mapping):
    """Read-only mapping uid -> _Residency of one device (rows fetched on access)."""

    def __init__(self, dev: "DeviceState"):
        self._dev = dev

    def __getitem__(self, uid: str) -> _Residency:
        h = self._dev._resident[uid]
        row = nat.GsResidency()
        blocks = np.zeros(self._dev.spec.sm_count, dtype=np.int32)
        nat.check(self._dev._lib.gs_residency_read(self._dev._ptr, h, ctypes.byref(row),
                                                   blocks.ctypes.data))
        return _Residency(uid, row.mem_bytes, row.warps,
                          [int(x) for x in blocks] if row.has_blocks else None,
                          row.regs_per_block, row.smem_per_block, row.warps_per_block)

    def __iter__(self):
        return iter(list(self._dev._resident))

    def __len__(self) -> int:
        return len(self._dev._resident)

    def __contains__(self, uid) -> bool:
        return uid in self._dev._resident


class LedgerArray(np.ndarray):
    """Per-SM ledger array view over mapped memory; element writes from the
    host bump the device's grow epoch (the reference exposes plain lists
    that tests mutate directly, tests/test_device_model.py:168-170)."""

    _ledger = None

    def __array_finalize__(self, obj):
        self._ledger = getattr(obj, "_ledger", None)

    def __setitem__(self, key, value):
        super().__setitem__(key, value)
        if self._ledger is not None:
            self._ledger.grow_epoch += 1


def _destroy_device(lib, ptr) -> None:
    lib.gs_device_destroy(ptr)


class DeviceState:
    """device_model.py:80-245 over libgs ledgers."""

    def __init__(self, spec: DeviceSpec, index: int = 0):
        self.spec = spec
        self.index = index
        eng = nat.engine()
        self._eng = eng
        self._lib = eng.lib
        self._handles = handle_table()
        cspec = nat.GsSpec(int(spec.sm_count), int(spec.mem_bytes), int(spec.max_warps_per_sm),
                           int(spec.max_tbs_per_sm), int(spec.regs_per_sm),
                           int(spec.smem_per_sm_bytes))
        ptr = ctypes.c_void_p()
        rc = self._lib.gs_device_create(eng.ptr, ctypes.byref(cspec), int(index), ctypes.byref(ptr))
        if rc == nat.GS_ERR_CONFIG:
            raise ConfigError(nat.last_error())
        nat.check(rc)
        self._ptr = ptr
        self._led = nat.GsLedger.from_address(self._lib.gs_device_ledger(ptr))
        n = int(spec.sm_count)
        arrs = []
        for which in range(4):
            addr = self._lib.gs_device_sm_array(ptr, which)
            a = np.ctypeslib.as_array((ctypes.c_int32 * n).from_address(addr)).view(LedgerArray)
            a._ledger = self._led
            arrs.append(a)
        self._sm_warps, self._sm_tbs, self._sm_regs, self._sm_smem = arrs
        self._resident: dict[str, int] = {}
        self._finalizer = weakref.finalize(self, _destroy_device, self._lib, ptr)

    # -- ledger fields (mapped memory) ------------------------------------
    # Host-side writes bump the ledger's grow epoch so the FIFO re-drive
    # re-scores this device (see gs_ledger.grow_epoch in include/gs.h).

    def _field(name):  # noqa: N805
        def get(self):
            return getattr(self._led, name)

        def set_(self, v):
            setattr(self._led, name, int(v))
            self._led.grow_epoch += 1

        return property(get, set_)

    free_mem = _field("free_mem")
    in_use_warps = _field("in_use_warps")
    rr_cursor = _field("rr_cursor")
    version = _field("version")
    del _field

    def _arr_prop(name):  # noqa: N805
        def get(self):
            return getattr(self, name)

        def set_(self, values):
            getattr(self, name)[:] = values

        return property(get, set_)

    sm_warps = _arr_prop("_sm_warps")
    sm_tbs = _arr_prop("_sm_tbs")
    sm_regs = _arr_prop("_sm_regs")
    sm_smem = _arr_prop("_sm_smem")
    del _arr_prop

    @property
    def resident(self) -> _ResidentView:
        return _ResidentView(self)

    def __repr__(self) -> str:
        return (f"DeviceState(spec={self.spec!r}, index={self.index}, free_mem={self.free_mem}, "
                f"in_use_warps={self.in_use_warps}, rr_cursor={self.rr_cursor}, "
                f"version={self.version})")

    # -- residency bookkeeping (handle refcounts) ---------------------------

    def _mark_resident(self, uid: str, h: int) -> None:
        if uid not in self._resident:
            self._resident[uid] = h
            self._handles.incref(uid)

    # -- placement ------------------------------------------------------------

    def try_place_blocks(self, res) -> PlacementPlan | None:
        """device_model.py:120-139 (closed-form on the GPU); pure."""
        probe = pack_probe(res)
        n = int(self.spec.sm_count)
        blocks = np.zeros(n, dtype=np.int32)
        cursor = ctypes.c_int32()
        version = ctypes.c_int64()
        rc = nat.check(self._lib.gs_try_place(self._ptr, ctypes.byref(probe), blocks.ctypes.data,
                                              ctypes.byref(cursor), ctypes.byref(version)))
        if rc == nat.GS_INFEASIBLE:
            return None
        return PlacementPlan(tuple(int(b) for b in blocks), cursor.value, version.value)

    def commit_placement(self, plan: PlacementPlan, task_uid: str, res) -> None:
        """device_model.py:141-161."""
        probe = pack_probe(res)
        h = self._handles.get(task_uid)
        blocks = np.asarray(plan.blocks_per_sm, dtype=np.int32)
        if blocks.shape != (self.spec.sm_count,):
            self._handles.settle(task_uid)
            raise ContractViolation("placement plan does not match this device's SM count")
        rc = self._lib.gs_commit(self._ptr, h, ctypes.byref(probe), blocks.ctypes.data,
                                 int(plan.final_cursor), int(plan.version))
        if rc == nat.GS_ERR_CONTRACT:
            self._handles.settle(task_uid)
            raise ContractViolation(nat.last_error())
        nat.check(rc)
        self._mark_resident(task_uid, h)

    def empty_capacity_blocks(self, res) -> int:
        """device_model.py:163-165."""
        return occupancy_limit_per_sm(self.spec, res) * self.spec.sm_count

    # -- memory and warp accounting -------------------------------------------

    def reserve_memory(self, nbytes: int) -> bool:
        return nat.check(self._lib.gs_reserve_memory(self._ptr, _i64("nbytes", nbytes))) == nat.GS_OK

    def assign_memory(self, task_uid: str, nbytes: int) -> None:
        h = self._handles.get(task_uid)
        nat.check(self._lib.gs_assign_memory(self._ptr, h, _i64("nbytes", nbytes)))
        self._mark_resident(task_uid, h)

    def add_warps(self, task_uid: str, warps: int) -> None:
        h = self._handles.get(task_uid)
        nat.check(self._lib.gs_add_warps(self._ptr, h, _i64("warps", warps)))
        self._mark_resident(task_uid, h)

    def allocate_raw(self, task_uid: str, nbytes: int) -> bool:
        """Memory-only grab used by the job-granular policies (:185-190)."""
        h = self._handles.get(task_uid)
        rc = nat.check(self._lib.gs_allocate_raw(self._ptr, h, _i64("nbytes", nbytes)))
        if rc == nat.GS_OK:
            self._mark_resident(task_uid, h)
            return True
        self._handles.settle(task_uid)
        return False

    def release_task(self, task_uid: str) -> int:
        """Return every resource held under task_uid (:192-209)."""
        h = self._resident.get(task_uid)
        if h is None:
            raise ContractViolation(f"release of unknown task {task_uid!r} on device {self.index}")
        freed = ctypes.c_int64()
        rc = self._lib.gs_release(self._ptr, h, ctypes.byref(freed))
        if rc == nat.GS_ERR_CONTRACT:
            raise ContractViolation(f"release of unknown task {task_uid!r} on device {self.index}")
        nat.check(rc)
        del self._resident[task_uid]
        self._handles.decref(task_uid)
        return freed.value

    # -- invariants -------------------------------------------------------------

    def check_conservation(self) -> None:
        """device_model.py:220-245 (audited on the GPU)."""
        kind, sm = ctypes.c_int32(), ctypes.c_int32()
        held, warps = ctypes.c_int64(), ctypes.c_int64()
        rc = self._lib.gs_check_conservation(self._ptr, ctypes.byref(kind), ctypes.byref(sm),
                                             ctypes.byref(held), ctypes.byref(warps))
        if rc == nat.GS_OK:
            return
        if rc != nat.GS_ERR_CONTRACT:
            nat.check(rc)
        k, s, i = kind.value, sm.value, self.index
        if k == 1:
            raise ContractViolation(f"device {i}: free {self.free_mem} + held {held.value} "
                                    f"!= capacity {self.spec.mem_bytes}")
        if k == 2:
            raise ContractViolation(f"device {i}: warp ledger {self.in_use_warps} "
                                    f"!= sum of residents {warps.value}")
        what = {3: (self.sm_tbs, "blocks"), 4: (self.sm_warps, "warps"),
                5: (self.sm_regs, "regs"), 6: (self.sm_smem, "smem")}[k]
        raise ContractViolation(f"device {i} sm {s}: {int(what[0][s])} {what[1]}")
