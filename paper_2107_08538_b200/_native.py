"""ctypes binding of libgs (include/gs.h).

This module is the whole Python<->native boundary of the placement engine.
It loads the in-tree ``libgs.so`` (built by ``paper_2107_08538_b200.build``)
and fails loudly when the library or a CUDA device is missing: the product
path has no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
import threading
from ctypes import POINTER, c_double, c_float, c_int32, c_int64, c_void_p

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgs.so")

GS_OK = 0
GS_INFEASIBLE = 1
GS_REJECT = 2
GS_ERR_CONFIG = -2
GS_ERR_CONTRACT = -3
GS_ERR_CUDA = -4
GS_ERR_NOMEM = -5

GS_ASSIGN, GS_DEFER, GS_REJECTED, GS_NOT_TRIED = 0, 1, 2, 3
POLICY_CODES = {"sa": 0, "cg": 1, "mgb-sm": 2, "mgb-warps": 3}


class GsSpec(ctypes.Structure):
    _fields_ = [(n, c_int64) for n in (
        "sm_count", "mem_bytes", "max_warps_per_sm", "max_tbs_per_sm",
        "regs_per_sm", "smem_per_sm_bytes")]


class GsProbe(ctypes.Structure):
    _fields_ = [
        ("mem_bytes", c_int64), ("heap_limit_bytes", c_int64),
        ("total_warps", c_int64), ("est_duration_ms", c_double),
        ("thread_blocks", c_int32), ("warps_per_block", c_int32),
        ("threads_per_block", c_int32), ("regs_per_thread", c_int32),
        ("smem_per_block", c_int32), ("handle", c_int32), ("job", c_int32),
        ("level", c_int32)]


PROBE_DTYPE = np.dtype([
    ("mem_bytes", "<i8"), ("heap_limit_bytes", "<i8"), ("total_warps", "<i8"),
    ("est_duration_ms", "<f8"), ("thread_blocks", "<i4"),
    ("warps_per_block", "<i4"), ("threads_per_block", "<i4"),
    ("regs_per_thread", "<i4"), ("smem_per_block", "<i4"), ("handle", "<i4"),
    ("job", "<i4"), ("level", "<i4")])
assert PROBE_DTYPE.itemsize == ctypes.sizeof(GsProbe) == 64


class GsLedger(ctypes.Structure):
    _fields_ = [("free_mem", c_int64), ("in_use_warps", c_int64),
                ("version", c_int64), ("held_mem", c_int64),
                ("held_warps", c_int64), ("grow_epoch", c_int64),
                ("reserved", c_int64), ("rr_cursor", c_int32),
                ("sm_count", c_int32)]


class GsDecision(ctypes.Structure):
    _fields_ = [("outcome", c_int32), ("device", c_int32),
                ("free_mem_after", c_int64), ("in_use_warps_after", c_int64),
                ("pending_index", c_int32), ("handle", c_int32)]


DECISION_DTYPE = np.dtype([
    ("outcome", "<i4"), ("device", "<i4"), ("free_mem_after", "<i8"),
    ("in_use_warps_after", "<i8"), ("pending_index", "<i4"), ("handle", "<i4")])
assert DECISION_DTYPE.itemsize == ctypes.sizeof(GsDecision) == 32


class GsResidency(ctypes.Structure):
    _fields_ = [("mem_bytes", c_int64), ("warps", c_int64),
                ("regs_per_block", c_int64), ("smem_per_block", c_int64),
                ("present", c_int32), ("has_blocks", c_int32),
                ("warps_per_block", c_int32), ("pad", c_int32)]


# name -> (restype, argtypes); the complete export list of include/gs.h
SIGNATURES = {
    "gs_abi_version": (c_int32, []),
    "gs_last_error": (ctypes.c_char_p, []),
    "gs_engine_open": (c_int32, [c_int32, POINTER(c_void_p)]),
    "gs_engine_close": (None, [c_void_p]),
    "gs_engine_reserve_handles": (c_int32, [c_void_p, c_int32]),
    "gs_engine_handle_capacity": (c_int32, [c_void_p]),
    "gs_engine_launches": (c_int64, [c_void_p]),
    "gs_device_create": (c_int32, [c_void_p, POINTER(GsSpec), c_int32, POINTER(c_void_p)]),
    "gs_device_destroy": (None, [c_void_p]),
    "gs_device_ledger": (c_void_p, [c_void_p]),
    "gs_device_sm_array": (c_void_p, [c_void_p, c_int32]),
    "gs_try_place": (c_int32, [c_void_p, POINTER(GsProbe), c_void_p, POINTER(c_int32), POINTER(c_int64)]),
    "gs_commit": (c_int32, [c_void_p, c_int32, POINTER(GsProbe), c_void_p, c_int32, c_int64]),
    "gs_reserve_memory": (c_int32, [c_void_p, c_int64]),
    "gs_assign_memory": (c_int32, [c_void_p, c_int32, c_int64]),
    "gs_add_warps": (c_int32, [c_void_p, c_int32, c_int64]),
    "gs_allocate_raw": (c_int32, [c_void_p, c_int32, c_int64]),
    "gs_release": (c_int32, [c_void_p, c_int32, POINTER(c_int64)]),
    "gs_check_conservation": (c_int32, [c_void_p, POINTER(c_int32), POINTER(c_int32),
                                        POINTER(c_int64), POINTER(c_int64)]),
    "gs_residency_read": (c_int32, [c_void_p, c_int32, POINTER(GsResidency), c_void_p]),
    "gs_sched_create": (c_int32, [c_void_p, POINTER(c_void_p), c_int32, c_int32, c_int32,
                                  c_int32, POINTER(c_void_p)]),
    "gs_sched_destroy": (None, [c_void_p]),
    "gs_submit": (c_int32, [c_void_p, POINTER(GsProbe), POINTER(GsDecision)]),
    "gs_submit_batch": (c_int32, [c_void_p, c_void_p, c_int32, c_void_p]),
    "gs_on_release": (c_int32, [c_void_p, c_void_p, c_int32, POINTER(c_int32), POINTER(c_int32)]),
    "gs_release_redrive": (c_int32, [c_void_p, c_int32, c_int32, POINTER(c_int64), c_void_p, c_int32,
                                     POINTER(c_int32), POINTER(c_int32)]),
    "gs_job_ended": (c_int32, [c_void_p, c_int32]),
    "gs_pending_count": (c_int32, [c_void_p]),
    "gs_sched_job_state": (c_int32, [c_void_p, c_void_p, c_void_p, POINTER(c_int32)]),
    "gs_sweep": (c_int32, [c_void_p, c_void_p, c_int32, c_int32, c_void_p, c_int64,
                           POINTER(c_int64), POINTER(c_float)]),
    "gs_sched_ring_start": (c_int32, [c_void_p, c_int32, c_int32, c_int32]),
    "gs_sched_ring_stop": (c_int32, [c_void_p]),
    "gs_engine_decisions": (c_int64, [c_void_p]),
}

_lib = None
_lib_lock = threading.Lock()


def lib() -> ctypes.CDLL:
    """Load libgs.so (in-tree build).  Raises when it is absent."""
    global _lib
    with _lib_lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                    "(there is no CPU fallback for the placement engine)")
            handle = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def last_error() -> str:
    msg = lib().gs_last_error()
    return msg.decode() if msg else ""


class NativeError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"libgs error {code}: {msg}")
        self.code = code


def check(rc: int) -> int:
    if rc < 0:
        raise NativeError(rc, last_error())
    return rc


class Engine:
    """One engine per process: the decision stream's single authority."""

    def __init__(self, cuda_device: int = 0):
        self.lib = lib()
        ptr = c_void_p()
        rc = self.lib.gs_engine_open(cuda_device, ctypes.byref(ptr))
        if rc < 0:
            raise RuntimeError(
                f"libgs engine unavailable on cuda:{cuda_device}: {last_error()} "
                "(placement runs on the GPU only)")
        self.ptr = ptr
        self.cuda_device = cuda_device
        self.lock = threading.RLock()
        self._cap = self.lib.gs_engine_handle_capacity(ptr)

    def reserve_handles(self, n: int) -> None:
        if n > self._cap:
            check(self.lib.gs_engine_reserve_handles(self.ptr, n))
            self._cap = self.lib.gs_engine_handle_capacity(self.ptr)

    @property
    def launches(self) -> int:
        return int(self.lib.gs_engine_launches(self.ptr))


_engine: Engine | None = None


def engine() -> Engine:
    global _engine
    if _engine is None:
        _engine = Engine(int(os.environ.get("GS_CUDA_DEVICE", "0")))
    return _engine
