"""ctypes wrapper of oracle/libkernels_cpu.so — test infrastructure only.

CPU restatements of the workload kernels, used as the parity checker for
the GPU kernels and as the timed CPU baseline (bench.py --impl reference).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from ctypes import POINTER, c_float, c_int32, c_int64, c_uint64, c_void_p

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libkernels_cpu.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            subprocess.run(["make", "-s", "-C", HERE, "libkernels_cpu.so"], check=True)
        L = ctypes.CDLL(LIB)
        sig = {
            "cpu_bfs": (c_int32, [c_int64, c_uint64, c_void_p]),
            "cpu_hotspot": (None, [c_int64, c_int32, c_uint64, c_void_p]),
            "cpu_srad": (None, [c_int64, c_int32, c_uint64, c_void_p]),
            "cpu_kmeans": (None, [c_int64, c_int32, c_int32, c_uint64, c_void_p, c_void_p]),
            "cpu_backprop": (None, [c_int64, c_int32, c_int32, c_uint64, c_void_p, c_void_p, c_void_p,
                                    POINTER(c_float)]),
            "cpu_needle": (None, [c_int64, c_uint64, c_void_p]),
            "cpu_lud": (None, [c_int64, c_uint64, c_void_p]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def bfs(n, seed):
    out = np.zeros(n, np.int32)
    depth = lib().cpu_bfs(n, seed, out.ctypes.data)
    return out, depth


def hotspot(n, iters, seed):
    out = np.zeros((n, n), np.float32)
    lib().cpu_hotspot(n, iters, seed, out.ctypes.data)
    return out


def srad(n, iters, seed):
    out = np.zeros((n, n), np.float32)
    lib().cpu_srad(n, iters, seed, out.ctypes.data)
    return out


def kmeans(n, nf, iters, seed):
    mem = np.zeros(n, np.int32)
    cent = np.zeros((5, nf), np.float32)
    lib().cpu_kmeans(n, nf, iters, seed, mem.ctypes.data, cent.ctypes.data)
    return mem, cent


def backprop(n_in, n_hid, iters, seed):
    w1 = np.zeros((n_in + 1, n_hid), np.float32)  # [input][hidden]
    w2 = np.zeros(n_hid + 1, np.float32)
    hid = np.zeros(n_hid + 1, np.float32)
    o = c_float()
    lib().cpu_backprop(n_in, n_hid, iters, seed, w1.ctypes.data, w2.ctypes.data, hid.ctypes.data,
                       ctypes.byref(o))
    return w1, w2, hid, o.value


def needle(n, seed):
    out = np.zeros((n + 1, n + 1), np.int32)
    lib().cpu_needle(n, seed, out.ctypes.data)
    return out


def lud(n, seed):
    out = np.zeros((n, n), np.float32)
    lib().cpu_lud(n, seed, out.ctypes.data)
    return out


def run(kind, n, iters=1, m=0, seed=1):
    """Primary output of a job, shaped like workloads.run_solo's."""
    if kind == "bfs":
        return bfs(n, seed)[0]
    if kind == "hotspot":
        return hotspot(n, iters, seed)
    if kind == "srad":
        return srad(n, iters, seed)
    if kind == "kmeans":
        return kmeans(n, m, iters, seed)[0]
    if kind == "backprop":
        return backprop(n, m, iters, seed)[0]
    if kind == "needle":
        return needle(n, seed)
    if kind == "lud":
        return lud(n, seed)
    raise ValueError(kind)


_C = 0x9E3779B1
_M64 = (1 << 64) - 1


def digest(kind, out):
    """The executor's order-independent output digest (gs_kernels.cuh
    checksum_words: C * sum of the 32-bit words + n(n-1)/2 mod 2^64) of an
    oracle output, laid out like the job's device buffer (needle: pitch
    n + 4 with three leading zero columns, which add no word value)."""
    a = np.ascontiguousarray(out)
    words = a.view(np.uint32).ravel()
    s = int(words.sum(dtype=np.uint64))
    nwords = words.size
    if kind == "needle":
        n1 = a.shape[0]
        nwords = n1 * (n1 + 3)
    return (_C * s + nwords * (nwords - 1) // 2) & _M64
