"""Workload jobs and the executor (include/gs_work.h) from Python.

A job is the executable counterpart of a reference catalog template
(gpushare/data/catalog.json): Rodinia-class kernels (bfs, hotspot, srad,
kmeans, backprop, needle, lud) written for sm_100a in csrc/gs_kernels.cuh.
`run_jobs` is the wall-clock analogue of gpushare.metrics.run_workload ->
sim_engine.run_sim (metrics.py:101-119): same policies (sa, cg:<r>,
mgb-sm, mgb-warps), same worker-pool semantics, real B200 execution.
"""

from __future__ import annotations

import ctypes
from ctypes import POINTER, c_double, c_float, c_int32, c_int64, c_uint64, c_void_p
from dataclasses import dataclass

import numpy as np

from . import _native as nat

KINDS = {"bfs": 0, "hotspot": 1, "srad": 2, "kmeans": 3, "backprop": 4, "needle": 5, "lud": 6, "yolo": 7, "resnet": 8}
KIND_NAMES = {v: k for k, v in KINDS.items()}
MODE_DEVICE, MODE_E2E = 0, 1


class GsJobDesc(ctypes.Structure):
    _fields_ = [("kind", c_int32), ("iters", c_int32), ("n", c_int64), ("m", c_int64), ("seed", c_uint64)]


class GsJobRecord(ctypes.Structure):
    _fields_ = [("state", c_int32), ("device", c_int32), ("arrival_ms", c_double), ("pull_ms", c_double),
                ("admit_ms", c_double),
                ("end_ms", c_double), ("wait_ms", c_double), ("compute_ms", c_double),
                ("mem_bytes", c_int64), ("h2d_bytes", c_int64), ("d2h_bytes", c_int64),
                ("checksum", c_uint64), ("n_kernels", c_int32), ("sm_share", c_int32),
                ("setup_ms", c_double), ("gen_ms", c_double), ("tail_ms", c_double)]


class GsExecStats(ctypes.Structure):
    _fields_ = [("makespan_ms", c_double), ("completed", c_int32), ("crashed", c_int32), ("oom", c_int32),
                ("rejected", c_int32), ("kernel_launches", c_int64), ("decision_launches", c_int64),
                ("decision_ms", c_double)]


class GsExecEvent(ctypes.Structure):
    """One entry of the executor's placement log (gs_work.h gs_exec_event)."""

    _fields_ = [("kind", c_int32), ("handle", c_int32), ("device", c_int32), ("outcome", c_int32),
                ("freed", c_int64), ("free_mem_after", c_int64), ("in_use_warps_after", c_int64),
                ("t_ms", c_double), ("probe", nat.GsProbe)]


EV_SUBMIT, EV_RELEASE, EV_JOB_ENDED, EV_DRAIN = 0, 1, 2, 3


class GsLaunchDesc(ctypes.Structure):
    _fields_ = [("thread_blocks", c_int32), ("threads_per_block", c_int32), ("regs_per_thread", c_int32),
                ("smem_per_block", c_int32), ("est_duration_ms", c_double)]


WORK_SIGNATURES = {
    "gs_job_probe": (c_int32, [POINTER(GsJobDesc), POINTER(nat.GsProbe)]),
    "gs_request_from_launches": (c_int32, [POINTER(GsLaunchDesc), c_int32, POINTER(c_int64), c_int32, c_int64,
                                           POINTER(nat.GsProbe)]),
    "gs_launch_desc_of": (c_int32, [c_void_p, c_int32, c_int32, c_int32, POINTER(GsLaunchDesc)]),
    "gs_job_io_bytes": (c_int32, [POINTER(GsJobDesc), POINTER(c_int64), POINTER(c_int64)]),
    "gs_job_run_solo": (c_int32, [POINTER(GsJobDesc), c_int32, c_int32, c_void_p, c_int64,
                                  POINTER(GsJobRecord)]),
    "gs_exec_run": (c_int32, [c_void_p, c_int32, c_int32, c_int32, POINTER(c_int32), c_int32, c_int32,
                              c_int32, c_int64, c_void_p, POINTER(GsExecStats)]),
    "gs_exec_run_arrivals": (c_int32, [c_void_p, c_int32, c_void_p, c_int32, c_int32, POINTER(c_int32), c_int32,
                                       c_int32, c_int32, c_int64, c_void_p, POINTER(GsExecStats)]),
    "gs_exec_stage": (c_int32, [c_void_p, c_int32, POINTER(c_int32), c_int32, c_int32]),
    "gs_exec_ledger_capacity": (c_int32, [c_int32, POINTER(c_int64)]),
    "gs_exec_unstage": (None, []),
    "gs_measure_fp32_peak": (c_int32, [c_int32, POINTER(c_double)]),
    "gs_selftest_division": (c_int32, [c_int32, c_int64, c_uint64, c_float, POINTER(c_int64)]),
    "gs_exec_set_sm_parts": (c_int32, [c_int32]),
    "gs_capture_begin": (c_int32, [c_int32, POINTER(c_void_p)]),
    "gs_capture_malloc": (c_int32, [c_void_p, c_int64, POINTER(c_void_p)]),
    "gs_capture_free": (c_int32, [c_void_p, c_void_p]),
    "gs_capture_end": (c_int32, [c_void_p, c_int64, POINTER(c_void_p)]),
    "gs_task_graph_probe": (c_int32, [c_void_p, POINTER(nat.GsProbe), POINTER(c_int32), POINTER(c_int32)]),
    "gs_task_graph_run": (c_int32, [c_void_p, c_void_p, POINTER(c_uint64), POINTER(c_float)]),
    "gs_task_graph_device": (c_int32, [c_void_p]),
    "gs_task_graph_destroy": (None, [c_void_p]),
    "gs_job_capture": (c_int32, [POINTER(GsJobDesc), c_int32, POINTER(c_void_p)]),
    "gs_exec_set_capture": (c_int32, [c_int32]),
    "gs_exec_drop_graphs": (None, []),
    "gs_exec_release_memory": (None, []),
    "gs_exec_sm_parts_layout": (c_int32, [c_int32, c_int32, POINTER(c_int32), c_int32, POINTER(c_int32)]),
    "gs_exec_log": (c_int32, [c_void_p, c_int64, POINTER(c_int64), c_void_p, c_int32, POINTER(c_int32),
                              POINTER(c_int32), POINTER(c_int32)]),
    "gs_gemm_bf16": (c_int32, [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_void_p, c_int64, c_int32,
                               c_int32, c_int32, c_int32, c_int32, c_void_p]),
}

_bound = False


def lib():
    global _bound
    L = nat.lib()
    if not _bound:
        for name, (res, args) in WORK_SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _bound = True
    return L


@dataclass(frozen=True)
class Job:
    """One job: kind, problem size n (nodes / grid edge / points / inputs /
    sequence length / matrix edge), secondary size m (kmeans features,
    backprop hidden units), iterations and seed."""

    kind: str
    n: int
    iters: int = 1
    m: int = 0
    seed: int = 1

    def desc(self) -> GsJobDesc:
        return GsJobDesc(KINDS[self.kind], int(self.iters), int(self.n), int(self.m), int(self.seed))


def probe(job: Job) -> nat.GsProbe:
    """The job's probe: footprint + widest launch (gs_job_probe)."""
    out = nat.GsProbe()
    nat.check(lib().gs_job_probe(ctypes.byref(job.desc()), ctypes.byref(out)))
    return out


def io_bytes(job: Job) -> tuple[int, int]:
    i, o = c_int64(), c_int64()
    nat.check(lib().gs_job_io_bytes(ctypes.byref(job.desc()), ctypes.byref(i), ctypes.byref(o)))
    return i.value, o.value


OUTPUT_DTYPES = {"bfs": np.int32, "hotspot": np.float32, "srad": np.float32, "kmeans": np.int32,
                 "backprop": np.float32, "needle": np.int32, "lud": np.float32, "yolo": np.float32,
                 "resnet": np.float32}


def output_shape(job: Job) -> tuple[int, ...]:
    n = job.n
    if job.kind == "yolo":  # both YOLO heads, NHWC, 255 channels each
        return ((job.m * (n // 32) ** 2 + job.m * (n // 16) ** 2) * 255,)
    if job.kind == "resnet":  # logits
        return (job.m, 1000)
    return {"bfs": (n,), "hotspot": (n, n), "srad": (n, n), "kmeans": (n,), "backprop": (n + 1, job.m),
            "needle": (n + 1, n + 4), "lud": (n, n)}.get(job.kind, (0,))


def run_solo(job: Job, device: int = 0) -> tuple[np.ndarray, GsJobRecord]:
    """Run one job alone on cuda:device; returns (primary output, record)."""
    out = np.zeros(output_shape(job), dtype=OUTPUT_DTYPES[job.kind])
    rec = GsJobRecord()
    nat.check(lib().gs_job_run_solo(ctypes.byref(job.desc()), device, MODE_DEVICE, out.ctypes.data,
                                    out.nbytes, ctypes.byref(rec)))
    if job.kind == "needle":  # aligned device layout: pitch n+4, column j at 3+j -> Rodinia (n+1) x (n+1)
        out = np.ascontiguousarray(out[:, 3:])
    return out, rec


def gemm_bf16(a, b, bias=None, out=None, act: int = 0, out_f32: bool = True):
    """D = act(a @ b.T + bias) on the tcgen05 GEMM (csrc/gs_gemm.cu).

    a [m, k] and b [n, k] are CUDA bf16 tensors (k % 8 == 0), bias fp32 [n];
    torch provides the device memory and the current stream only."""
    import torch

    m, k = a.shape
    n = b.shape[0]
    if out is None:
        out = torch.empty((m, n), dtype=torch.float32 if out_f32 else torch.bfloat16, device=a.device)
    stream = torch.cuda.current_stream(a.device).cuda_stream
    nat.check(lib().gs_gemm_bf16(a.data_ptr(), a.stride(0), b.data_ptr(), b.stride(0),
                                 bias.data_ptr() if bias is not None else None, out.data_ptr(), out.stride(0),
                                 m, n, k, 1 if out.dtype == torch.float32 else 0, act, stream))
    return out


def policy_code(policy: str) -> tuple[int, int]:
    from .gpushare.schedulers import parse_policy

    p = parse_policy(policy)
    return nat.POLICY_CODES[p.kind], p.cg_ratio


def stage(jobs: list[Job], devices: list[int], mode: int) -> None:
    arr = (GsJobDesc * len(jobs))(*[j.desc() for j in jobs])
    devs = (c_int32 * len(devices))(*devices)
    nat.check(lib().gs_exec_stage(arr, len(jobs), devs, len(devices), mode))


def unstage() -> None:
    lib().gs_exec_unstage()


@dataclass
class ExecResult:
    records: list[dict]
    makespan_ms: float
    completed: int
    crashed: int
    oom: int
    rejected: int
    kernel_launches: int
    decision_launches: int
    decision_ms: float


def request_from_launches(launches, buffers, heap_limit_bytes: int = 8 << 20):
    """Probe capture for any task: `launches` are
    (thread_blocks, threads_per_block, regs_per_thread, smem_per_block
    [, est_duration_ms]) as a launch wrapper records them, `buffers` the
    task's distinct allocation sizes; returns the 64 B gs_probe the
    placement engine takes (compute_resource_request's aggregation).  Host
    arithmetic in libgs; no GPU needed."""
    ls = (GsLaunchDesc * len(launches))(*[GsLaunchDesc(*l) for l in launches])
    bs = (c_int64 * max(len(buffers), 1))(*[int(b) for b in buffers])
    out = nat.GsProbe()
    nat.check(lib().gs_request_from_launches(ls, len(launches), bs, len(buffers), int(heap_limit_bytes),
                                             ctypes.byref(out)))
    return out


def fp32_peak_tflops(device: int = 0) -> float:
    """Measured FP32 FMA peak of the device (gs_measure_fp32_peak)."""
    t = c_double()
    nat.check(lib().gs_measure_fp32_peak(device, ctypes.byref(t)))
    return t.value


def selftest_division(n: int, seed: int = 1, q0sqr: float = 0.05, device: int = 0) -> dict:
    """srad's branch-free division against __fdiv_rn (gs_selftest_division)."""
    out = (c_int64 * 4)()
    nat.check(lib().gs_selftest_division(device, n, seed, q0sqr, out))
    return {"div_mismatches": out[0], "div_checked": out[1], "coeff_mismatches": out[2], "coeff_checked": out[3]}


def ledger_capacity(device: int = 0) -> int:
    """Bytes a run's ledger gets on `device` by default (free HBM + pool-held
    unused memory - 6 GiB); query once and pass as run_jobs(ledger_bytes=)
    when timing many runs."""
    cap = c_int64(0)
    nat.check(lib().gs_exec_ledger_capacity(device, ctypes.byref(cap)))
    return cap.value


@dataclass
class ExecLog:
    """The placement log of the last run: every decision-engine call in the
    single decision authority's order (gs_exec_log)."""

    events: list  # GsExecEvent
    specs: list   # GsSpec per ledger
    policy: int
    cg_ratio: int


def exec_log() -> ExecLog:
    L = lib()
    n = c_int64()
    nd, pol, ratio = c_int32(), c_int32(), c_int32()
    nat.check(L.gs_exec_log(None, 0, ctypes.byref(n), None, 0, ctypes.byref(nd), ctypes.byref(pol),
                            ctypes.byref(ratio)))
    evs = (GsExecEvent * max(n.value, 1))()
    specs = (nat.GsSpec * max(nd.value, 1))()
    nat.check(L.gs_exec_log(evs, n.value, ctypes.byref(n), specs, nd.value, ctypes.byref(nd), ctypes.byref(pol),
                            ctypes.byref(ratio)))
    return ExecLog(list(evs)[: n.value], list(specs)[: nd.value], pol.value, ratio.value)


class TaskGraph:
    """A task recorded by stream capture (csrc/gs_capture.cu): nothing ran
    and nothing was allocated; `probe` is computed from the recorded
    launches and allocations (kernel_launch_prepare), `run` replays the
    queue on the recording device (lazy_runtime.replay)."""

    def __init__(self, handle: int):
        self._h = c_void_p(handle)

    @property
    def device(self) -> int:
        return lib().gs_task_graph_device(self._h)

    def probe(self) -> tuple[nat.GsProbe, int, int]:
        """(probe, kernel launches recorded, allocations recorded)."""
        out, nk, na = nat.GsProbe(), c_int32(), c_int32()
        nat.check(lib().gs_task_graph_probe(self._h, ctypes.byref(out), ctypes.byref(nk), ctypes.byref(na)))
        return out, nk.value, na.value

    def run(self, stream: int = 0) -> tuple[int, float]:
        """Replay on `stream` of the recording device and wait: (output
        digest of a catalog job, device ms)."""
        cs, ms = c_uint64(), c_float()
        nat.check(lib().gs_task_graph_run(self._h, c_void_p(stream), ctypes.byref(cs), ctypes.byref(ms)))
        return cs.value, ms.value

    def close(self) -> None:
        if self._h:
            lib().gs_task_graph_destroy(self._h)
            self._h = c_void_p(0)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Capture:
    """Record arbitrary host code issued on `stream` into a TaskGraph:

        with W.Capture(device) as cap:
            a = cap.malloc(nbytes)        # an address, no memory yet
            launch_something(..., stream=cap.stream)
        graph = cap.graph                 # its probe, then replay
    """

    def __init__(self, device: int = 0, heap_limit_bytes: int = 0):
        self.device, self.heap = device, heap_limit_bytes
        self.stream = 0
        self.graph: TaskGraph | None = None

    def __enter__(self):
        s = c_void_p()
        nat.check(lib().gs_capture_begin(self.device, ctypes.byref(s)))
        self.stream = s.value
        return self

    def malloc(self, nbytes: int) -> int:
        p = c_void_p()
        nat.check(lib().gs_capture_malloc(c_void_p(self.stream), int(nbytes), ctypes.byref(p)))
        return p.value

    def free(self, ptr: int) -> None:
        nat.check(lib().gs_capture_free(c_void_p(self.stream), c_void_p(ptr)))

    def __exit__(self, *exc):
        g = c_void_p()
        rc = lib().gs_capture_end(c_void_p(self.stream), int(self.heap), ctypes.byref(g))
        if exc[0] is None:
            nat.check(rc)
            self.graph = TaskGraph(g.value)
        elif rc == 0:
            lib().gs_task_graph_destroy(g)
        return False


def capture_job(job: Job, device: int = 0) -> TaskGraph:
    """A staged catalog job's whole device-side life as a TaskGraph."""
    g = c_void_p()
    nat.check(lib().gs_job_capture(ctypes.byref(job.desc()), device, ctypes.byref(g)))
    return TaskGraph(g.value)


def set_capture(on: bool) -> None:
    """Executor capture mode: probes from recorded task graphs, jobs run by
    replaying them (gs_exec_set_capture)."""
    nat.check(lib().gs_exec_set_capture(1 if on else 0))


def release_memory() -> None:
    """Free the executor's idle job arenas (gs_exec_release_memory)."""
    lib().gs_exec_release_memory()


def set_sm_parts(parts: int) -> None:
    """Run later jobs on `parts` disjoint green-context SM partitions per
    device (<= 1: whole-device streams) — gs_exec_set_sm_parts."""
    nat.check(lib().gs_exec_set_sm_parts(int(parts)))


def sm_parts_layout(parts: int, device: int = 0) -> list[int]:
    """SM count of each of the `parts` partitions of `device`."""
    out = (c_int32 * 64)()
    n = c_int32()
    nat.check(lib().gs_exec_sm_parts_layout(device, parts, out, 64, ctypes.byref(n)))
    return list(out)[: n.value]


def run_jobs(jobs: list[Job], policy: str = "mgb-warps", devices: list[int] = (0,), workers: int = 8,
             mode: int = MODE_DEVICE, ledger_bytes: int = 0, arrivals_ms=None) -> ExecResult:
    """Run a job list under `policy` (wall clock; see module docstring).
    `arrivals_ms`: optional non-decreasing arrival time per job (ms)."""
    code, ratio = policy_code(policy)
    arr = (GsJobDesc * len(jobs))(*[j.desc() for j in jobs])
    recs = (GsJobRecord * len(jobs))()
    st = GsExecStats()
    devs = (c_int32 * len(devices))(*devices)
    arrv = None
    if arrivals_ms is not None:
        arrv = (c_double * len(jobs))(*[float(a) for a in arrivals_ms])
    nat.check(lib().gs_exec_run_arrivals(arr, len(jobs), arrv, code, ratio, devs, len(devices), workers, mode,
                                         int(ledger_bytes), recs, ctypes.byref(st)))
    rows = []
    for j, r in zip(jobs, recs):
        rows.append({"kind": j.kind, "n": j.n, "state": ("done", "oom", "rejected")[r.state],
                     "device": r.device, "arrival_ms": r.arrival_ms, "pull_ms": r.pull_ms,
                     "admit_ms": r.admit_ms, "end_ms": r.end_ms, "turnaround_ms": r.end_ms - r.arrival_ms,
                     "wait_ms": r.wait_ms, "compute_ms": r.compute_ms,
                     "mem_bytes": r.mem_bytes, "h2d_bytes": r.h2d_bytes, "d2h_bytes": r.d2h_bytes,
                     "checksum": r.checksum, "n_kernels": r.n_kernels, "sm_share": r.sm_share,
                     "setup_ms": r.setup_ms, "gen_ms": r.gen_ms, "tail_ms": r.tail_ms})
    return ExecResult(rows, st.makespan_ms, st.completed, st.crashed, st.oom, st.rejected,
                      st.kernel_launches, st.decision_launches, st.decision_ms)
