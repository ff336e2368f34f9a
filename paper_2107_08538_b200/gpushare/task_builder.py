"""Probe payload: ResourceRequest and its aggregation arithmetic.

Mirrors the hot-path part of gpushare/task_builder.py: the ResourceRequest
record (:45-55) and compute_resource_request (:258-290).  The trace-language
front end (CFG, dominators, task merging, :115-411) is out of scope (host
compile-time analysis); here a task is described
directly by its buffers and its kernel launch shapes, which is what the
executor's probe capture records for real CUDA launches.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Mapping

from .errors import AnalysisError

DEFAULT_HEAP_LIMIT = 8 * 2**20  # cudaLimitMallocHeapSize default (task_builder.py:29)
BYTE_LIMIT = 2**63  # task_builder.py:30
WARP_SIZE = 32


@dataclass(frozen=True)
class ResourceRequest:
    """The probe record (task_builder.py:45-55); 64 B packed in the ring."""

    mem_bytes: int
    heap_limit_bytes: int
    thread_blocks: int
    warps_per_block: int
    total_warps: int
    threads_per_block: int
    regs_per_thread: int
    smem_per_block: int
    est_duration_ms: float


@dataclass(frozen=True)
class LaunchShape:
    """One kernel launch of a task: grid, block and per-thread/per-block
    resources as the occupancy API reports them (cudaFuncGetAttributes)."""

    kernel: str
    thread_blocks: int
    threads_per_block: int
    regs_per_thread: int = 0
    smem_per_block: int = 0
    base_duration_ms: float = 0.0


def warps_per_block(threads_per_block: int) -> int:
    return -(-threads_per_block // WARP_SIZE)


def compute_resource_request(allocs, launches, heap_limit_bytes: int | None = None) -> ResourceRequest:
    """Aggregate a task's footprint and widest launch (task_builder.py:258-290).

    Two call forms:

    * ``compute_resource_request(allocs, launches, heap_limit_bytes=None)``:
      `allocs` are the task's allocation RECORDS, one per malloc call — a
      ``{name: bytes}`` mapping or ``(key, bytes)`` pairs.  Every record
      counts, as every distinct alloc op does in the reference
      (task_builder.py:260-262): a symbol allocated twice is two records.
      `launches` are LaunchShape (or objects with the same fields) in
      program order.
    * ``compute_resource_request(units, fn)`` — the reference's own
      signature: `units` are the merged task's UnitTasks and `fn` the
      inlined FunctionGraph (duck-typed: ``alloc_ops`` / ``heap_ops`` /
      ``launch_op`` / ``order`` on the units, ``blocks[*].ops[*]`` with
      ``op_id`` / ``bytes`` and the launch fields on `fn`).

    Arithmetic: mem = Σ record bytes + the device heap limit (8 MiB default,
    counted once per task); the widest launch is the FIRST maximum of
    tbs·ceil(threads/32) and gives threads_per_block; regs and smem are
    maxima over all launches; the duration estimate is the sum.
    """
    if hasattr(launches, "blocks"):  # reference form (units, fn)
        units, fn = allocs, launches
        by_id = {op.op_id: op for blk in fn.blocks.values() for op in blk.ops}
        alloc_ids = sorted({a for u in units for a in u.alloc_ops})
        first = min(units, key=lambda u: u.order)
        heap = by_id[next(iter(first.heap_ops))].bytes if first.heap_ops else None
        records = [(a, by_id[a].bytes) for a in alloc_ids]
        shapes = [by_id[u.launch_op] for u in units]
        return compute_resource_request(records, shapes, heap)
    if not launches:
        raise AnalysisError("a task needs at least one launch")
    items = allocs.items() if isinstance(allocs, Mapping) else allocs
    heap = DEFAULT_HEAP_LIMIT if heap_limit_bytes is None else int(heap_limit_bytes)
    mem = sum(int(nbytes) for _, nbytes in items) + heap
    if mem >= BYTE_LIMIT:
        raise AnalysisError(f"task memory request {mem} bytes overflows the byte limit")
    widest = max(launches, key=lambda op: op.thread_blocks * warps_per_block(op.threads_per_block))
    tbs, wpb = widest.thread_blocks, warps_per_block(widest.threads_per_block)
    return ResourceRequest(
        mem_bytes=mem,
        heap_limit_bytes=heap,
        thread_blocks=tbs,
        warps_per_block=wpb,
        total_warps=tbs * wpb,
        threads_per_block=widest.threads_per_block,
        regs_per_thread=max(op.regs_per_thread for op in launches),
        smem_per_block=max(op.smem_per_block for op in launches),
        est_duration_ms=sum(op.base_duration_ms for op in launches),
    )
