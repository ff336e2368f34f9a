"""Probe producer pinned to the reference.

tests/golden/probe_requests.json holds, for 225 programs (both reference
catalogs, the reference's own resource test cases, a symbol malloc'ed twice,
200 random programs from the reference's randprog generator), every task's
allocation records, heap limit and launch shapes together with the
ResourceRequest the UNMODIFIED reference compute_resource_request
(gs/task_builder.py:258-290) returned for them (make_probe_golden.py).

Both producers here must reproduce every request exactly:
* gpushare.compute_resource_request (host Python drop-in);
* libgs gs_request_from_launches (the C-ABI probe capture the executor
  uses for real CUDA launches) — pure host arithmetic, runs on CPU.
"""

import json
import os
import sys

import pytest

from paper_2107_08538_b200 import workloads as W
from paper_2107_08538_b200.gpushare.task_builder import LaunchShape, compute_resource_request

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "probe_requests.json")))
CASES = [(name, i, t) for name, prog in sorted(GOLDEN.items()) for i, t in enumerate(prog["tasks"])]
HEAP_DEFAULT = 8 << 20


def test_fixture_covers_the_reference_cases():
    assert len(GOLDEN) == 225 and len(CASES) >= 225
    assert any(n.startswith("std:") for n in GOLDEN) and any(n.startswith("neural:") for n in GOLDEN)
    # tests/test_task_builder.py:149-162 of the reference
    assert GOLDEN["res_example"]["tasks"][0]["resources"] == [1000 + 24 + 4096, 4096, 2, 8, 16, 256, 10, 128, 7.5]
    # a symbol malloc'ed twice counts twice (distinct alloc ops)
    assert GOLDEN["malloc_twice"]["tasks"][0]["resources"][0] == 100 + 300 + 7 + HEAP_DEFAULT


@pytest.mark.parametrize("name,i,task", CASES, ids=[f"{c[0]}#{c[1]}" for c in CASES])
def test_python_request_matches_reference(name, i, task):
    shapes = [LaunchShape("k", *l) for l in task["launches"]]
    r = compute_resource_request([tuple(a) for a in task["allocs"]], shapes, task["heap"])
    got = [r.mem_bytes, r.heap_limit_bytes, r.thread_blocks, r.warps_per_block, r.total_warps,
           r.threads_per_block, r.regs_per_thread, r.smem_per_block, r.est_duration_ms]
    assert got == task["resources"]


@pytest.mark.parametrize("name,i,task", CASES, ids=[f"{c[0]}#{c[1]}" for c in CASES])
def test_c_abi_request_matches_reference(name, i, task):
    heap = HEAP_DEFAULT if task["heap"] is None else task["heap"]
    p = W.request_from_launches([tuple(l) for l in task["launches"]], [a[1] for a in task["allocs"]], heap)
    got = [p.mem_bytes, p.heap_limit_bytes, p.thread_blocks, p.warps_per_block, p.total_warps,
           p.threads_per_block, p.regs_per_thread, p.smem_per_block]
    assert got == task["resources"][:8]
    assert p.est_duration_ms == pytest.approx(task["resources"][8], rel=1e-12)


REF = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present (GPU box)")
def test_reference_signature_against_live_reference():
    """compute_resource_request(units, fn) — the reference's own call form —
    on the reference's analysis objects equals the reference's result."""
    sys.path.insert(0, REF)
    try:
        from gpushare.task_builder import analyze_program
        from gpushare.trace_model import parse_program
        from gpushare.workload_gen import builtin_catalog, template_trace
    finally:
        sys.path.remove(REF)
    n = 0
    for cat in ("std", "neural"):
        for t in builtin_catalog(cat)["templates"]:
            ana = analyze_program(parse_program(template_trace(t)))
            for task in ana.tasks:
                r = compute_resource_request(task.units, ana.fn)
                assert tuple(vars(r).values()) == tuple(vars(task.resources).values())
                n += 1
    assert n >= 17
