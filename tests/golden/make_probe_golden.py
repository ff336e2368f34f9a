"""Record the reference probe producer's outputs (compute_resource_request).

Run in the build container (the reference is importable only here):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_probe_golden.py

For every program below it runs the UNMODIFIED reference pipeline
`analyze_program(parse_program(text))` (gpushare/task_builder.py:370-411)
and writes, per task, the inputs compute_resource_request
(gpushare/task_builder.py:258-290) aggregated and the ResourceRequest it
returned:

    allocs    [[alloc op id, bytes], ...]  every bound malloc of the task
    heap      bytes of the first unit's dominating set_heap_limit, or null
    launches  [[thread_blocks, threads_per_block, regs, smem, dur_ms], ...]
              in unit (program) order
    resources the nine ResourceRequest fields

Programs: every template of the reference's std and neural catalogs
(workload_gen.template_trace), the resource cases of the reference's own
tests/test_task_builder.py (RES_EXAMPLE, default heap), a symbol malloc'ed
twice, and 200 random programs from the reference's randprog fixture
generator.  tests/test_probe_golden.py checks gpushare.compute_resource_request
and libgs's gs_request_from_launches against this file.
"""

from __future__ import annotations

import json
import os
import random
import sys

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, os.path.join(REF, "..", "tests"))

from gpushare.errors import AnalysisError  # noqa: E402
from gpushare.task_builder import analyze_program  # noqa: E402
from gpushare.trace_model import parse_program  # noqa: E402
from gpushare.workload_gen import builtin_catalog, template_trace  # noqa: E402

import randprog as rp  # noqa: E402  (reference test fixtures)
import test_task_builder as ttb  # noqa: E402

EXTRA = {
    "res_example": ttb.RES_EXAMPLE,
    "default_heap": ("program t\nfunc t\nblock e\n  malloc a 100\n"
                     "  launch k grid 1 1 1 block 32 1 1 args a dur 1\nend\n"),
    # the same symbol allocated twice: two alloc ops, both counted
    "malloc_twice": ("program t\nfunc t\nblock e\n  malloc a 100\n  malloc a 300\n  malloc b 7\n"
                     "  launch k grid 4 1 1 block 64 1 1 args a,b dur 2 regs 32\n"
                     "  launch k2 grid 2 1 1 block 128 1 1 args a dur 1 smem 4096\nend\n"),
}


def record(text: str) -> list[dict]:
    ana = analyze_program(parse_program(text))
    by_id = {op.op_id: op for blk in ana.fn.blocks.values() for op in blk.ops}
    out = []
    for t in ana.tasks:
        allocs = sorted({a for u in t.units for a in u.alloc_ops})
        first = min(t.units, key=lambda u: u.order)
        heap = by_id[next(iter(first.heap_ops))].bytes if first.heap_ops else None
        launches = [[by_id[u.launch_op].thread_blocks, by_id[u.launch_op].threads_per_block,
                     by_id[u.launch_op].regs_per_thread, by_id[u.launch_op].smem_per_block,
                     by_id[u.launch_op].base_duration_ms] for u in t.units]
        r = t.resources
        out.append({"allocs": [[a, by_id[a].bytes] for a in allocs], "heap": heap, "launches": launches,
                    "lazy": t.lazy,
                    "resources": [r.mem_bytes, r.heap_limit_bytes, r.thread_blocks, r.warps_per_block,
                                  r.total_warps, r.threads_per_block, r.regs_per_thread, r.smem_per_block,
                                  r.est_duration_ms]})
    return out


def main() -> None:
    progs: dict[str, str] = dict(EXTRA)
    for cat in ("std", "neural"):
        c = builtin_catalog(cat)
        for t in c["templates"]:
            progs[f"{cat}:{t['name']}"] = template_trace(t)
    rng = random.Random(20260417)
    n_rand = 0
    while n_rand < 200:
        text = rp.gen_program(rng)
        try:
            rec = record(text)
        except AnalysisError:
            continue
        progs[f"rand{n_rand:03d}"] = text
        n_rand += 1
    out = {}
    for name, text in progs.items():
        out[name] = {"tasks": record(text)}
    path = os.path.join(HERE, "probe_requests.json")
    with open(path, "w") as f:
        json.dump(out, f, sort_keys=True, separators=(",", ":"))
    n_tasks = sum(len(v["tasks"]) for v in out.values())
    print(f"wrote {path}: {len(out)} programs, {n_tasks} tasks")


if __name__ == "__main__":
    main()
