"""The ctypes mirrors in workloads.py follow the C structs of
include/gs_work.h field by field (name order and type width), so a field
added on one side cannot silently shift the other (CPU only)."""

import ctypes
import os
import re

from paper_2107_08538_b200 import workloads as W

HDR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "gs_work.h")
WIDTH = {"int32_t": 4, "int64_t": 8, "uint64_t": 8, "double": 8}


def c_fields(struct: str) -> list[tuple[str, int]]:
    src = open(HDR).read()
    body = re.search(r"typedef struct %s \{(.*?)\} %s;" % (struct, struct), src, re.S).group(1)
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    out = []
    for decl in body.split(";"):
        m = re.match(r"\s*(\w+)\s+(.*)", decl.strip())
        if not m:
            continue
        for name in m.group(2).split(","):
            out.append((name.strip(), WIDTH[m.group(1)]))
    return out


def py_fields(cls) -> list[tuple[str, int]]:
    return [(n, ctypes.sizeof(t)) for n, t in cls._fields_]


def test_job_record_layout():
    assert py_fields(W.GsJobRecord) == c_fields("gs_job_record")


def test_exec_stats_layout():
    assert py_fields(W.GsExecStats) == c_fields("gs_exec_stats")


def test_job_desc_layout():
    assert py_fields(W.GsJobDesc) == c_fields("gs_job_desc")


def test_launch_desc_layout():
    assert py_fields(W.GsLaunchDesc) == c_fields("gs_launch_desc")
