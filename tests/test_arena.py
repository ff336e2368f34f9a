"""The executor's job arena (csrc/gs_arena.h) on the host: randomized
all-or-nothing placement against a granule occupancy model (no overlap,
exact accounting, full coalescing), the per-run limit, and the wait a
memory-safe job makes when only fragmentation stands in its way."""

import os
import shutil
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_arena_random_ops(tmp_path, seed):
    exe = tmp_path / "arena_check"
    cuda_inc = "/usr/local/cuda/include"
    subprocess.run(["g++", "-O2", "-std=c++17", "-pthread", f"-I{cuda_inc}",
                    os.path.join(HERE, "native", "arena_check.cpp"), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe), str(seed)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    ok, placed, refused = out.stdout.split()
    assert ok == "ok" and int(placed) > 1000 and int(refused) > 10
