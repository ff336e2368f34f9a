"""In-tree build of the native library (sm_100a only).

    python -m paper_2107_08538_b200.build [--force]

Each csrc/*.cu is compiled to an object with nvcc (in parallel), then linked
into paper_2107_08538_b200/libgs.so so it travels with the repo snapshot to
the GPU box.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "build")
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-I", os.path.join(REPO, "include")]

# source -> extra flags.  Workload kernels are built without FMA
# contraction: their arithmetic order is pinned to the CPU oracle's.
SOURCES = {
    "gs_sched.cu": [],
    "gs_work.cu": ["-fmad=false"],
    "gs_exec.cu": [],
    "gs_gemm.cu": [],
    "gs_darknet.cu": [],
    "gs_capture.cu": [],
}
TARGET = os.path.join(PKG, "libgs.so")


def _deps() -> list[str]:
    out = [os.path.join(REPO, "include", f) for f in os.listdir(os.path.join(REPO, "include"))]
    out += [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    return out


def _newer(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src: str, flags: list[str], verbose: bool) -> str:
    obj = os.path.join(OBJ, src.replace(".cu", ".o"))
    cmd = [NVCC, *ARCH, *COMMON, *flags, "-c", os.path.join(CSRC, src), "-o", obj]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    return obj


def build(force: bool = False, verbose: bool = False) -> list[str]:
    os.makedirs(OBJ, exist_ok=True)
    hdrs = _deps()
    todo = []
    for src, flags in SOURCES.items():
        obj = os.path.join(OBJ, src.replace(".cu", ".o"))
        if force or _newer(obj, [os.path.join(CSRC, src), *hdrs]):
            todo.append((src, flags))
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        list(ex.map(lambda sf: _compile(sf[0], sf[1], verbose), todo))
    objs = [os.path.join(OBJ, s.replace(".cu", ".o")) for s in SOURCES]
    if todo or force or _newer(TARGET, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", TARGET, *objs, "-lpthread"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        return [TARGET]
    return []


if __name__ == "__main__":
    for path in build(force="--force" in sys.argv, verbose=True):
        print("built", path)
