"""In-tree build of the native libraries (sm_100a only).

    python -m paper_2107_08538_b200.build

Each shared library is compiled with nvcc straight from csrc/ into the
package directory so it travels with the repo snapshot to the GPU box.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC,-O3",
          "-I", os.path.join(REPO, "include")]

# library -> (sources, extra flags)
LIBS = {
    "libgs.so": (["gs_sched.cu"], []),
}


def _stale(target: str, sources: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    deps = sources + [os.path.join(REPO, "include", f) for f in os.listdir(os.path.join(REPO, "include"))]
    deps += [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    return any(os.path.getmtime(s) > t for s in deps)


def build(force: bool = False, verbose: bool = False) -> list[str]:
    built = []
    for lib, (srcs, extra) in LIBS.items():
        sources = [os.path.join(CSRC, s) for s in srcs]
        target = os.path.join(PKG, lib)
        if not force and not _stale(target, sources):
            continue
        cmd = [NVCC, *ARCH, *COMMON, *extra, "-o", target, *sources]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
        built.append(target)
    return built


if __name__ == "__main__":
    for path in build(force="--force" in sys.argv, verbose=True):
        print("built", path)
