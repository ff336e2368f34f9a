"""tcgen05 GEMM throughput (csrc/gs_gemm.cu) vs cuBLAS on the same shapes.

    python tools/gemm_bench.py
"""

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2107_08538_b200 import workloads as W  # noqa: E402


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for m, n, k in [(8192, 8192, 8192), (16384, 1024, 4608), (65536, 256, 1152), (200704, 64, 576), (12544, 512, 4608)]:
    a = torch.randn(m, k, device="cuda").to(torch.bfloat16)
    b = torch.randn(n, k, device="cuda").to(torch.bfloat16)
    out = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    ms = timeit(lambda: W.gemm_bf16(a, b, None, out=out))
    ms_cublas = timeit(lambda: torch.matmul(a, b.T))
    fl = 2.0 * m * n * k
    print(json.dumps({"m": m, "n": n, "k": k, "ours_ms": round(ms, 4), "ours_tflops": round(fl / ms / 1e9, 1),
                      "cublas_ms": round(ms_cublas, 4), "cublas_tflops": round(fl / ms_cublas / 1e9, 1)}), flush=True)
