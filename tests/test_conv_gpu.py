"""Implicit-GEMM convolution (gemm_bf16_tc<BN, true>: A gathered from the
NHWC activation by cp.async, no im2row matrix) against the im2row + GEMM
path it replaces.  The gather writes the same K-major swizzled tile the TMA
wrote from the im2row matrix, so the networks' outputs must be bit-identical
(same products, same accumulation order).  GS_IM2ROW=1 forces the old path
in a subprocess."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

W = pytest.importorskip("paper_2107_08538_b200.workloads")

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = [("yolo", 160, 2), ("yolo", 416, 4), ("resnet", 64, 2), ("resnet", 224, 3)]


def _digest(kind, n, m, im2row: bool, env_extra=None) -> tuple[int, float]:
    code = ("import json,sys; sys.path.insert(0, %r); from paper_2107_08538_b200 import workloads as W; "
            "o, r = W.run_solo(W.Job(%r, n=%d, m=%d, iters=1, seed=7)); "
            "print(json.dumps([int(r.checksum), float(r.compute_ms)]))") % (REPO, kind, n, m)
    env = dict(os.environ, GS_IM2ROW="1" if im2row else "0", **(env_extra or {}))
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    cs, ms = json.loads(out.stdout.strip().splitlines()[-1])
    return cs, ms


@pytest.mark.parametrize("kind,n,m", CASES, ids=[f"{k}{n}x{m}" for k, n, m in CASES])
def test_implicit_conv_equals_im2row(kind, n, m):
    a, ta = _digest(kind, n, m, im2row=False)
    b, tb = _digest(kind, n, m, im2row=True)
    print(f"{kind} {n}^2 x {m}: implicit {ta:.3f} ms, im2row {tb:.3f} ms")
    assert a == b


@pytest.mark.parametrize("n,m", [(160, 2), (608, 2)])
def test_fused_layer0_pool_equals_separate(n, m):
    """YOLO layer 0 fused with its 2x2 max-pool (conv3x3_pool2) == the direct
    convolution + the max-pool kernel, bit for bit (the network's output)."""
    a, ta = _digest("yolo", n, m, im2row=False)
    b, tb = _digest("yolo", n, m, im2row=False, env_extra={"GS_NO_POOL_FUSION": "1"})
    print(f"yolo {n}^2 x {m}: fused {ta:.3f} ms, separate {tb:.3f} ms")
    assert a == b
