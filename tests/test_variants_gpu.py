"""Opt-in kernel variants, run in a subprocess with their switch set, against
the CPU oracle: hotspot's four-step pass (GS_HOTSPOT_STEPS=4, four
barrier-separated steps per shared-memory tile; edge tiles re-clamp every
intermediate buffer) — kept for measurement, bit-exact like the default."""

import json
import os
import subprocess
import sys

import pytest

from oracle import kernels as K

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _checksum(kind, env, **kw) -> int:
    args = ", ".join(f"{k}={v!r}" for k, v in kw.items())
    code = ("import json,sys; sys.path.insert(0, %r); from paper_2107_08538_b200 import workloads as W; "
            "o, r = W.run_solo(W.Job(%r, %s)); print(json.dumps(int(r.checksum)))") % (REPO, kind, args)
    out = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env), capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("n,iters", [(256, 4), (512, 9), (1024, 10), (384, 7)])
def test_hotspot_four_step_pass_matches_oracle(n, iters):
    got = _checksum("hotspot", {"GS_HOTSPOT_STEPS": "4"}, n=n, iters=iters, seed=5)
    want = K.run("hotspot", n=n, iters=iters, seed=5)
    assert got == K.digest("hotspot", want)


@pytest.mark.parametrize("n", [256, 512, 1024])
def test_needle_8x8_bands_match_oracle(n):
    """needle_bands8 (GS_NEEDLE8=1: 8 x 8 blocks per lane step, 256-row
    bands, tagged-word band handoff) — bit-exact scores."""
    got = _checksum("needle", {"GS_NEEDLE8": "1"}, n=n, seed=9)
    want = K.run("needle", n=n, seed=9)
    assert got == K.digest("needle", want)
