"""Workload kernels at the BENCHMARKED sizes vs the CPU oracle (pytest -m gpu).

Every template the bench's cfg 1 mix draws from (catalog.RODINIA, small and
large class, the exact job sizes bench.py runs) is run on the GPU and by the
oracle (oracle/kernels_cpu.c, all host threads) on the same seeded inputs:

* bfs levels, needle scores, kmeans membership, hotspot and srad grids:
  bit-exact (the kernels are built with -fmad=false and the oracle's
  arithmetic order);
* backprop weights and lud factors: within 1e-5 relative (north_star's float
  bar; double / FMA-chain accumulation order), and the exactness is
  reported.

The executor's output digest of the GPU run must also equal the oracle's
digest of the oracle output (oracle.kernels.digest), which is what the bench
line's "parity" block checks for the co-located jobs of every timed step.
"""

import numpy as np
import pytest

from oracle import kernels as K

pytestmark = pytest.mark.gpu

W = pytest.importorskip("paper_2107_08538_b200.workloads")
C = pytest.importorskip("paper_2107_08538_b200.catalog")

EXACT = {"bfs", "hotspot", "srad", "kmeans", "needle"}
CASES = [(f"{kind}_{cls}", kind, kw) for kind, (small, large) in C.RODINIA.items()
         for cls, kw in (("small", small), ("large", large))]


@pytest.mark.parametrize("tpl,kind,kw", CASES, ids=[c[0] for c in CASES])
def test_bench_size_kernel_matches_oracle(tpl, kind, kw):
    job = W.Job(kind, seed=1001, **kw)
    got, rec = W.run_solo(job)
    assert rec.state == 0 and rec.n_kernels > 0
    want = K.run(kind, n=job.n, iters=job.iters, m=job.m, seed=job.seed)
    if kind in EXACT:
        np.testing.assert_array_equal(got, want)
        assert rec.checksum == K.digest(kind, want)
    else:
        np.testing.assert_allclose(got, want, rtol=1e-5, atol=1e-5)
        exact = bool(np.array_equal(got, want))
        print(f"{tpl}: max |err| {float(np.max(np.abs(got - want))):.3g}, bit-exact {exact}")
        if exact:
            assert rec.checksum == K.digest(kind, want)


@pytest.mark.parametrize("tpl,kind,kw", CASES, ids=[c[0] for c in CASES])
def test_bench_template_probe_matches_host_footprint(tpl, kind, kw):
    """The CPU reference arm places the mix with catalog.host_footprint; it
    must be the probe's mem_bytes (gs_job_probe, the executor's capture)."""
    job = W.Job(kind, seed=1001, **kw)
    assert W.probe(job).mem_bytes == C.host_footprint(job)
