"""srad's branch-free IEEE division (gs_kernels.cuh srad_coeff_fast) is
bit-identical to __fdiv_rn inside its proven operand domain, and the fast
coefficient equals srad_coeff_one wherever it claims its proof
(pytest -m gpu).  The kernel-level parity (srad vs the oracle, bit-exact)
is in test_kernels_gpu.py / test_kernels_bench_gpu.py."""

import pytest

pytestmark = pytest.mark.gpu

W = pytest.importorskip("paper_2107_08538_b200.workloads")


@pytest.mark.parametrize("q0sqr", [0.037, 0.05, 1e-3, 3.0])
def test_fast_division_matches_ieee(q0sqr):
    r = W.selftest_division(1 << 27, seed=11 + int(q0sqr * 1000), q0sqr=q0sqr)
    assert r["div_checked"] > (1 << 25)        # most pairs fall inside the domain
    assert r["coeff_checked"] > (1 << 25)      # most windows take the fast path
    assert r["div_mismatches"] == 0
    assert r["coeff_mismatches"] == 0
