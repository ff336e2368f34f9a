"""GPU workload kernels vs the CPU oracle (pytest -m gpu).

Integer outputs (bfs levels, needle scores, kmeans membership) must be
bit-exact; float outputs within 1e-5 relative (BASELINE.json north_star).
"""

import numpy as np
import pytest

from oracle import kernels as K

pytestmark = pytest.mark.gpu

W = pytest.importorskip("paper_2107_08538_b200.workloads")

CASES = [
    ("bfs", dict(n=200_000, seed=3), "exact"),
    ("bfs", dict(n=1_000_003, seed=8), "exact"),
    ("hotspot", dict(n=512, iters=10, seed=2), "exact"),   # 5 two-step passes
    ("hotspot", dict(n=1024, iters=3, seed=5), "exact"),   # one two-step pass + one single step
    ("hotspot", dict(n=128, iters=2, seed=6), "exact"),    # grid edges on every side of one tile column
    ("hotspot", dict(n=256, iters=5, seed=7), "exact"),
    # four-step passes (120 x 32 tiles in 128-wide boxes): an east edge that
    # falls exactly on a tile boundary (1920 = 16 x 120), one inside the last
    # tile (640), and pass4 + two-step + single-step remainders
    ("hotspot", dict(n=1920, iters=8, seed=11), "exact"),
    ("hotspot", dict(n=640, iters=4, seed=12), "exact"),
    ("hotspot", dict(n=640, iters=7, seed=13), "exact"),
    ("hotspot", dict(n=384, iters=6, seed=14), "exact"),
    ("srad", dict(n=512, iters=5, seed=4), "exact"),
    ("srad", dict(n=128, iters=3, seed=8), "exact"),     # one tile: every halo is a grid edge
    ("srad", dict(n=384, iters=2, seed=9), "exact"),
    ("kmeans", dict(n=200_000, m=34, iters=5, seed=6), "exact"),
    ("backprop", dict(n=300_000, m=16, iters=2, seed=7), 1e-5),
    ("needle", dict(n=128, seed=2), "exact"),     # one chunk, 4 bands
    ("needle", dict(n=384, seed=3), "exact"),     # odd chunk count
    ("needle", dict(n=512, seed=1), "exact"),
    ("needle", dict(n=1024, seed=9), "exact"),
    ("needle", dict(n=4096, seed=4), "exact"),    # 128 bands in a wavefront
    ("kmeans", dict(n=100_003, m=8, iters=3, seed=5), "exact"),    # nf < 32, ragged tail
    ("kmeans", dict(n=65_537, m=40, iters=2, seed=6), "exact"),    # generic nf > 32
    ("kmeans", dict(n=200_004, m=34, iters=3, seed=7), "exact"),   # the catalog's 34 features, partial last tile
    ("lud", dict(n=160, seed=4), 1e-5),           # trailing edge exactly one 128 tile
    ("lud", dict(n=512, seed=3), 1e-5),
    ("lud", dict(n=1056, seed=5), 1e-5),          # partial 128 tiles
]


@pytest.mark.parametrize("kind,kw,tol", CASES, ids=[f"{c[0]}-{c[1]['n']}" for c in CASES])
def test_gpu_kernel_matches_oracle(kind, kw, tol):
    job = W.Job(kind, **kw)
    got, rec = W.run_solo(job)
    want = K.run(kind, **kw)
    assert rec.state == 0 and rec.n_kernels > 0
    if tol == "exact":
        np.testing.assert_array_equal(got, want)
    else:
        np.testing.assert_allclose(got, want, rtol=tol, atol=tol)


def test_kmeans_centroids_exact():
    """Fixed-point centroid sums make the recentering exact."""
    from paper_2107_08538_b200 import workloads as Wm

    job = Wm.Job("kmeans", n=50_000, m=8, iters=3, seed=2)
    mem, _ = Wm.run_solo(job)
    cmem, _ = K.kmeans(50_000, 8, 3, 2)
    np.testing.assert_array_equal(mem, cmem)


def test_probe_reports_footprint_and_shape():
    job = W.Job("hotspot", n=1024, iters=1)
    p = W.probe(job)
    assert p.mem_bytes == 8 * 2**20 + 3 * 4 * 2**20 + 2 * 2**20  # 3 x 4 MiB buffers + control granule + 8 MiB heap
    assert p.thread_blocks == 296 and p.threads_per_block == 256 and p.warps_per_block == 8
    assert 0 < p.regs_per_thread <= 255


MIX = [W.Job("bfs", n=300_000, seed=1), W.Job("hotspot", n=1024, iters=20, seed=2),
       W.Job("srad", n=1024, iters=5, seed=3), W.Job("kmeans", n=200_000, m=34, iters=3, seed=4),
       W.Job("backprop", n=200_000, m=16, iters=1, seed=5), W.Job("needle", n=1024, seed=6),
       W.Job("lud", n=1024, seed=7), W.Job("bfs", n=500_000, seed=8)]


@pytest.mark.parametrize("policy", ["mgb-warps", "mgb-sm", "sa", "cg:4"])
def test_executor_runs_mix_with_solo_checksums(policy):
    solo = [W.run_solo(j)[1].checksum for j in MIX]
    res = W.run_jobs(MIX, policy=policy, workers=4)
    assert res.completed == len(MIX) and res.crashed == 0 and res.oom == 0
    assert [r["checksum"] for r in res.records] == solo
    assert res.kernel_launches > len(MIX) and res.decision_launches >= len(MIX)


def test_executor_memory_safe_under_a_tight_ledger():
    """A ledger smaller than the mix's footprint forces deferrals; mgb never
    OOMs and every job still completes."""
    tight = max(W.probe(j).mem_bytes for j in MIX) * 2
    res = W.run_jobs(MIX, policy="mgb-warps", workers=8, ledger_bytes=tight)
    assert res.completed == len(MIX) and res.oom == 0
    assert max(r["wait_ms"] for r in res.records) > 0.0


def test_executor_e2e_mode_moves_bytes():
    W.stage(MIX[:3], [0], W.MODE_E2E)
    try:
        res = W.run_jobs(MIX[:3], policy="mgb-warps", workers=3, mode=W.MODE_E2E)
    finally:
        W.unstage()
    assert res.completed == 3
    for r, j in zip(res.records, MIX[:3]):
        i, _ = W.io_bytes(j)
        assert r["h2d_bytes"] == i and r["d2h_bytes"] > 0


def test_executor_colocated_darknet_jobs_match_solo():
    """YOLO / ResNet jobs co-located with each other and with Rodinia kinds:
    the GEMM's tiles come from the job's ticket counter, whose order differs
    run to run, yet every output checksum equals the job's solo run."""
    jobs = [W.Job("yolo", n=416, m=2, iters=1, seed=11), W.Job("resnet", n=224, m=2, iters=1, seed=12),
            W.Job("yolo", n=320, m=4, iters=1, seed=13), MIX[1], MIX[3], W.Job("resnet", n=224, m=1, iters=1, seed=14)]
    solo = [W.run_solo(j)[1].checksum for j in jobs]
    for policy in ("mgb-warps", "cg:6"):
        res = W.run_jobs(jobs, policy=policy, workers=6)
        assert res.completed == len(jobs) and res.oom == 0
        assert [r["checksum"] for r in res.records] == solo


def test_executor_poisson_arrivals():
    """Jobs arrive over time (cfg 3): none is pulled before it arrives,
    turnaround is measured from arrival, outputs equal the solo runs."""
    arrivals = [0.0, 2.0, 4.0, 30.0, 31.0, 60.0, 61.0, 90.0]
    solo = [W.run_solo(j)[1].checksum for j in MIX]
    res = W.run_jobs(MIX, policy="mgb-warps", workers=4, arrivals_ms=arrivals)
    assert res.completed == len(MIX)
    for r, a, c in zip(res.records, arrivals, solo):
        assert r["arrival_ms"] == a and r["pull_ms"] >= a - 0.5
        assert abs(r["turnaround_ms"] - (r["end_ms"] - a)) < 1e-6
        assert r["checksum"] == c
    assert res.makespan_ms >= arrivals[-1]


def test_lud_panels_colocated_are_deterministic():
    """lud's panel launches read the diagonal block in every CTA and write
    it back factored; under co-location some CTAs start late, so the write
    must wait for the last reader (it once came from block 0 and raced)."""
    jobs = [W.Job("lud", n=1024, seed=21), W.Job("hotspot", n=2048, iters=20, seed=22),
            W.Job("lud", n=2048, seed=23), W.Job("srad", n=2048, iters=4, seed=24),
            W.Job("lud", n=1056, seed=25), W.Job("hotspot", n=2048, iters=20, seed=26)]
    solo = [W.run_solo(j)[1].checksum for j in jobs]
    for _ in range(4):
        res = W.run_jobs(jobs, policy="cg:6", workers=6)
        assert [r["checksum"] for r in res.records] == solo


@pytest.mark.parametrize("policy", ["mgb-warps", "sa"])
def test_executor_places_across_two_ledgers(policy):
    """Two ledgers (both on this GPU, memory split between them): one
    decision authority places the mix across devices; every job lands on one
    of them and reproduces its solo output."""
    solo = [W.run_solo(j)[1].checksum for j in MIX]
    cap = W.ledger_capacity(0) // 2
    res = W.run_jobs(MIX, policy=policy, devices=[0, 0], workers=8, ledger_bytes=cap)
    assert res.completed == len(MIX) and res.oom == 0
    assert [r["checksum"] for r in res.records] == solo
    used = {r["device"] for r in res.records}
    assert used <= {0, 1} and len(used) == 2


def test_executor_resident_inputs_match_solo():
    """Inputs staged in HBM (bench cfg 1): IN buffers are read in place and
    the INOUT buffers of hotspot / srad / backprop / needle are read by the
    job's first kernel straight from the staged copy (no private copy), yet
    every output checksum equals the job's solo run, which generates its
    inputs into its own buffers.  Odd and even pass counts cover both
    ping-pong parities; each template runs twice so two jobs read one staged
    input concurrently."""
    jobs = [W.Job("hotspot", n=512, iters=1, seed=21), W.Job("hotspot", n=512, iters=4, seed=22),
            W.Job("hotspot", n=1024, iters=5, seed=23), W.Job("srad", n=512, iters=1, seed=24),
            W.Job("srad", n=384, iters=4, seed=25), W.Job("backprop", n=300_000, m=16, iters=1, seed=26),
            W.Job("backprop", n=300_000, m=8, iters=3, seed=27), W.Job("needle", n=512, seed=28),
            W.Job("needle", n=1024, seed=29), W.Job("bfs", n=200_000, seed=30),
            W.Job("kmeans", n=100_003, m=34, iters=2, seed=31), W.Job("lud", n=512, seed=32)]
    solo = [W.run_solo(j)[1].checksum for j in jobs]
    W.stage(jobs, [0], W.MODE_DEVICE)
    try:
        res = W.run_jobs(jobs + jobs, policy="mgb-warps", workers=6)
    finally:
        W.unstage()
    assert res.completed == 2 * len(jobs) and res.oom == 0
    assert [r["checksum"] for r in res.records] == solo + solo


def test_executor_e2e_rebuilds_derived_inputs():
    """Inputs in pinned host memory: bfs rebuilds its transposed CSR on the
    device instead of copying it, needle copies only its score matrix's
    boundary; outputs still equal the solo runs and the bytes moved equal
    gs_job_io_bytes (less than the jobs' whole input buffers)."""
    jobs = [W.Job("bfs", n=300_000, seed=41), W.Job("needle", n=1024, seed=42), W.Job("bfs", n=1_000_003, seed=43),
            W.Job("bfs", n=1000, seed=46),  # bitmap smaller than the scan's scratch
            W.Job("needle", n=512, seed=44), W.Job("hotspot", n=512, iters=3, seed=45)]
    solo = [W.run_solo(j)[1].checksum for j in jobs]
    W.stage(jobs, [0], W.MODE_E2E)
    try:
        res = W.run_jobs(jobs, policy="mgb-warps", workers=3, mode=W.MODE_E2E)
    finally:
        W.unstage()
    assert res.completed == len(jobs) and res.oom == 0
    assert [r["checksum"] for r in res.records] == solo
    for r, j in zip(res.records, jobs):
        i, _ = W.io_bytes(j)
        assert r["h2d_bytes"] == i
        n = j.n
        if j.kind == "bfs":  # row_ptr + col only (not the transposed pair)
            assert i == (n + 1) * 4 + n * 6 * 4
        if j.kind == "needle":  # the reference matrix + the score boundary
            assert i == n * n * 4 + (n + 4) * 4 + 16 * n
