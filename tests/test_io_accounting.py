"""Byte accounting the bench reports (CPU only): the bytes an e2e job moves
over PCIe (gs_job_io_bytes: bfs's transposed CSR rebuilt on the device,
needle's score boundary only) and the executed algorithm's HBM bytes of a
hotspot job (four-step passes while four steps remain)."""

import pytest

from paper_2107_08538_b200 import catalog as C
from paper_2107_08538_b200 import workloads as W


@pytest.mark.parametrize("n", [1000, 300_000, 128_000_000])
def test_bfs_moves_its_csr_only(n):
    i, o = W.io_bytes(W.Job("bfs", n=n, seed=1))
    assert i == (n + 1) * 4 + n * 6 * 4      # row_ptr + col, not the transposed pair
    assert o == n * 4                          # the levels


@pytest.mark.parametrize("n", [512, 24576])
def test_needle_moves_reference_and_score_boundary(n):
    i, o = W.io_bytes(W.Job("needle", n=n, seed=1))
    assert i == n * n * 4 + (n + 4) * 4 + 16 * n
    assert o == (n + 1) * (n + 4) * 4          # the whole score matrix comes back


def test_hotspot_moves_both_maps():
    n = 1024
    i, o = W.io_bytes(W.Job("hotspot", n=n, iters=40, seed=1))
    assert i == 2 * n * n * 4 and o == n * n * 4


@pytest.mark.parametrize("iters,passes", [(40, 10), (4, 1), (6, 2), (7, 3), (3, 2), (1, 1)])
def test_hotspot_algorithmic_bytes_follow_the_passes(iters, passes, monkeypatch):
    monkeypatch.delenv("GS_HOTSPOT_STEPS", raising=False)
    n = 2048
    work, unit = C.algorithmic_work(W.Job("hotspot", n=n, iters=iters, seed=1))
    assert unit == "B" and work == 12.0 * n * n * passes


def test_hotspot_two_step_mode(monkeypatch):
    monkeypatch.setenv("GS_HOTSPOT_STEPS", "2")
    work, _ = C.algorithmic_work(W.Job("hotspot", n=2048, iters=40, seed=1))
    assert work == 12.0 * 2048 * 2048 * 20
