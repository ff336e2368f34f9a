"""Pin the C workload oracle (oracle/kernels_cpu.c) against independent
numpy / pure-Python restatements at tiny sizes (CPU only)."""

import numpy as np
import pytest

import kernels_ref as R
from oracle import kernels as K


@pytest.mark.parametrize("n,seed", [(64, 1), (1000, 7), (4096, 3)])
def test_bfs_levels_match(n, seed):
    lv, depth = K.bfs(n, seed)
    np.testing.assert_array_equal(lv, R.bfs(n, seed))
    assert depth == lv.max() + 1


@pytest.mark.parametrize("n,iters", [(128, 1), (128, 5)])
def test_hotspot_matches(n, iters):
    np.testing.assert_array_equal(K.hotspot(n, iters, 3), R.hotspot(n, iters, 3))


@pytest.mark.parametrize("n,iters", [(128, 1), (256, 3)])
def test_srad_matches(n, iters):
    np.testing.assert_allclose(K.srad(n, iters, 5), R.srad(n, iters, 5), rtol=1e-6)


def test_kmeans_matches():
    mem, cent = K.kmeans(3000, 8, 4, 11)
    rmem, rcent = R.kmeans(3000, 8, 4, 11)
    np.testing.assert_array_equal(mem, rmem)
    np.testing.assert_allclose(cent, rcent, rtol=1e-6)


@pytest.mark.parametrize("n,seed", [(32, 1), (96, 4)])
def test_needle_matches(n, seed):
    np.testing.assert_array_equal(K.needle(n, seed), R.needle(n, seed))


def test_needle_known_answer():
    """Hand-checkable corner: score[0][j] = -10 j, score[i][0] = -10 i, and
    score[1][1] = max(0 + blosum, -20, -20)."""
    s = K.needle(32, 9)
    assert list(s[0, :4]) == [0, -10, -20, -30]
    assert list(s[:4, 0]) == [0, -10, -20, -30]
    b = R._blosum62()
    s1 = int(R.hash64(9, 1) % np.uint64(10)) + 1
    s2 = int(R.hash64(10, 1) % np.uint64(10)) + 1
    assert s[1, 1] == max(int(b[s1, s2]), -20)


def test_lud_matches_and_factors():
    n = 96
    a = K.lud(n, 2)
    np.testing.assert_allclose(a, R.lud(n, 2), rtol=1e-5, atol=1e-5)
    L = np.tril(a, -1).astype(np.float64) + np.eye(n)
    U = np.triu(a).astype(np.float64)
    i = np.arange(n)
    A = R.unit(2, np.arange(n * n)).reshape(n, n).astype(np.float64) + np.where(i[:, None] == i[None, :], n, 0)
    np.testing.assert_allclose(L @ U, A, rtol=1e-5, atol=1e-3)


def test_backprop_forward_and_update():
    w1, w2, hid, o = K.backprop(4000, 16, 1, 3)
    x = np.concatenate([[1.0], R.unit(3, np.arange(1, 4001)).astype(np.float64)])
    w1_0 = ((R.unit(4, np.arange(16 * 4001)) - np.float32(0.5)) * np.float32(2e-3)).reshape(16, 4001)
    s = w1_0.astype(np.float64) @ x
    h = 1.0 / (1.0 + np.exp(-s.astype(np.float32).astype(np.float64)))
    np.testing.assert_allclose(hid[1:], h, rtol=1e-5)
    assert 0.0 < o < 1.0
    assert w1.shape == (4001, 16)  # [input][hidden], Rodinia's input_weights layout
    assert not np.array_equal(w1, w1_0.T)  # weights moved
