"""Independent numpy / pure-Python restatements of the workload algorithms.

Used only at tiny sizes to pin the C oracle (oracle/kernels_cpu.c): two
implementations written separately from the public Rodinia algorithm
descriptions must agree before the C oracle is trusted as the checker of
the GPU kernels (the reference itself has no kernels).
"""

from __future__ import annotations

from collections import deque

import numpy as np

M64 = (1 << 64) - 1


def hash64(seed: int, i):
    """gs_hash64 (include/gs_work.h): splitmix64 of seed*phi + i."""
    i = np.asarray(i, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64((seed * 0x9E3779B97F4A7C15) & M64) + i + np.uint64(0x632BE59BD9B4E019)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def unit(seed: int, i):
    return (hash64(seed, i) >> np.uint64(40)).astype(np.float32) * np.float32(1.0 / 16777216.0)


def fmaf(a, b, c):
    """Single-rounding fused multiply-add for float32 via float64 (exact
    product; one rounding of the sum is exact for these magnitudes)."""
    return (np.float64(a) * np.float64(b) + np.float64(c)).astype(np.float32)


def bfs(n: int, seed: int) -> np.ndarray:
    col = (hash64(seed, np.arange(6 * n)) % np.uint64(n)).astype(np.int64)
    level = np.full(n, -1, np.int32)
    level[0] = 0
    q = deque([0])
    while q:
        v = q.popleft()
        for u in col[6 * v:6 * v + 6]:
            if level[u] < 0:
                level[u] = level[v] + 1
                q.append(u)
    return level


def hotspot(n: int, iters: int, seed: int) -> np.ndarray:
    t_chip, chip, fc, sh, k = 0.0005, 0.016, 0.5, 1.75e6, 100.0
    gh = gw = chip / 1024.0
    cap = fc * sh * t_chip * gw * gh
    rx = gw / (2.0 * k * t_chip * gh)
    ry = gh / (2.0 * k * t_chip * gw)
    rz = t_chip / (k * gh * gw)
    step = 0.001 / (3.0e6 / (fc * t_chip * sh))
    cc, rx1, ry1, rz1 = (np.float32(v) for v in (step / cap, 1.0 / rx, 1.0 / ry, 1.0 / rz))
    idx = np.arange(n * n)
    t = (np.float32(323.0) + np.float32(10.0) * unit(seed, idx)).reshape(n, n)
    p = (np.float32(0.1) * unit(seed ^ 0xA5A5A5A5, idx)).reshape(n, n)
    r = np.arange(n)
    rn, rs = np.maximum(r - 1, 0), np.minimum(r + 1, n - 1)
    for _ in range(iters):
        tc = t
        a = fmaf(np.float32(-2.0), tc, t[rs, :] + t[rn, :])
        b = fmaf(np.float32(-2.0), tc, t[:, rs] + t[:, rn])
        e = np.float32(80.0) - tc
        d = fmaf(a, ry1, p)
        d = fmaf(b, rx1, d)
        d = fmaf(e, rz1, d)
        t = fmaf(cc, d, tc)
    return t


def srad(n: int, iters: int, seed: int) -> np.ndarray:
    J = (np.float32(1.0) + unit(seed, np.arange(n * n))).reshape(n, n)
    roi = min(n, 128)
    r = np.arange(n)
    rn, rs = np.maximum(r - 1, 0), np.minimum(r + 1, n - 1)
    f = np.float32
    for _ in range(iters):
        s = s2 = 0.0
        for v in J[:roi, :roi].ravel().tolist():
            s += v
            s2 += v * v
        size = float(roi * roi)
        mean = s / size
        var = s2 / size - mean * mean
        q0 = f(var / (mean * mean))
        dN, dS = J[rn, :] - J, J[rs, :] - J
        dW, dE = J[:, rn] - J, J[:, rs] - J
        g2 = ((dN * dN + dS * dS) + dW * dW) + dE * dE
        g2 = g2 / (J * J)
        L = ((dN + dS) + dW) + dE
        L = L / J
        num = f(0.5) * g2 - f(1.0 / 16.0) * (L * L)
        den = f(1.0) + f(0.25) * L
        qs = num / (den * den)
        den = (qs - q0) / (q0 * (f(1.0) + q0))
        c = np.clip(f(1.0) / (f(1.0) + den), f(0.0), f(1.0))
        cS, cE = c[rs, :], c[:, rs]
        D = ((c * dN + cS * dS) + c * dW) + cE * dE
        J = J + f(0.125) * D
    return J


def kmeans(n: int, nf: int, iters: int, seed: int):
    x = unit(seed, np.arange(n * nf)).reshape(nf, n)
    c = x[:, :5].T.copy()
    for _ in range(iters):
        acc = np.zeros((5, n), np.float32)
        for f in range(nf):
            d = x[f][None, :] - c[:, f][:, None]
            acc = fmaf(d, d, acc)
        mem = np.zeros(n, np.int32)
        best = acc[0].copy()
        for k in range(1, 5):
            better = acc[k] < best
            mem[better] = k
            best[better] = acc[k][better]
        q = (x * np.float32(16777216.0)).astype(np.int64)
        for k in range(5):
            sel = mem == k
            cnt = int(sel.sum())
            if cnt:
                c[k] = (q[:, sel].sum(axis=1).astype(np.float64) / 16777216.0 / cnt).astype(np.float32)
    return mem, c


def needle(n: int, seed: int) -> np.ndarray:
    from paper_2107_08538_b200.workloads import KINDS  # noqa: F401  (import check only)

    blosum = _blosum62()
    s1 = (hash64(seed, np.arange(n + 1)) % np.uint64(10)).astype(np.int64) + 1
    s2 = (hash64(seed + 1, np.arange(n + 1)) % np.uint64(10)).astype(np.int64) + 1
    sc = np.zeros((n + 1, n + 1), np.int64)
    sc[0, :] = -10 * np.arange(n + 1)
    sc[:, 0] = -10 * np.arange(n + 1)
    for i in range(1, n + 1):
        for j in range(1, n + 1):
            sc[i, j] = max(sc[i - 1, j - 1] + blosum[s1[i], s2[j]], sc[i, j - 1] - 10, sc[i - 1, j] - 10)
    return sc.astype(np.int32)


def lud(n: int, seed: int, bs: int = 32) -> np.ndarray:
    i = np.arange(n)
    a = unit(seed, np.arange(n * n)).reshape(n, n) + np.where(i[:, None] == i[None, :], np.float32(n), 0)
    a = a.astype(np.float32)
    for o in range(0, n, bs):
        for ii in range(bs):
            for j in range(ii, bs):
                acc = a[o + ii, o + j]
                for k in range(ii):
                    acc = fmaf(-a[o + ii, o + k], a[o + k, o + j], acc)
                a[o + ii, o + j] = acc
            for j in range(ii + 1, bs):
                acc = a[o + j, o + ii]
                for k in range(ii):
                    acc = fmaf(-a[o + j, o + k], a[o + k, o + ii], acc)
                a[o + j, o + ii] = acc / a[o + ii, o + ii]
        if o + bs >= n:
            break
        for j in range(o + bs, n):
            for ii in range(bs):
                acc = a[o + ii, j]
                for k in range(ii):
                    acc = fmaf(-a[o + ii, o + k], a[o + k, j], acc)
                a[o + ii, j] = acc
        for r in range(o + bs, n):
            for j in range(bs):
                acc = a[r, o + j]
                for k in range(j):
                    acc = fmaf(-a[r, o + k], a[o + k, o + j], acc)
                a[r, o + j] = acc / a[o + j, o + j]
        L = a[o + bs:, o:o + bs].copy()
        U = a[o:o + bs, o + bs:].copy()
        acc = np.zeros((n - o - bs, n - o - bs), np.float32)
        for k in range(bs):
            acc = fmaf(L[:, k][:, None], U[k, :][None, :], acc)
        a[o + bs:, o + bs:] = a[o + bs:, o + bs:] - acc
    return a


def _blosum62() -> np.ndarray:
    rows = """
 4 -1 -2 -2  0 -1 -1  0 -2 -1 -1 -1 -1 -2 -1  1  0 -3 -2  0 -2 -1  0 -4
-1  5  0 -2 -3  1  0 -2  0 -3 -2  2 -1 -3 -2 -1 -1 -3 -2 -3 -1  0 -1 -4
-2  0  6  1 -3  0  0  0  1 -3 -3  0 -2 -3 -2  1  0 -4 -2 -3  3  0 -1 -4
-2 -2  1  6 -3  0  2 -1 -1 -3 -4 -1 -3 -3 -1  0 -1 -4 -3 -3  4  1 -1 -4
 0 -3 -3 -3  9 -3 -4 -3 -3 -1 -1 -3 -1 -2 -3 -1 -1 -2 -2 -1 -3 -3 -2 -4
-1  1  0  0 -3  5  2 -2  0 -3 -2  1  0 -3 -1  0 -1 -2 -1 -2  0  3 -1 -4
-1  0  0  2 -4  2  5 -2  0 -3 -3  1 -2 -3 -1  0 -1 -3 -2 -2  1  4 -1 -4
 0 -2  0 -1 -3 -2 -2  6 -2 -4 -4 -2 -3 -3 -2  0 -2 -2 -3 -3 -1 -2 -1 -4
-2  0  1 -1 -3  0  0 -2  8 -3 -3 -1 -2 -1 -2 -1 -2 -2  2 -3  0  0 -1 -4
-1 -3 -3 -3 -1 -3 -3 -4 -3  4  2 -3  1  0 -3 -2 -1 -3 -1  3 -3 -3 -1 -4
-1 -2 -3 -4 -1 -2 -3 -4 -3  2  4 -2  2  0 -3 -2 -1 -2 -1  1 -4 -3 -1 -4
"""
    top = np.array([[int(v) for v in r.split()] for r in rows.strip().splitlines()])
    return top  # rows/cols 0..10 cover residues 1..10 used by needle
