"""Reference Monte-Carlo random walk (numpy) -- TEST INFRASTRUCTURE ONLY.

Mirrors the walk rules of the paper's MC comparison (step length
l = sqrt(4 D t_s / T); rejection at barriers) with the same
counter-based generator as the GPU cross-check (Philox4x32-10, key = (seed,
walker), counter = (step low, step high, draw, 0x5eed5eed)), written
independently in numpy so that trajectories can be compared bit for bit.
Vectorised over walkers; meant for a few hundred walkers.
"""
from __future__ import annotations

import numpy as np

M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
W0, W1 = np.uint32(0x9E3779B9), np.uint32(0xBB67AE85)
MASK32 = np.uint64(0xFFFFFFFF)


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Philox4x32-10 on uint32 arrays (Salmon et al., SC'11)."""
    c0, c1, c2, c3 = (np.asarray(v, dtype=np.uint32) for v in (c0, c1, c2, c3))
    k0 = np.asarray(k0, dtype=np.uint32).copy()
    k1 = np.asarray(k1, dtype=np.uint32).copy()
    for _ in range(10):
        p0 = M0 * c0.astype(np.uint64)
        p1 = M1 * c2.astype(np.uint64)
        hi0, lo0 = (p0 >> np.uint64(32)).astype(np.uint32), (p0 & MASK32).astype(np.uint32)
        hi1, lo1 = (p1 >> np.uint64(32)).astype(np.uint32), (p1 & MASK32).astype(np.uint32)
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
        k0 = (k0 + W0).astype(np.uint32)
        k1 = (k1 + W1).astype(np.uint32)
    return c0, c1, c2, c3


def u01(hi, lo):
    m = ((hi.astype(np.uint64) >> np.uint64(5)) << np.uint64(26)) | (lo.astype(np.uint64) >> np.uint64(6))
    return m.astype(np.float64) * (1.0 / 9007199254740992.0)


def walk(mask, sources, K, T, l, seed, walkers=None):
    """Displacements [W][2] (pixel units) of walkers w = 0 .. S*K-1 (walker w
    starts at source w mod S), or of the given walker indices, after T steps
    of length l pixels."""
    mask = np.asarray(mask).astype(bool)
    ny, nx = mask.shape
    src = np.asarray(sources, dtype=np.int64).reshape(-1, 2)
    w = np.arange(len(src) * K) if walkers is None else np.asarray(walkers)
    s = w % len(src)
    x0 = src[s, 0] + 0.5
    y0 = src[s, 1] + 0.5
    x, y = x0.copy(), y0.copy()
    key0 = np.full(w.shape, seed, dtype=np.uint32)
    key1 = w.astype(np.uint32)

    def blocked(i, j):
        out = (i < 0) | (j < 0) | (i >= nx) | (j >= ny)
        ok = ~out
        res = out.copy()
        res[ok] = mask[j[ok], i[ok]]
        return res

    for t in range(T):
        a = np.zeros_like(x)
        b = np.zeros_like(x)
        r2 = np.zeros_like(x)
        todo = np.ones(x.shape, dtype=bool)
        draw = 0
        while todo.any():
            idx = np.nonzero(todo)[0]
            c = philox4x32_10(np.full(idx.shape, t & 0xFFFFFFFF, np.uint32), np.full(idx.shape, t >> 32, np.uint32),
                              np.full(idx.shape, draw, np.uint32), np.full(idx.shape, 0x5eed5eed, np.uint32),
                              key0[idx], key1[idx])
            aa = 2.0 * u01(c[0], c[1]) - 1.0
            bb = 2.0 * u01(c[2], c[3]) - 1.0
            rr = aa * aa + bb * bb
            acc = (rr > 0.0) & (rr <= 1.0)
            a[idx[acc]], b[idx[acc]], r2[idx[acc]] = aa[acc], bb[acc], rr[acc]
            todo[idx[acc]] = False
            draw += 1
        sc = l / np.sqrt(r2)
        nxp, nyp = x + a * sc, y + b * sc
        ci, cj = np.floor(x).astype(np.int64), np.floor(y).astype(np.int64)
        ei, ej = np.floor(nxp).astype(np.int64), np.floor(nyp).astype(np.int64)
        moved = (ei != ci) | (ej != cj)
        ok = np.ones(x.shape, dtype=bool)
        with np.errstate(divide="ignore", invalid="ignore"):
            tx = np.where(ei != ci, (np.where(ei > ci, ei, ci) - x) / (nxp - x), 2.0)
            ty = np.where(ej != cj, (np.where(ej > cj, ej, cj) - y) / (nyp - y), 2.0)
        fi = np.where(tx <= ty, ei, ci)          # first crossing: x edge first (or the corner)
        fj = np.where(ty <= tx, ej, cj)
        ok &= ~(moved & blocked(fi, fj))
        second = moved & ((fi != ei) | (fj != ej))
        ok &= ~(second & blocked(ei, ej))
        x = np.where(ok, nxp, x)
        y = np.where(ok, nyp, y)
    return np.stack([x - x0, y - y0], axis=1)
