"""G1 -- seeded synthetic inputs: Gamma-axon substrates and point sources.

This module holds none of the method's arithmetic (no DG, no moments): it is
the one module both the product path and the oracle tests draw inputs from.

Substrate (§2.2; "diameters computed from a Gamma
distribution"):
  - radii r ~ Gamma(shape, scale) clipped to [rmin, rmax] micrometres.  Default
    shape 11.27, scale 0.0446 um fit 0.150 / 1.141 um as the expected
    min / max of 1901 draws (reading R17);
  - random sequential adsorption, largest first, centres uniform in the square
    (disks may be clipped by the domain edge), non-overlapping;
  - rasterisation: pixel (i, j) is axon (mask = 1) iff its centre lies in a
    closed disk (reading R16);
  - disks are added until the rasterised axon fraction reaches the target
    (the a-priori disk count undershoots on small boxes).
Sources ("randomly and uniformly in Omega_e", "centered box of
side 20 um" = 40 % of the 50 um side): unmasked pixel centres drawn uniformly,
with replacement, from a centred box of ceil(0.4 n) pixels (reading R11).

RNG: numpy PCG64 (np.random.default_rng(seed)).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

GAMMA_SHAPE = 11.27
GAMMA_SCALE_UM = 0.0446
RMIN_UM = 0.150
RMAX_UM = 1.141
H_UM = 0.125          # the paper's resolution: 50 um / 400 pixels


@dataclass
class Substrate:
    mask: np.ndarray                 # uint8 [ny][nx], 1 = axon (k = 0)
    circles: np.ndarray              # float64 [n][3]: x, y, r in micrometres
    h_um: float = H_UM
    meta: dict = field(default_factory=dict)

    @property
    def fraction(self) -> float:
        return float(self.mask.mean())


def sample_radii(n, seed, shape=GAMMA_SHAPE, scale=GAMMA_SCALE_UM, rmin=RMIN_UM, rmax=RMAX_UM):
    if n < 0 or shape <= 0 or scale <= 0 or not (0 < rmin < rmax):
        raise ValueError("bad Gamma parameters")
    rng = np.random.default_rng(seed)
    return np.clip(rng.gamma(shape, scale, size=n), rmin, rmax)


def rasterise_disk(mask, h, cx, cy, r):
    """Set mask = 1 on pixels whose centre lies in the closed disk; returns the
    number of newly masked pixels."""
    ny, nx = mask.shape
    i0 = max(0, int(math.floor((cx - r) / h - 0.5)))
    i1 = min(nx - 1, int(math.ceil((cx + r) / h - 0.5)))
    j0 = max(0, int(math.floor((cy - r) / h - 0.5)))
    j1 = min(ny - 1, int(math.ceil((cy + r) / h - 0.5)))
    if i1 < i0 or j1 < j0:
        return 0
    xs = (np.arange(i0, i1 + 1) + 0.5) * h - cx
    ys = (np.arange(j0, j1 + 1) + 0.5) * h - cy
    inside = (xs[None, :] ** 2 + ys[:, None] ** 2) <= r * r
    sub = mask[j0:j1 + 1, i0:i1 + 1]
    new = int(np.count_nonzero(inside & (sub == 0)))
    sub[inside] = 1
    return new


_rsa = None


def _rsa_lib():
    """Build (gcc) and load the RSA helper csrc/rsa.c (input generation only)."""
    global _rsa
    if _rsa is None:
        import ctypes
        import os
        import subprocess
        here = os.path.dirname(os.path.abspath(__file__))
        src = os.path.join(here, "csrc", "rsa.c")
        so = os.path.join(here, "librsa.so")
        if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
            tmp = so + f".tmp{os.getpid()}"
            subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-o", tmp, src, "-lm"])
            os.replace(tmp, so)
        L = ctypes.CDLL(so)
        dp, i64p = ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)
        L.rsa_place.restype = ctypes.c_int64
        L.rsa_place.argtypes = [dp, ctypes.c_int64, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                ctypes.c_int, dp, ctypes.c_int64, i64p, ctypes.POINTER(ctypes.c_uint8),
                                ctypes.c_int, ctypes.c_int, ctypes.c_double, i64p, ctypes.c_int64, dp,
                                ctypes.c_int64, dp, ctypes.c_int64, i64p]
        _rsa = L
    return _rsa


def gen_substrate(nx, ny, target_fraction, seed, h_um=H_UM, shape=GAMMA_SHAPE, scale=GAMMA_SCALE_UM,
                  rmin=RMIN_UM, rmax=RMAX_UM, max_attempts=4096) -> Substrate:
    """RSA Gamma-disk substrate rasterised to an nx x ny pixel mask.

    First the a-priori count n_est = f A / (pi E[r^2]) is drawn and placed
    largest-first; while the rasterised fraction is below f, further batches of
    n_est/10 radii are drawn from the same Gamma stream and placed largest-first.
    A radius that finds no free spot in max_attempts uniform draws is skipped.
    Candidate centres are consecutive PCG64 uniform pairs.
    """
    import ctypes
    if nx < 1 or ny < 1 or not (0 <= target_fraction < 1):
        raise ValueError("bad substrate size / fraction")
    L = _rsa_lib()
    Lx, Ly = nx * h_um, ny * h_um
    mean_r2 = shape * scale * scale + (shape * scale) ** 2
    n_est = max(1, int(math.ceil(target_fraction * Lx * Ly / (math.pi * mean_r2))))
    rrng = np.random.default_rng(np.random.SeedSequence([seed, 0]))
    prng = np.random.default_rng(np.random.SeedSequence([seed, 1]))
    mask = np.zeros((ny, nx), dtype=np.uint8)
    target = int(math.ceil(target_fraction * nx * ny))
    masked = ctypes.c_int64(0)
    circles = np.zeros((0, 3))
    first = True
    drawn = 0
    dp = ctypes.POINTER(ctypes.c_double)
    while masked.value < target and drawn < 50 * n_est:
        nb = n_est if first else max(1, n_est // 10)
        first = False
        radii = np.ascontiguousarray(np.sort(np.clip(rrng.gamma(shape, scale, size=nb), rmin, rmax))[::-1])
        drawn += nb
        pos = 0
        while pos < nb and masked.value < target:
            uni = np.ascontiguousarray(prng.uniform(0.0, 1.0, size=(1 << 18, 2)))
            used, done = ctypes.c_int64(0), ctypes.c_int64(0)
            rest = np.ascontiguousarray(radii[pos:])
            out = np.zeros((rest.shape[0], 3))
            prev = np.ascontiguousarray(circles)
            k = L.rsa_place(rest.ctypes.data_as(dp), rest.shape[0], Lx, Ly, 2.0 * rmax, max_attempts,
                            uni.ctypes.data_as(dp), uni.shape[0], ctypes.byref(used),
                            mask.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), nx, ny, h_um,
                            ctypes.byref(masked), target, out.ctypes.data_as(dp), rest.shape[0],
                            prev.ctypes.data_as(dp), prev.shape[0], ctypes.byref(done))
            circles = np.concatenate([circles, out[:k]], axis=0)
            pos += max(1, done.value)
    return Substrate(mask=mask, circles=circles, h_um=h_um,
                     meta=dict(seed=seed, target_fraction=target_fraction, n_disks=len(circles),
                               fraction=float(mask.mean()), shape=shape, scale=scale))


def disk_substrate(n, cx, cy, r_px) -> np.ndarray:
    """Single disk in pixel units (config c1): centre (cx, cy), radius r_px."""
    c = np.arange(n) + 0.5
    X, Y = np.meshgrid(c, c)
    return (((X - cx) ** 2 + (Y - cy) ** 2) <= r_px * r_px).astype(np.uint8)


def sample_sources(mask, n, seed, box_frac=0.4) -> np.ndarray:
    """n pixel-centre sources [n][2] = (i, j), uniform over unmasked pixels of
    the centred box of side ceil(box_frac * size), with replacement."""
    ny, nx = mask.shape
    bx, by = int(math.ceil(box_frac * nx)), int(math.ceil(box_frac * ny))
    x0, y0 = (nx - bx) // 2, (ny - by) // 2
    sub = mask[y0:y0 + by, x0:x0 + bx]
    jj, ii = np.nonzero(sub == 0)
    if ii.size == 0:
        raise ValueError("no extracellular pixel in the source box")
    rng = np.random.default_rng(seed)
    pick = rng.integers(0, ii.size, size=n)
    return np.stack([ii[pick] + x0, jj[pick] + y0], axis=1).astype(np.int32)


def lattice_sources(lo, hi, step) -> np.ndarray:
    """Regular lattice of sources, i, j in range(lo, hi + 1, step) (config c2)."""
    v = np.arange(lo, hi + 1, step)
    J, I = np.meshgrid(v, v, indexing="ij")
    return np.stack([I.ravel(), J.ravel()], axis=1).astype(np.int32)


def save_substrate(path, sub: Substrate, k0=450.0):
    """SPEC S:93 text format: '# substrate side=<L> k0=<k0>', then 'x,y,r' lines."""
    ny, nx = sub.mask.shape
    with open(path, "w") as f:
        f.write(f"# substrate side={float(nx * sub.h_um)!r} k0={float(k0)!r}\n")
        for x, y, r in sub.circles:   # repr of a Python float round-trips exactly
            f.write(f"{float(x)!r},{float(y)!r},{float(r)!r}\n")


def load_circles(path):
    rows = []
    with open(path) as f:
        for ln, line in enumerate(f, 1):
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            parts = line.split(",")
            if len(parts) != 3:
                raise ValueError(f"{path}:{ln}: expected x,y,r")
            rows.append([float(v) for v in parts])
    return np.array(rows, dtype=np.float64).reshape(-1, 3)
