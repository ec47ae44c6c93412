"""ctypes binding of O1 (oracle/dg_oracle.c) -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
--impl reference) may import this module.  It never imports the product
package, and the product package never imports it.

Every function follows PAPER.md (cited in dg_oracle.c); readings R1..R19 of
the paper's silent/garbled points are listed in DESIGN.md.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dg_oracle.c")
_LIB = os.path.join(_HERE, "libdgoracle.so")

REFLECT, ABSORB = 0, 1

_dp = ctypes.POINTER(ctypes.c_double)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_i32p = ctypes.POINTER(ctypes.c_int32)


def build(force: bool = False) -> str:
    """Compile the oracle (plain gcc -O2 -fopenmp)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        c_int, c_double, c_i64 = ctypes.c_int, ctypes.c_double, ctypes.c_int64
        L.orc_reference.argtypes = [c_int, c_double] + [_dp] * 7
        L.orc_basis.argtypes = [c_int, c_int, c_int, _dp, _dp]
        L.orc_apply_L.argtypes = [c_int, c_double, c_double, c_int, c_int, _u8p, c_int, _dp, _dp]
        L.orc_advance.argtypes = [c_int, c_double, c_double, c_int, c_int, _u8p, c_int, _dp, c_double, c_i64]
        L.orc_moments.argtypes = [c_int, c_double, c_int, c_int, _dp, c_int, c_int, _dp]
        L.orc_project_delta.argtypes = [c_int, c_double, c_int, c_int, c_int, c_int, _dp]
        L.orc_solve.argtypes = [c_int, c_double, c_double, c_int, c_int, _u8p, c_int, _i32p, c_i64,
                                c_double, c_i64, _dp, _dp, c_int]
        L.orc_sigma.argtypes = [_dp, c_i64, c_int, _dp, _dp]
        L.orc_q_reference.argtypes = [c_int, c_double] + [_dp] * 5
        L.orc_q_apply_L.argtypes = [c_int, c_double, c_double, c_int, c_int, _u8p, c_int, _dp, _dp]
        L.orc_q_solve.argtypes = [c_int, c_double, c_double, c_int, c_int, _u8p, c_int, _i32p, c_i64, c_double,
                                  c_i64, _dp, _dp, c_int]
        L.orc_q_solve_points.argtypes = [c_int, c_double, c_double, c_int, c_int, _u8p, _dp, c_i64, c_double,
                                         c_i64, _dp, _dp, c_int]
        L.orc_solve_points.argtypes = [c_int, c_double, c_double, c_int, c_int, _u8p, c_int, _dp, c_i64,
                                       c_double, c_i64, _dp, _dp, c_int]
        L.orc_mixture.argtypes = [c_int, c_int, c_int, _dp, _i32p, _dp, c_i64, c_int, _dp]
        L.orc_residual.argtypes = [_dp, c_int, c_double, _dp, _dp, _dp]
        L.orc_project_gaussian.argtypes = [c_int, c_double, c_int, c_int, c_double, c_double, c_double, _dp]
        L.orc_l2_err_gaussian.argtypes = [c_int, c_double, c_int, c_int, _dp, c_double, c_double, c_double, _dp]
        for f in (L.orc_reference, L.orc_basis, L.orc_apply_L, L.orc_advance, L.orc_moments,
                  L.orc_project_delta, L.orc_solve, L.orc_solve_points, L.orc_sigma, L.orc_q_reference,
                  L.orc_q_apply_L, L.orc_q_solve, L.orc_q_solve_points, L.orc_project_gaussian, L.orc_l2_err_gaussian, L.orc_mixture, L.orc_residual):
            f.restype = c_int
        _lib = L
    return _lib


def _p(a, t=_dp):
    return a.ctypes.data_as(t) if a is not None else None


def ndof(p: int) -> int:
    return (p + 1) * (p + 2) // 2


class OracleError(RuntimeError):
    def __init__(self, code, what):
        super().__init__(f"{what}: oracle status {code}")
        self.code = code


def _chk(rc, what):
    if rc != 0:
        raise OracleError(rc, what)


def reference(p: int, h: float = 1.0) -> dict:
    d = ndof(p)
    out = dict(M=np.zeros((2, d, d)), Minv=np.zeros((2, d, d)), Dc=np.zeros((2, 2, d, d)),
               Em=np.zeros((2, 3, d, d)), Ep=np.zeros((2, 3, d, d)), nrm=np.zeros((2, 3, 2)),
               nodes=np.zeros((2, d, 2)))
    _chk(lib().orc_reference(p, h, *[_p(out[k]) for k in ("M", "Minv", "Dc", "Em", "Ep", "nrm", "nodes")]),
         "orc_reference")
    return out


def basis(p: int, t: int, pts) -> np.ndarray:
    pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 2)
    out = np.zeros((pts.shape[0], ndof(p)))
    _chk(lib().orc_basis(p, t, pts.shape[0], _p(pts), _p(out)), "orc_basis")
    return out


def _mask(mask):
    return np.ascontiguousarray(mask, dtype=np.uint8)


def apply_L(p, h, D, mask, u, outer_bc=REFLECT) -> np.ndarray:
    mask = _mask(mask)
    ny, nx = mask.shape
    u = np.ascontiguousarray(u, dtype=np.float64).reshape(ny, nx, 2, ndof(p))
    out = np.zeros_like(u)
    _chk(lib().orc_apply_L(p, h, D, nx, ny, _p(mask, _u8p), outer_bc, _p(u), _p(out)), "orc_apply_L")
    return out


def advance(p, h, D, mask, u, dt, nsteps, outer_bc=REFLECT) -> np.ndarray:
    mask = _mask(mask)
    ny, nx = mask.shape
    u = np.array(u, dtype=np.float64).reshape(ny, nx, 2, ndof(p)).copy()
    _chk(lib().orc_advance(p, h, D, nx, ny, _p(mask, _u8p), outer_bc, _p(u), dt, nsteps), "orc_advance")
    return u


def moments(p, h, u, src) -> np.ndarray:
    u = np.ascontiguousarray(u, dtype=np.float64)
    ny, nx = u.shape[:2]
    m = np.zeros(6)
    _chk(lib().orc_moments(p, h, nx, ny, _p(u), int(src[0]), int(src[1]), _p(m)), "orc_moments")
    return m


def project_delta(p, h, nx, ny, src) -> np.ndarray:
    u = np.zeros((ny, nx, 2, ndof(p)))
    _chk(lib().orc_project_delta(p, h, nx, ny, int(src[0]), int(src[1]), _p(u)), "orc_project_delta")
    return u


def solve(p, h, D, mask, sources, dt, nsteps, outer_bc=REFLECT, keep_density=False, nthreads=0):
    """Per-source moments [n][6] (m00 m10 m01 m20 m11 m02), and optionally the
    final densities [n][ny][nx][2][d]."""
    mask = _mask(mask)
    ny, nx = mask.shape
    src = np.ascontiguousarray(sources, dtype=np.int32).reshape(-1, 2)
    n = src.shape[0]
    mom = np.zeros((n, 6))
    dens = np.zeros((n, ny, nx, 2, ndof(p))) if keep_density else None
    _chk(lib().orc_solve(p, h, D, nx, ny, _p(mask, _u8p), outer_bc, _p(src, _i32p), n, dt, nsteps,
                         _p(mom), _p(dens), nthreads), "orc_solve")
    return (mom, dens) if keep_density else mom


def solve_points(p, h, D, mask, points, dt, nsteps, outer_bc=REFLECT, keep_density=False, nthreads=0):
    """As solve(), for physical source points anywhere in extracellular pixels (N4)."""
    mask = _mask(mask)
    ny, nx = mask.shape
    pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 2)
    n = pts.shape[0]
    mom = np.zeros((n, 6))
    dens = np.zeros((n, ny, nx, 2, ndof(p))) if keep_density else None
    _chk(lib().orc_solve_points(p, h, D, nx, ny, _p(mask, _u8p), outer_bc, _p(pts), n, dt, nsteps,
                                _p(mom), _p(dens), nthreads), "orc_solve_points")
    return (mom, dens) if keep_density else mom


# ---- N4: quadrilateral Q_p elements (one per pixel), REFLECT --------------------
def qdof(p: int) -> int:
    return (p + 1) * (p + 1)


def q_reference(p, h=1.0) -> dict:
    d = qdof(p)
    out = dict(M=np.zeros((d, d)), Minv=np.zeros((d, d)), Dc=np.zeros((2, d, d)), Em=np.zeros((4, d, d)),
               Ep=np.zeros((4, d, d)))
    _chk(lib().orc_q_reference(p, h, *[_p(out[k]) for k in ("M", "Minv", "Dc", "Em", "Ep")]), "orc_q_reference")
    return out


def q_apply_L(p, h, D, mask, u, outer_bc=REFLECT) -> np.ndarray:
    mask = _mask(mask)
    ny, nx = mask.shape
    u = np.ascontiguousarray(u, dtype=np.float64).reshape(ny, nx, qdof(p))
    out = np.zeros_like(u)
    _chk(lib().orc_q_apply_L(p, h, D, nx, ny, _p(mask, _u8p), outer_bc, _p(u), _p(out)), "orc_q_apply_L")
    return out


def q_solve(p, h, D, mask, sources, dt, nsteps, keep_density=False, nthreads=0, outer_bc=REFLECT):
    mask = _mask(mask)
    ny, nx = mask.shape
    src = np.ascontiguousarray(sources, dtype=np.int32).reshape(-1, 2)
    n = src.shape[0]
    mom = np.zeros((n, 6))
    dens = np.zeros((n, ny, nx, qdof(p))) if keep_density else None
    _chk(lib().orc_q_solve(p, h, D, nx, ny, _p(mask, _u8p), outer_bc, _p(src, _i32p), n, dt, nsteps, _p(mom),
                           _p(dens), nthreads), "orc_q_solve")
    return (mom, dens) if keep_density else mom


def q_solve_points(p, h, D, mask, points, dt, nsteps, keep_density=False, nthreads=0):
    """Quads (N4) with physical point sources (reading R21)."""
    mask = _mask(mask)
    ny, nx = mask.shape
    pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 2)
    n = pts.shape[0]
    mom = np.zeros((n, 6))
    dens = np.zeros((n, ny, nx, qdof(p))) if keep_density else None
    _chk(lib().orc_q_solve_points(p, h, D, nx, ny, _p(mask, _u8p), _p(pts), n, dt, nsteps, _p(mom), _p(dens),
                                  nthreads), "orc_q_solve_points")
    return (mom, dens) if keep_density else mom


def sigma(mom, centering=0):
    mom = np.ascontiguousarray(mom, dtype=np.float64).reshape(-1, 6)
    s = np.zeros(4)
    mu = np.zeros(2)
    _chk(lib().orc_sigma(_p(mom), mom.shape[0], centering, _p(s), _p(mu)), "orc_sigma")
    return s.reshape(2, 2), mu


def project_gaussian(p, h, nx, ny, x0, y0, s2) -> np.ndarray:
    """L2 projection of exp(-|x-x0|^2/(2 s2))/(2 pi s2) onto V_h."""
    u = np.zeros((ny, nx, 2, ndof(p)))
    _chk(lib().orc_project_gaussian(p, h, nx, ny, x0, y0, s2, _p(u)), "orc_project_gaussian")
    return u


def l2_err_gaussian(p, h, u, x0, y0, s2) -> float:
    u = np.ascontiguousarray(u, dtype=np.float64)
    ny, nx = u.shape[:2]
    e = np.zeros(1)
    _chk(lib().orc_l2_err_gaussian(p, h, nx, ny, _p(u), x0, y0, s2, _p(e)), "orc_l2_err_gaussian")
    return float(e[0])


def mixture(p, dens, sources, mom, R) -> np.ndarray:
    """Mixture grid [(2R+1)][(2R+1)] of the centred, normalised densities."""
    dens = np.ascontiguousarray(dens, dtype=np.float64)
    n, ny, nx = dens.shape[:3]
    src = np.ascontiguousarray(sources, dtype=np.int32).reshape(-1, 2)
    mom = np.ascontiguousarray(mom, dtype=np.float64).reshape(-1, 6)
    g = np.zeros((2 * R + 1, 2 * R + 1))
    _chk(lib().orc_mixture(p, nx, ny, _p(dens), _p(src, _i32p), _p(mom), n, R, _p(g)), "orc_mixture")
    return g


def residual(grid, h, S, mu) -> float:
    """Eq. (9): sum over nodes of (N(x; mu, Sigma) - grid)^2."""
    grid = np.ascontiguousarray(grid, dtype=np.float64)
    R = (grid.shape[0] - 1) // 2
    S = np.ascontiguousarray(S, dtype=np.float64).reshape(4)
    mu = np.ascontiguousarray(mu, dtype=np.float64).reshape(2)
    r = np.zeros(1)
    _chk(lib().orc_residual(_p(grid), R, h, _p(S), _p(mu), _p(r)), "orc_residual")
    return float(r[0])
