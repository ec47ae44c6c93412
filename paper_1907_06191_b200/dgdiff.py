"""Thin ctypes binding of the C-ABI in include/dgdiff.h (argument marshalling
only: every step of the path runs in the CUDA kernels of libdgdiff.so).

The names mirror the C functions.  There is no fallback: if the in-tree
libdgdiff.so is missing or cannot load, importing the binding raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdgdiff.so")
# experiments only: the tuning build reads DGDIFF_* knobs from the environment
# (its stats report tuning_build = 1); the product library never does
if os.environ.get("DGDIFF_TUNING_LIB") == "1":
    LIB_PATH = os.path.join(_HERE, "libdgdiff_tuning.so")

OK, E_ARG, E_SOURCE, E_UNSTABLE, E_NONFINITE, E_STATE, E_DEGENERATE, E_CUDA, E_NCCL, E_NOMEM = range(10)
STATUS_NAMES = ["OK", "E_ARG", "E_SOURCE", "E_UNSTABLE", "E_NONFINITE", "E_STATE", "E_DEGENERATE",
                "E_CUDA", "E_NCCL", "E_NOMEM"]

EXPORTED = ["dgdiff_opts_default", "dgdiff_create", "dgdiff_solve_batch", "dgdiff_covariance",
            "dgdiff_source_moments", "dgdiff_get_density", "dgdiff_dt_max", "dgdiff_last_error",
            "dgdiff_destroy", "dgdiff_operator_table", "dgdiff_shard", "dgdiff_set_timing",
            "dgdiff_get_stats", "dgdiff_reset_stats", "dgdiff_mixture", "dgdiff_centre_weights",
            "dgdiff_absorb_table", "dgdiff_mc_covariance", "dgdiff_solve_batch_points", "dgdiff_quad_table",
            "dgdiff_covariance_table"]


class dgdiff_opts(ctypes.Structure):
    _fields_ = [("precision", ctypes.c_int32), ("outer_bc", ctypes.c_int32), ("centering", ctypes.c_int32),
                ("temporal_steps", ctypes.c_int32), ("device", ctypes.c_int32), ("rank", ctypes.c_int32),
                ("nranks", ctypes.c_int32), ("nccl_id", ctypes.c_void_p), ("keep_density", ctypes.c_int32),
                ("max_chunk", ctypes.c_int32), ("stream", ctypes.c_void_p), ("kernel", ctypes.c_int32),
                ("mixture_radius", ctypes.c_int32), ("windows", ctypes.c_int32),
                ("element", ctypes.c_int32), ("adjoint", ctypes.c_int32)]


class dgdiff_stats_t(ctypes.Structure):
    _fields_ = [("launches", ctypes.c_int64), ("stage_launches", ctypes.c_int64), ("stage_ms", ctypes.c_double),
                ("stage_bytes", ctypes.c_double), ("stage_flops", ctypes.c_double), ("n_active", ctypes.c_int64), ("chunk", ctypes.c_int64),
                ("h2d_bytes", ctypes.c_int64), ("d2h_bytes", ctypes.c_int64),
                ("env_overrides", ctypes.c_int64), ("tuning_build", ctypes.c_int64),
                ("dom_ms", ctypes.c_double), ("dom_bytes", ctypes.c_double), ("dom_launches", ctypes.c_int64)]


class DGDiffError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else status}: {msg}")
        self.status = status


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(the CUDA path has no fallback)")
    L = ctypes.CDLL(LIB_PATH)
    H = ctypes.c_void_p
    i32, i64, dbl = ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    dp = ctypes.POINTER(ctypes.c_double)
    L.dgdiff_opts_default.argtypes = [ctypes.POINTER(dgdiff_opts)]
    L.dgdiff_opts_default.restype = None
    L.dgdiff_create.argtypes = [ctypes.POINTER(H), ctypes.POINTER(ctypes.c_uint8), i32, i32, dbl, dbl, i32,
                                ctypes.POINTER(dgdiff_opts)]
    L.dgdiff_solve_batch.argtypes = [H, ctypes.POINTER(ctypes.c_int32), i64, dbl, i64]
    L.dgdiff_covariance.argtypes = [H, dbl, dp, dp]
    L.dgdiff_source_moments.argtypes = [H, dp]
    L.dgdiff_get_density.argtypes = [H, i64, dp]
    L.dgdiff_dt_max.argtypes = [i32, dbl, dbl]
    L.dgdiff_dt_max.restype = dbl
    L.dgdiff_last_error.argtypes = []
    L.dgdiff_last_error.restype = ctypes.c_char_p
    L.dgdiff_destroy.argtypes = [H]
    L.dgdiff_destroy.restype = None
    L.dgdiff_operator_table.argtypes = [i32, dp, dp, dp]
    L.dgdiff_shard.argtypes = [i64, i32, i32, ctypes.POINTER(i64), ctypes.POINTER(i64)]
    L.dgdiff_shard.restype = None
    L.dgdiff_set_timing.argtypes = [H, i32]
    L.dgdiff_get_stats.argtypes = [H, ctypes.POINTER(dgdiff_stats_t)]
    L.dgdiff_reset_stats.argtypes = [H]
    for name, args in (("dgdiff_mixture", [H, dp, dp]), ("dgdiff_centre_weights", [i32, dp]),
                       ("dgdiff_absorb_table", [i32, dp]), ("dgdiff_solve_batch_points", [H, dp, i64, dbl, i64]),
                       ("dgdiff_quad_table", [i32, dp]), ("dgdiff_covariance_table", [H, dp, i64, dp, dp]),
                       ("dgdiff_mc_covariance", [H, ctypes.POINTER(ctypes.c_int32), i64, i32, i64, dbl,
                                                 ctypes.c_uint32, dp, dp, dp, dp])):
        if hasattr(L, name):
            getattr(L, name).argtypes = args
            getattr(L, name).restype = ctypes.c_int
    for f in ("dgdiff_create", "dgdiff_solve_batch", "dgdiff_covariance", "dgdiff_source_moments",
              "dgdiff_get_density", "dgdiff_operator_table", "dgdiff_set_timing", "dgdiff_get_stats",
              "dgdiff_reset_stats"):
        getattr(L, f).restype = ctypes.c_int
    return L


lib = _load()


def _check(status):
    if status != OK:
        raise DGDiffError(status, lib.dgdiff_last_error().decode())


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def ndof(degree):
    return (degree + 1) * (degree + 2) // 2


# ---- C names ---------------------------------------------------------------
def dgdiff_opts_default(**overrides) -> dgdiff_opts:
    o = dgdiff_opts()
    lib.dgdiff_opts_default(ctypes.byref(o))
    for k, v in overrides.items():
        setattr(o, k, v)
    return o


def dgdiff_create(mask, h, D, degree, opts: dgdiff_opts | None = None):
    mask = np.ascontiguousarray(mask, dtype=np.uint8)
    ny, nx = mask.shape
    handle = ctypes.c_void_p()
    _check(lib.dgdiff_create(ctypes.byref(handle), mask.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), nx, ny,
                             float(h), float(D), int(degree), ctypes.byref(opts) if opts is not None else None))
    return handle


def dgdiff_solve_batch(handle, sources, dt, nsteps):
    src = np.ascontiguousarray(sources, dtype=np.int32).reshape(-1, 2)
    _check(lib.dgdiff_solve_batch(handle, src.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), src.shape[0],
                                  float(dt), int(nsteps)))


def dgdiff_quad_table(degree):
    """N4 Q_p composite blocks [28][(p+1)^2][(p+1)^2] (host K0)."""
    d = (degree + 1) ** 2
    out = np.zeros((28, d, d))
    _check(lib.dgdiff_quad_table(int(degree), _dp(out)))
    return out


def dgdiff_solve_batch_points(handle, points, dt, nsteps):
    """N4: point sources (x, y) in physical units anywhere in extracellular pixels."""
    pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 2)
    _check(lib.dgdiff_solve_batch_points(handle, _dp(pts), pts.shape[0], float(dt), int(nsteps)))


def dgdiff_covariance(handle, delta):
    s = np.zeros(4)
    mu = np.zeros(2)
    _check(lib.dgdiff_covariance(handle, float(delta), _dp(s), _dp(mu)))
    return s.reshape(2, 2), mu


def dgdiff_covariance_table(handle, mom):
    """K5 on a caller-provided [n][6] moment table (logical ranks: their sum)."""
    mom = np.ascontiguousarray(mom, dtype=np.float64).reshape(-1, 6)
    s = np.zeros(4)
    mu = np.zeros(2)
    _check(lib.dgdiff_covariance_table(handle, _dp(mom), mom.shape[0], _dp(s), _dp(mu)))
    return s.reshape(2, 2), mu


def dgdiff_source_moments(handle, n):
    out = np.zeros((n, 6))
    _check(lib.dgdiff_source_moments(handle, _dp(out)))
    return out


def dgdiff_get_density(handle, src, nx, ny, degree, element=0):
    """Canonical fp64 density: [ny][nx][2][d] (triangles) or [ny][nx][(p+1)^2] (quads)."""
    out = np.zeros((ny, nx, 2, ndof(degree)) if element == 0 else (ny, nx, (degree + 1) ** 2))
    _check(lib.dgdiff_get_density(handle, int(src), _dp(out)))
    return out


def dgdiff_dt_max(degree, h, D):
    return lib.dgdiff_dt_max(int(degree), float(h), float(D))


def dgdiff_destroy(handle):
    lib.dgdiff_destroy(handle)


def dgdiff_operator_table(degree):
    d = ndof(degree)
    A = np.zeros((16, 5, 2 * d, 2 * d))
    W = np.zeros((2, 6, d))
    init = np.zeros((2, d))
    _check(lib.dgdiff_operator_table(int(degree), _dp(A), _dp(W), _dp(init)))
    return A, W, init


def dgdiff_shard(n, rank, nranks):
    b, e = ctypes.c_int64(), ctypes.c_int64()
    lib.dgdiff_shard(int(n), int(rank), int(nranks), ctypes.byref(b), ctypes.byref(e))
    return b.value, e.value


def dgdiff_mixture(handle, R):
    grid = np.zeros((2 * R + 1, 2 * R + 1))
    res = np.zeros(1)
    _check(lib.dgdiff_mixture(handle, _dp(grid), _dp(res)))
    return grid, float(res[0])


def dgdiff_mc_covariance(handle, sources, walkers_per_source, nsteps, delta, seed=1, want_disp=False):
    src = np.ascontiguousarray(sources, dtype=np.int32).reshape(-1, 2)
    S = np.zeros(4)
    mu = np.zeros(2)
    se = np.zeros(3)
    disp = np.zeros((src.shape[0] * walkers_per_source, 2)) if want_disp else None
    _check(lib.dgdiff_mc_covariance(handle, src.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), src.shape[0],
                                    int(walkers_per_source), int(nsteps), float(delta), int(seed) & 0xFFFFFFFF,
                                    _dp(S), _dp(mu), _dp(se), _dp(disp) if disp is not None else None))
    return (S.reshape(2, 2), mu, se, disp) if want_disp else (S.reshape(2, 2), mu, se)


def dgdiff_absorb_table(degree):
    d2 = 2 * ndof(degree)
    A = np.zeros((16, 16, 5, d2, d2))
    _check(lib.dgdiff_absorb_table(int(degree), _dp(A)))
    return A


def dgdiff_centre_weights(degree):
    cw = np.zeros((2, ndof(degree)))
    _check(lib.dgdiff_centre_weights(int(degree), _dp(cw)))
    return cw


def dgdiff_set_timing(handle, enable):
    _check(lib.dgdiff_set_timing(handle, int(bool(enable))))


def dgdiff_get_stats(handle) -> dict:
    s = dgdiff_stats_t()
    _check(lib.dgdiff_get_stats(handle, ctypes.byref(s)))
    return {k: getattr(s, k) for k, _ in dgdiff_stats_t._fields_}


def dgdiff_reset_stats(handle):
    _check(lib.dgdiff_reset_stats(handle))


# ---- convenience wrapper -----------------------------------------------------
class Solver:
    """Owns one dgdiff handle: Solver(mask, h, D, degree, precision=64, ...)."""

    def __init__(self, mask, h=1.0, D=1.0, degree=1, **opts):
        self.mask = np.ascontiguousarray(mask, dtype=np.uint8)
        self.ny, self.nx = self.mask.shape
        self.h, self.D, self.degree = float(h), float(D), int(degree)
        self._id_buf = None
        nccl_id = opts.pop("nccl_id", None)
        o = dgdiff_opts_default(**opts)
        if nccl_id is not None:
            self._id_buf = ctypes.create_string_buffer(bytes(nccl_id), len(nccl_id))
            o.nccl_id = ctypes.cast(self._id_buf, ctypes.c_void_p)
        self.opts = o
        self.handle = dgdiff_create(self.mask, h, D, degree, o)
        self.n = 0

    def solve(self, sources, dt, nsteps):
        src = np.ascontiguousarray(sources, dtype=np.int32).reshape(-1, 2)
        dgdiff_solve_batch(self.handle, src, dt, nsteps)
        self.n = src.shape[0]
        self.delta = nsteps * dt

    def solve_points(self, points, dt, nsteps):
        pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 2)
        dgdiff_solve_batch_points(self.handle, pts, dt, nsteps)
        self.n = pts.shape[0]
        self.delta = nsteps * dt

    def covariance(self, delta=None):
        return dgdiff_covariance(self.handle, self.delta if delta is None else delta)

    def moments(self):
        return dgdiff_source_moments(self.handle, self.n)

    def covariance_table(self, mom):
        return dgdiff_covariance_table(self.handle, mom)

    def mixture(self):
        """(grid [(2R+1)][(2R+1)], Eq. (9) residual); needs mixture_radius=R."""
        return dgdiff_mixture(self.handle, self.opts.mixture_radius)

    def mc_covariance(self, sources, walkers_per_source, nsteps, delta, seed=1, want_disp=False):
        """Monte-Carlo cross-check of Sigma on this substrate."""
        return dgdiff_mc_covariance(self.handle, sources, walkers_per_source, nsteps, delta, seed, want_disp)

    def density(self, src):
        return dgdiff_get_density(self.handle, src, self.nx, self.ny, self.degree, self.opts.element)

    def stats(self):
        return dgdiff_get_stats(self.handle)

    def close(self):
        if self.handle:
            dgdiff_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
