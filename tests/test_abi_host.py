"""CPU tests of the product library: it loads, exports every symbol that
include/dgdiff.h declares, its host precompute K0 (exact rational composite
stencil) matches the independently derived dense assembly O2, and it refuses
to run without a GPU (no CPU fallback)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def dg():
    from paper_1907_06191_b200 import build
    build.build_all()
    from paper_1907_06191_b200 import dgdiff
    return dgdiff


def declared_functions():
    txt = open(os.path.join(ROOT, "include", "dgdiff.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(dgdiff_[a-z_]+)\s*\(", txt)))


def test_every_declared_symbol_is_exported(dg):
    names = declared_functions()
    assert len(names) >= 14
    so = ctypes.CDLL(dg.LIB_PATH)
    for n in names:
        assert hasattr(so, n), n
    assert set(names) == set(dg.EXPORTED)


def test_library_is_sm100a(dg):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", dg.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("p", [1, 2, 3])
def test_operator_table_matches_dense_assembly(dg, p):
    """K0 (exact rationals, monomial Vandermonde, q eliminated on a 3x3 patch)
    == blocks of O2's dense operator, for all 16 open-face codes."""
    from oracle import dense as O2
    A, W, init = dg.dgdiff_operator_table(p)
    offs = [(0, 0), (1, 0), (-1, 0), (0, 1), (0, -1)]
    for code in range(16):
        blocks, stray = O2.composite_blocks(p, code)
        assert stray < 1e-11
        for o, off in enumerate(offs):
            used = o == 0 or (code >> (o - 1)) & 1
            ref = blocks[off] if used else np.zeros_like(blocks[off])
            # (O2's floating-point Vandermonde inverse loses ~1e-12 relative at P3)
            assert np.allclose(A[code, o], ref, atol=1e-11 * max(1.0, np.abs(ref).max())), (code, o)
    tol = 1e-15 if p <= 2 else 1e-12     # O2's P3 Vandermonde inverse: ~1e-13 rounding
    assert np.allclose(W, O2.moment_weights(p), atol=tol)
    assert np.allclose(init, O2.delta(p, 1.0, 1, 1, (0, 0))[0, 0], atol=1e-13 if p <= 2 else 1e-10)


def test_p1_table_is_survey_A11(dg):
    """SURVEY App. A.11 (independent implementation): P1 all-open blocks."""
    A, W, init = dg.dgdiff_operator_table(1)
    h = 0.5
    E = np.array([[-3 / 2, 0, 3 / 2, 2, -9 / 2, 5 / 2], [11 / 2, 0, 1 / 2, 0, 5 / 2, -5 / 2],
                  [-5 / 2, 0, -7 / 2, 7, 13 / 2, 9 / 2], [0, 0, 0, -7 / 2, 0, -5 / 2],
                  [0, 0, 0, 1 / 2, 0, 11 / 2], [0, 0, 0, 3 / 2, 0, -3 / 2]])
    S = np.array([[-7 / 2, 0, -5 / 2, 13 / 2, 7, 9 / 2], [1 / 2, 0, 11 / 2, 5 / 2, 0, -5 / 2],
                  [3 / 2, 0, -3 / 2, -9 / 2, 2, 5 / 2], [0, 0, 0, 0, 1 / 2, 11 / 2],
                  [0, 0, 0, 0, -7 / 2, -5 / 2], [0, 0, 0, 0, 3 / 2, -3 / 2]])
    assert np.array_equal(A[15, 1], E)
    assert np.array_equal(A[15, 4], S)
    assert np.count_nonzero(A[15, 0]) == 36
    assert [np.count_nonzero(A[15, o]) for o in range(1, 5)] == [20, 20, 20, 20]
    assert np.array_equal(init, np.array([[3, -3, 3], [3, 3, -3]], float))
    assert np.allclose(W[0, 1], [1 / 12, 1 / 8, 1 / 8]) and np.allclose(W[1, 5], [1 / 20, 1 / 10, 1 / 10])
    # row sums over the 5 blocks vanish for the all-open pixel
    assert np.abs(A[15].sum(axis=(0, 2))).max() == 0.0


@pytest.mark.parametrize("p", [1, 2])
def test_operator_table_exact_in_fp32(dg, p):
    """Every entry is dyadic with a short mantissa: fp32 holds it exactly (F4)."""
    A, _, _ = dg.dgdiff_operator_table(p)
    assert np.array_equal(A.astype(np.float32).astype(np.float64), A)
    frac = A * 2.0 ** 20
    assert np.array_equal(frac, np.round(frac))


def composite_apply(A, mask, u):
    """du/dt in units D/h^2 from the K0 table, pixel by pixel (test helper)."""
    ny, nx = mask.shape
    out = np.zeros_like(u)
    offs = [(1, 0), (-1, 0), (0, 1), (0, -1)]
    for j in range(ny):
        for i in range(nx):
            if mask[j, i]:
                continue
            nb = []
            code = 0
            for bit, (di, dj) in enumerate(offs):
                ii, jj = i + di, j + dj
                if 0 <= ii < nx and 0 <= jj < ny and not mask[jj, ii]:
                    code |= 1 << bit
                    nb.append((bit + 1, ii, jj))
            acc = A[code, 0] @ u[j, i].reshape(-1)
            for o, ii, jj in nb:
                acc += A[code, o] @ u[jj, ii].reshape(-1)
            out[j, i] = acc.reshape(u.shape[2:])
    return out


@pytest.mark.parametrize("p", [1, 2, 3])
def test_table_reproduces_oracle_operator(dg, p, orc):
    """On random masks (all 16 codes, outer walls), the K0 table applied pixel
    by pixel equals O1's element-loop L(u) scaled by h^2/D, and conserves
    mass exactly (sum of int N_j du_j = 0: no flux through walls)."""
    A, W, _ = dg.dgdiff_operator_table(p)
    rng = np.random.default_rng(40 + p)
    d = (p + 1) * (p + 2) // 2
    for _ in range(3):
        mask = (rng.random((9, 11)) < 0.4).astype(np.uint8)
        u = rng.standard_normal((9, 11, 2, d))
        u[mask.astype(bool)] = 0
        h, D = 0.5, 3.0
        ref = orc.apply_L(p, h, D, mask, u) * h * h / D
        got = composite_apply(A, mask, u)
        assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)
        w = np.concatenate([W[0, 0], W[1, 0]])
        mass_rate = np.einsum("k,jik->", w, got.reshape(9, 11, 2 * d))
        assert abs(mass_rate) < 1e-11 * np.abs(got).sum()


def composite_apply_absorb(A, Aabs, mask, u):
    """K0 tables applied pixel by pixel under ABSORB (test helper)."""
    ny, nx = mask.shape
    out = np.zeros_like(u)
    offs = [(1, 0), (-1, 0), (0, 1), (0, -1)]
    for j in range(ny):
        for i in range(nx):
            if mask[j, i]:
                continue
            code = outer = 0
            nb = []
            for bit, (di, dj) in enumerate(offs):
                ii, jj = i + di, j + dj
                if not (0 <= ii < nx and 0 <= jj < ny):
                    outer |= 1 << bit
                elif not mask[jj, ii]:
                    code |= 1 << bit
                    nb.append((bit + 1, ii, jj))
            B = A[code] if outer == 0 else Aabs[code, outer]
            acc = B[0] @ u[j, i].reshape(-1)
            for o, ii, jj in nb:
                acc += B[o] @ u[jj, ii].reshape(-1)
            out[j, i] = acc.reshape(u.shape[2:])
    return out


@pytest.mark.parametrize("p", [1, 2, 3])
def test_absorb_table_reproduces_oracle_operator(dg, p, orc):
    """ABSORB (Eq. (4)): K0's boundary-pixel blocks + the interior table equal
    O1's L(u) with outer_bc=1 on random masks touching every grid edge."""
    A, _, _ = dg.dgdiff_operator_table(p)
    Aabs = dg.dgdiff_absorb_table(p)
    rng = np.random.default_rng(60 + p)
    d = (p + 1) * (p + 2) // 2
    for _ in range(3):
        mask = (rng.random((9, 10)) < 0.3).astype(np.uint8)
        u = rng.standard_normal((9, 10, 2, d))
        u[mask.astype(bool)] = 0
        h, D = 0.7, 1.9
        ref = orc.apply_L(p, h, D, mask, u, outer_bc=1) * h * h / D
        got = composite_apply_absorb(A, Aabs, mask, u)
        assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)


def test_dt_max_and_shard(dg):
    assert abs(dg.dgdiff_dt_max(1, 1.0, 1.0) - 2.5127453 / 60) < 1e-15
    assert abs(dg.dgdiff_dt_max(1, 0.5, 2.0) - 2.5127453 / 60 * 0.125) < 1e-15
    assert abs(dg.dgdiff_dt_max(3, 1.0, 1.0) - 2.5127453 / 462.37) < 1e-15
    assert dg.dgdiff_dt_max(4, 1.0, 1.0) == 0.0
    # the P3 limit sits inside the stability interval of the assembled operator
    from oracle import dense as O2
    lam = np.linalg.eigvals(O2.assemble(3, 1.0, 1.0, np.zeros((8, 8), np.uint8)))
    assert np.abs(lam).max() * dg.dgdiff_dt_max(3, 1.0, 1.0) < 2.5127453
    n = 65537
    spans = [dg.dgdiff_shard(n, r, 8) for r in range(8)]
    assert spans[0][0] == 0 and spans[-1][1] == n
    assert all(spans[k][1] == spans[k + 1][0] for k in range(7))
    assert max(e - b for b, e in spans) - min(e - b for b, e in spans) <= 1


def test_no_cpu_fallback(dg):
    """Without a CUDA device the library refuses (E_CUDA), never computes."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(dg.DGDiffError) as e:
        dg.Solver(np.zeros((8, 8), np.uint8), 1.0, 1.0, 1)
    assert e.value.status == dg.E_CUDA


def test_argument_errors_are_reported(dg):
    with pytest.raises(dg.DGDiffError) as e:
        dg.dgdiff_create(np.zeros((4, 4), np.uint8), 1.0, 1.0, 4)
    assert e.value.status == dg.E_ARG
    # P3 (N4): ring kernel and REFLECT only
    for bad in (dict(kernel=1), dict(temporal_steps=2)):
        with pytest.raises(dg.DGDiffError) as e:
            dg.dgdiff_create(np.zeros((4, 4), np.uint8), 1.0, 1.0, 3, dg.dgdiff_opts_default(**bad))
        assert e.value.status == dg.E_ARG, bad
    with pytest.raises(dg.DGDiffError) as e:
        dg.dgdiff_create(np.zeros((4, 4), np.uint8), -1.0, 1.0, 1)
    assert e.value.status == dg.E_ARG
    with pytest.raises(dg.DGDiffError) as e:
        dg.dgdiff_create(np.zeros((4, 4), np.uint8), 1.0, 1.0, 1, dg.dgdiff_opts_default(outer_bc=2))
    assert e.value.status == dg.E_ARG
    # K3b is fp64 only; K3c (4) and K3d (5) need the ring kernel and REFLECT;
    # temporal_steps in 0..5; opts.kernel in 0..3
    for bad in (dict(temporal_steps=3, precision=32), dict(temporal_steps=4, kernel=1), dict(temporal_steps=6),
                dict(temporal_steps=4, outer_bc=1), dict(temporal_steps=4, windows=1),
                dict(temporal_steps=5, kernel=1), dict(temporal_steps=5, outer_bc=1), dict(temporal_steps=5, element=1),
                dict(kernel=4), dict(kernel=9), dict(kernel=-1)):
        with pytest.raises(dg.DGDiffError) as e:
            dg.dgdiff_create(np.zeros((4, 4), np.uint8), 1.0, 1.0, 1, dg.dgdiff_opts_default(**bad))
        assert e.value.status == dg.E_ARG, bad
    # adjoint moments: P1/P2 triangles, REFLECT, none of windows / temporal
    # blocking / mixture / densities; fp32 handles on the ring kernel only
    for bad in (dict(adjoint=2), dict(adjoint=1, precision=32, kernel=1), dict(adjoint=1, element=1, kernel=1),
                dict(adjoint=1, outer_bc=1), dict(adjoint=1, windows=1), dict(adjoint=1, temporal_steps=5),
                dict(adjoint=1, mixture_radius=3), dict(adjoint=1, keep_density=1), dict(adjoint=1, kernel=3)):
        with pytest.raises(dg.DGDiffError) as e:
            dg.dgdiff_create(np.zeros((4, 4), np.uint8), 1.0, 1.0, 1, dg.dgdiff_opts_default(**bad))
        assert e.value.status == dg.E_ARG, bad
    with pytest.raises(dg.DGDiffError) as e:
        dg.dgdiff_create(np.zeros((4, 4), np.uint8), 1.0, 1.0, 3, dg.dgdiff_opts_default(adjoint=1))
    assert e.value.status == dg.E_ARG
    # N1 windows: 0/1 only, and only on the ring kernel
    for bad in (dict(windows=3), dict(windows=1, kernel=1), dict(windows=2, temporal_steps=2)):
        with pytest.raises(dg.DGDiffError) as e:
            dg.dgdiff_create(np.zeros((4, 4), np.uint8), 1.0, 1.0, 1, dg.dgdiff_opts_default(**bad))
        assert e.value.status == dg.E_ARG, bad


@pytest.mark.parametrize("p", [1, 2])
def test_quad_table_matches_dense_assembly(dg, p):
    """N4 Q_p: K0's 9-point-cross blocks (exact rationals) == O2q's dense
    operator for all 16 codes; the face-neighbour block has exactly two
    variants (opposite face open / closed), the far block one; corners are 0."""
    from oracle import dense_quad as Q
    T = dg.dgdiff_quad_table(p)
    tol = 1e-12 * max(1.0, np.abs(T).max())
    offs = [(1, 0), (-1, 0), (0, 1), (0, -1)]
    opp = [1, 0, 3, 2]
    for code in range(16):
        B = Q.composite_blocks(p, code)
        assert np.abs(T[code] - B[(0, 0)]).max() <= tol, code
        for f, (di, dj) in enumerate(offs):
            if not (code >> f) & 1:
                continue       # a masked neighbour holds u = 0: its column is never used
            N = T[16 + f] if (code >> opp[f]) & 1 else T[20 + f]
            assert np.abs(N - B[(di, dj)]).max() <= tol, (code, f)
            assert np.abs(T[24 + f] - B[(2 * di, 2 * dj)]).max() <= tol, (code, f)
        for off in [(1, 1), (1, -1), (-1, 1), (-1, -1), (2, 1), (1, 2), (3, 0)]:
            assert np.abs(B[off]).max() <= 1e-13
    assert np.abs(T[16] - T[20]).max() > 1e-3       # the two variants really differ
