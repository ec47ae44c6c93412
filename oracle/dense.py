"""O2 -- dense global-matrix brute force of the same DG scheme (numpy, fp64).

TEST INFRASTRUCTURE ONLY (see oracle/oracle.py header).  Used to pin O1 on
grids of at most ~12x12 pixels: the whole semi-discrete operator
    L = M^-1 sum_c B_c M^-1 G_c
is assembled as a dense matrix from Eq. (7) with the
fluxes of P:194-202, and stepped by matrix-vector products.

It is derived independently of O1: the Lagrange basis comes from inverting a
monomial Vandermonde matrix (not from barycentric formulas), volume integrals
are exact monomial integrals (not collapsed Gauss quadrature), and the scheme
is a global assembly (not an element loop).  The conventions it shares with O1
are the paper's readings listed in DESIGN.md: the mesh and diagonal (R1),
equispaced nodes in canonical order (R3), LDG reading of Eq. (7) (R4),
central/harmonic fluxes (R5), u+ = 0 from axon elements (R6), SSP-RK3 (R7),
REFLECT/ABSORB outer faces (R9).
"""
from __future__ import annotations

import itertools
from fractions import Fraction

import numpy as np

REFLECT, ABSORB = 0, 1

# triangle vertices in pixel-local coordinates (reading R1)
_VERT = {0: [(0, 0), (1, 0), (1, 1)],   # L = {eta < xi}
         1: [(0, 0), (1, 1), (0, 1)]}   # U = {eta > xi}
# faces: (start, end, outward normal, neighbour pixel offset); neighbour is the other type
_S2 = 1.0 / np.sqrt(2.0)
_FACES = {0: [((0, 0), (1, 0), (0.0, -1.0), (0, -1)),
              ((1, 0), (1, 1), (1.0, 0.0), (1, 0)),
              ((1, 1), (0, 0), (-_S2, _S2), (0, 0))],
          1: [((1, 1), (0, 1), (0.0, 1.0), (0, 1)),
              ((0, 1), (0, 0), (-1.0, 0.0), (-1, 0)),
              ((0, 0), (1, 1), (_S2, -_S2), (0, 0))]}


def ndof(p):
    return (p + 1) * (p + 2) // 2


def nodes(p, t):
    """Equispaced lattice, canonical order: vertices, edges v0v1, v1v2, v2v0, interior."""
    V = [np.array(v, dtype=float) for v in _VERT[t]]
    out = list(V)
    for a, b in ((0, 1), (1, 2), (2, 0)):
        for s in range(1, p):
            out.append(V[a] + (s / p) * (V[b] - V[a]))
    if p == 3:
        out.append((V[0] + V[1] + V[2]) / 3.0)
    return np.array(out)


def monomials(p):
    return [(a, b) for a in range(p + 1) for b in range(p + 1 - a)]


def coeffs(p, t):
    """C[m][j]: N_j = sum_m C[m][j] xi^a_m eta^b_m, from the Vandermonde inverse."""
    X = nodes(p, t)
    mons = monomials(p)
    V = np.array([[x ** a * y ** b for (a, b) in mons] for (x, y) in X])
    return np.linalg.inv(V)


def mono_int(t, a, b):
    """Exact int over the unit-pixel triangle of xi^a eta^b."""
    if t == 0:  # 0 < eta < xi < 1
        return 1.0 / ((b + 1) * (a + b + 2))
    return 1.0 / ((a + 1) * (a + b + 2))  # 0 < xi < eta < 1


def eval_basis(p, t, x, y):
    C = coeffs(p, t)
    m = np.array([x ** a * y ** b for (a, b) in monomials(p)])
    return m @ C


def ref_matrices(p, h):
    """M[t], Dc[t][c] (int d_c N_i N_j), Em[t][f], Ep[t][f] in physical units."""
    d = ndof(p)
    mons = monomials(p)
    M = np.zeros((2, d, d))
    Dc = np.zeros((2, 2, d, d))
    Em = np.zeros((2, 3, d, d))
    Ep = np.zeros((2, 3, d, d))
    gx, gw = np.polynomial.legendre.leggauss(p + 2)
    gx = 0.5 * (gx + 1.0)
    gw = 0.5 * gw
    for t in (0, 1):
        C = coeffs(p, t)
        # int N_i N_j = sum C[m,i] C[n,j] I(a_m+a_n, b_m+b_n)
        I2 = np.array([[mono_int(t, am + an, bm + bn) for (an, bn) in mons] for (am, bm) in mons])
        M[t] = h * h * C.T @ I2 @ C
        for c in (0, 1):
            # d_c of monomial m: coefficient times shifted monomial
            Id = np.zeros((len(mons), len(mons)))
            for i, (am, bm) in enumerate(mons):
                k = am if c == 0 else bm
                if k == 0:
                    continue
                da, db = (am - 1, bm) if c == 0 else (am, bm - 1)
                for j, (an, bn) in enumerate(mons):
                    Id[i, j] = k * mono_int(t, da + an, db + bn)
            Dc[t, c] = h * C.T @ Id @ C   # (1/h) * h^2
        for f, (A, B, n, off) in enumerate(_FACES[t]):
            A = np.array(A, float)
            B = np.array(B, float)
            length = h * np.linalg.norm(B - A)
            for s, w in zip(gx, gw):
                P = A + s * (B - A)
                pm = eval_basis(p, t, *P)
                pp = eval_basis(p, 1 - t, P[0] - off[0], P[1] - off[1])
                Em[t, f] += w * length * np.outer(pm, pm)
                Ep[t, f] += w * length * np.outer(pm, pp)
    return M, Dc, Em, Ep


def assemble(p, h, D, mask, outer_bc=REFLECT):
    """Dense L (N x N), N = ny*nx*2*d, dof order [j][i][t][k]."""
    mask = np.asarray(mask).astype(bool)
    ny, nx = mask.shape
    d = ndof(p)
    N = ny * nx * 2 * d
    M, Dc, Em, Ep = ref_matrices(p, h)
    Minv = np.linalg.inv(M)

    def sl(i, j, t):
        b = ((j * nx + i) * 2 + t) * d
        return slice(b, b + d)

    def inside(i, j):
        return 0 <= i < nx and 0 <= j < ny

    def k(i, j):
        return 0.0 if (not inside(i, j) or mask[j, i]) else D

    G = np.zeros((2, N, N))
    B = np.zeros((2, N, N))
    Mi = np.zeros((N, N))
    for j, i, t in itertools.product(range(ny), range(nx), (0, 1)):
        r = sl(i, j, t)
        Mi[r, r] = Minv[t]
        kT = k(i, j)
        for c in (0, 1):
            G[c, r, r] -= Dc[t, c]
            B[c, r, r] -= kT * Dc[t, c]
        for f, (_, _, n, off) in enumerate(_FACES[t]):
            ii, jj = i + off[0], j + off[1]
            if not inside(ii, jj):
                if outer_bc == ABSORB:
                    for c in (0, 1):
                        B[c, r, r] += kT * n[c] * Em[t, f]
                else:  # REFLECT: u+ = 0, k+ = 0
                    for c in (0, 1):
                        G[c, r, r] += 0.5 * n[c] * Em[t, f]
                continue
            rn = sl(ii, jj, 1 - t)
            kn = k(ii, jj)
            kf = 0.0 if kT + kn == 0 else 2 * kT * kn / (kT + kn)
            for c in (0, 1):
                G[c, r, r] += 0.5 * n[c] * Em[t, f]
                G[c, r, rn] += 0.5 * n[c] * Ep[t, f]
                B[c, r, r] += kf * 0.5 * n[c] * Em[t, f]
                B[c, r, rn] += kf * 0.5 * n[c] * Ep[t, f]
    L = Mi @ (B[0] @ Mi @ G[0] + B[1] @ Mi @ G[1])
    return L


def delta(p, h, nx, ny, src):
    """Dirac at the centre of pixel src, L2-projected, split 1/2-1/2."""
    d = ndof(p)
    M, _, _, _ = ref_matrices(p, h)
    u = np.zeros((ny, nx, 2, d))
    for t in (0, 1):
        u[src[1], src[0], t] = 0.5 * np.linalg.solve(M[t], eval_basis(p, t, 0.5, 0.5))
    return u


def ssprk3(L, u, dt, nsteps):
    u = u.reshape(-1).copy()
    for _ in range(nsteps):
        U1 = u + dt * (L @ u)
        U2 = U1 + 0.75 * (u - U1) + 0.25 * dt * (L @ U1)
        u = U2 + (1.0 / 3.0) * (u - U2) + (2.0 / 3.0) * dt * (L @ U2)
    return u


def moment_weights(p):
    """W[t][ab][j] = int_unit-triangle xi^a eta^b N_j, (a,b) in 00,10,01,20,11,02, exact."""
    ab = [(0, 0), (1, 0), (0, 1), (2, 0), (1, 1), (0, 2)]
    W = np.zeros((2, 6, ndof(p)))
    for t in (0, 1):
        C = coeffs(p, t)
        for q, (a, b) in enumerate(ab):
            W[t, q] = np.array([mono_int(t, a + am, b + bm) for (am, bm) in monomials(p)]) @ C
    return W


def moments(p, h, u, src):
    """Exact moments about the centre of pixel src."""
    ny, nx = u.shape[:2]
    W = moment_weights(p)
    m = np.zeros(6)
    for j in range(ny):
        for i in range(nx):
            X = i - src[0] - 0.5
            Y = j - src[1] - 0.5
            for t in (0, 1):
                P = W[t] @ u[j, i, t]
                m[0] += h ** 2 * P[0]
                m[1] += h ** 3 * (P[1] + X * P[0])
                m[2] += h ** 3 * (P[2] + Y * P[0])
                m[3] += h ** 4 * (P[3] + 2 * X * P[1] + X * X * P[0])
                m[4] += h ** 4 * (P[4] + X * P[2] + Y * P[1] + X * Y * P[0])
                m[5] += h ** 4 * (P[5] + 2 * Y * P[2] + Y * Y * P[0])
    return m


def composite_blocks(p, code):
    """Extract the 5-point composite blocks of L (units D/h^2) for a pixel whose
    4-bit open-face code is `code` (bit0 E, bit1 W, bit2 N, bit3 S), from a
    dense 5x5 assembly.  Returns dict offset -> (2d x 2d) block, and the max
    |entry| found outside the 5-point pattern."""
    d = ndof(p)
    mask = np.ones((5, 5), dtype=np.uint8)
    mask[2, 2] = 0
    for bit, (di, dj) in enumerate([(1, 0), (-1, 0), (0, 1), (0, -1)]):
        if code >> bit & 1:
            mask[2 + dj, 2 + di] = 0
    # open the corners too, so that only the 5-point structure can explain zeros
    for di, dj in ((1, 1), (1, -1), (-1, 1), (-1, -1)):
        mask[2 + dj, 2 + di] = 0
    L = assemble(p, 1.0, 1.0, mask)
    nx = 5

    def rows(i, j):
        b = (j * nx + i) * 2 * d
        return slice(b, b + 2 * d)

    blocks = {}
    stray = 0.0
    for dj in range(-2, 3):
        for di in range(-2, 3):
            blk = L[rows(2, 2), rows(2 + di, 2 + dj)]
            if (di, dj) in ((0, 0), (1, 0), (-1, 0), (0, 1), (0, -1)):
                blocks[(di, dj)] = blk
            else:
                stray = max(stray, np.abs(blk).max())
    return blocks, stray


def as_fraction(x, max_den=1 << 20):
    return Fraction(x).limit_denominator(max_den)
