"""O2q -- dense global-matrix brute force of the Q_p quadrilateral variant (N4).

TEST INFRASTRUCTURE ONLY (see oracle/oracle.py header).  Pins O1's quad path
(`orc_q_*` in dg_oracle.c) on grids of at most ~10x10 pixels.  Independent of
O1 in the same ways as oracle/dense.py: the tensor Lagrange basis comes from
inverting a monomial Vandermonde matrix on the nodes (a/p, b/p) (not from the
1-D product formula), volume and face integrals are exact monomial integrals
over the unit square and its edges (not Gauss quadrature), and the scheme is
a global assembly
    L = M^-1 sum_c B_c M^-1 G_c
(not an element loop).  Shared conventions: the readings R4-R7 (LDG form of
Eq. (7), central u-flux, harmonic q-flux, u+ = 0 from axons, SSP-RK3) and
REFLECT outer faces (R9); dof k = b (p+1) + a for the node (a/p, b/p).
"""
from __future__ import annotations

import numpy as np

# faces E W N S: (fixed variable, its value on K, neighbour offset, normal)
_FACES = [(0, 1.0, (1, 0), (1.0, 0.0)), (0, 0.0, (-1, 0), (-1.0, 0.0)),
          (1, 1.0, (0, 1), (0.0, 1.0)), (1, 0.0, (0, -1), (0.0, -1.0))]


def qdof(p):
    return (p + 1) ** 2


def _mons(p):
    return [(a, b) for b in range(p + 1) for a in range(p + 1)]


def coeffs(p):
    """C[m, k]: N_k = sum_m C[m, k] xi^a_m eta^b_m, from the nodal Vandermonde."""
    nodes = [(a / p, b / p) for b in range(p + 1) for a in range(p + 1)]
    V = np.array([[x ** a * y ** b for (a, b) in _mons(p)] for (x, y) in nodes])
    return np.linalg.inv(V)


def _int_sq(a, b):
    return 1.0 / ((a + 1) * (b + 1))


def local(p, h):
    """M, Dx, Dy (Dc[i][j] = int d_c N_i N_j), and per face (Em, Ep)."""
    C = coeffs(p)
    mons = _mons(p)
    d = qdof(p)
    M = np.zeros((d, d))
    D = np.zeros((2, d, d))
    for i in range(d):
        for j in range(d):
            for m1, (a1, b1) in enumerate(mons):
                for m2, (a2, b2) in enumerate(mons):
                    c = C[m1, i] * C[m2, j]
                    if c == 0.0:
                        continue
                    M[i, j] += c * _int_sq(a1 + a2, b1 + b2) * h * h
                    if a1 > 0:
                        D[0, i, j] += c * a1 * _int_sq(a1 - 1 + a2, b1 + b2) * h
                    if b1 > 0:
                        D[1, i, j] += c * b1 * _int_sq(a1 + a2, b1 - 1 + b2) * h
    faces = []
    for var, val, off, nrm in _FACES:
        Em = np.zeros((d, d))
        Ep = np.zeros((d, d))
        nval = val - (off[0] if var == 0 else off[1])      # the neighbour's local coordinate
        for i in range(d):
            for j in range(d):
                for m1, (a1, b1) in enumerate(mons):
                    for m2, (a2, b2) in enumerate(mons):
                        c = C[m1, i] * C[m2, j]
                        if c == 0.0:
                            continue
                        if var == 0:    # x fixed: integrate eta^(b1+b2) over [0,1]
                            Em[i, j] += c * val ** a1 * val ** a2 / (b1 + b2 + 1) * h
                            Ep[i, j] += c * val ** a1 * nval ** a2 / (b1 + b2 + 1) * h
                        else:
                            Em[i, j] += c * val ** b1 * val ** b2 / (a1 + a2 + 1) * h
                            Ep[i, j] += c * val ** b1 * nval ** b2 / (a1 + a2 + 1) * h
        faces.append((Em, Ep, off, nrm))
    return M, D, faces


def assemble(p, h, Dif, mask, outer_bc=0):
    """Dense L on the grid mask [ny][nx], dof order [j][i][k]; outer_bc 0 =
    REFLECT (outside = axon), 1 = ABSORB (Eq. (4): h_u = 0, h_q = k q- . n)."""
    ny, nx = mask.shape
    d = qdof(p)
    M, D, faces = local(p, h)
    Minv = np.linalg.inv(M)
    n = nx * ny * d
    G = [np.zeros((n, n)), np.zeros((n, n))]
    B = [np.zeros((n, n)), np.zeros((n, n))]
    k = np.where(mask == 0, Dif, 0.0)

    def blk(i, j):
        return slice((j * nx + i) * d, (j * nx + i + 1) * d)

    for j in range(ny):
        for i in range(nx):
            K = blk(i, j)
            for c in range(2):
                G[c][K, K] -= D[c]
                B[c][K, K] -= k[j, i] * D[c]
            for Em, Ep, (di, dj), nrm in faces:
                ii, jj = i + di, j + dj
                inside = 0 <= ii < nx and 0 <= jj < ny
                if not inside and outer_bc == 1:
                    for c in range(2):
                        B[c][K, K] += k[j, i] * nrm[c] * Em
                    continue
                for c in range(2):
                    G[c][K, K] += 0.5 * nrm[c] * Em
                    if inside:
                        G[c][K, blk(ii, jj)] += 0.5 * nrm[c] * Ep
                if inside:
                    kp = k[jj, ii]
                    kf = 0.0 if k[j, i] + kp == 0 else 2 * k[j, i] * kp / (k[j, i] + kp)
                    for c in range(2):
                        B[c][K, K] += 0.5 * kf * nrm[c] * Em
                        B[c][K, blk(ii, jj)] += 0.5 * kf * nrm[c] * Ep
    Mi = np.kron(np.eye(nx * ny), Minv)
    return Mi @ (B[0] @ Mi @ G[0] + B[1] @ Mi @ G[1])


def ssprk3(L, u, dt, nsteps):
    for _ in range(nsteps):
        U1 = u + dt * (L @ u)
        U2 = U1 + 0.75 * (u - U1) + 0.25 * dt * (L @ U1)
        u = U2 + (1 / 3) * (u - U2) + (2 / 3) * dt * (L @ U2)
    return u


def composite_blocks(p, code):
    """Blocks of L (units D/h^2) around the centre pixel of a 7x7 grid whose
    four face neighbours are open per `code` (bit0 E, bit1 W, bit2 N, bit3 S)
    and every other pixel open: dict offset -> (d x d) block."""
    d = qdof(p)
    mask = np.zeros((7, 7), np.uint8)
    for bit, (di, dj) in enumerate([(1, 0), (-1, 0), (0, 1), (0, -1)]):
        if not (code >> bit) & 1:
            mask[3 + dj, 3 + di] = 1
    L = assemble(p, 1.0, 1.0, mask)
    row = slice((3 * 7 + 3) * d, (3 * 7 + 4) * d)
    out = {}
    for dj in range(-3, 4):
        for di in range(-3, 4):
            col = slice(((3 + dj) * 7 + 3 + di) * d, ((3 + dj) * 7 + 4 + di) * d)
            out[(di, dj)] = L[row, col]
    return out
