"""Pins of the CPU oracle O1 (oracle/dg_oracle.c) against things other than
itself: closed forms, invariants, exact symmetries, a dense brute-force
assembly derived independently (O2, oracle/dense.py), the paper's printed
values, and an independent implementation's numbers.

Each test names the plausible mistake it is there to catch.
"""
import json
import os

import numpy as np
import pytest

from oracle import dense as O2

GOLD = os.path.join(os.path.dirname(__file__), "golden")
RNG = np.random.default_rng(20190715)


def c1_mask():
    n = 32
    c = np.arange(n) + 0.5
    X, Y = np.meshgrid(c, c)
    return (((X - 16) ** 2 + (Y - 16) ** 2) <= 64).astype(np.uint8)


# ---------------------------------------------------------------- basis / matrices
@pytest.mark.parametrize("p", [1, 2, 3])
def test_basis_partition_of_unity_and_nodal(orc, p):
    """Eq. (8) Lagrange basis: sum_j N_j = 1 and N_i(x_j) = delta_ij (catches a
    wrong node order or a mis-typed barycentric formula)."""
    ref = orc.reference(p)
    for t in (0, 1):
        nodes = ref["nodes"][t]
        V = orc.basis(p, t, nodes)
        assert np.allclose(V, np.eye(orc.ndof(p)), atol=1e-14)
        pts = RNG.random((50, 2))
        pts = np.where((pts[:, 1] < pts[:, 0])[:, None] == (t == 0), pts, pts[:, ::-1])
        assert np.allclose(orc.basis(p, t, pts).sum(axis=1), 1.0, atol=1e-13)


def test_p1_mass_matrix_closed_form(orc):
    """P1 M_T = (h^2/24)[[2,1,1],[1,2,1],[1,1,2]] on a triangle of area h^2/2."""
    h = 0.3
    ref = orc.reference(1, h)
    M = h * h / 24 * np.array([[2, 1, 1], [1, 2, 1], [1, 1, 2]])
    for t in (0, 1):
        assert np.allclose(ref["M"][t], M, rtol=1e-14, atol=0)


@pytest.mark.parametrize("p,expect", [(1, [1 / 6] * 3), (2, [0, 0, 0, 1 / 6, 1 / 6, 1 / 6])])
def test_mass_weights(orc, p, expect):
    """int N_j = row sums of M (partition of unity): P1 h^2/6 each; P2 vertex 0,
    edge h^2/6 (textbook quadratic-triangle weights)."""
    h = 0.7
    ref = orc.reference(p, h)
    for t in (0, 1):
        assert np.allclose(ref["M"][t].sum(axis=1), h * h * np.array(expect), atol=1e-15)
        w, _ = np.linalg.eigh(ref["M"][t])
        assert w.min() > 0                        # SPD


@pytest.mark.parametrize("p", [1, 2, 3])
def test_reference_matrices_match_exact_integration(orc, p):
    """O1's Gauss-quadrature M, Dc, E-, E+ equal O2's exact monomial integrals
    (catches a too-low quadrature order, a missing 1/h in the gradient, a wrong
    face length or a wrong neighbour parametrisation)."""
    h = 0.25
    ref = orc.reference(p, h)
    M, Dc, Em, Ep = O2.ref_matrices(p, h)
    tol = 1e-13 if p < 3 else 1e-11
    assert np.allclose(ref["M"], M, atol=tol * h * h)
    assert np.allclose(ref["Dc"], Dc, atol=tol * h)
    assert np.allclose(ref["Em"], Em, atol=tol * h)
    assert np.allclose(ref["Ep"], Ep, atol=tol * h)


def test_normals_outward_unit(orc):
    ref = orc.reference(1)
    n = ref["nrm"]
    assert np.allclose(np.linalg.norm(n, axis=2), 1.0)
    # L: bottom, right, diagonal; U: top, left, diagonal
    assert np.allclose(n[0, 0], [0, -1]) and np.allclose(n[0, 1], [1, 0])
    assert np.allclose(n[1, 0], [0, 1]) and np.allclose(n[1, 1], [-1, 0])
    assert np.allclose(n[0, 2], -n[1, 2]) and np.allclose(n[0, 2], np.array([-1, 1]) / np.sqrt(2))


# ---------------------------------------------------------------- operator vs dense brute force
@pytest.mark.parametrize("p", [1, 2, 3])
@pytest.mark.parametrize("bc", [0, 1])
def test_apply_L_matches_dense_assembly(orc, p, bc):
    """O1 element loops == O2 global dense assembly on random <=8x8 masks
    (SPEC S:252 'oracle equivalence ... to 1e-12'); catches sign, index,
    transposed-operand and flux-weight mistakes anywhere in Eq. (7)."""
    rng = np.random.default_rng(p * 10 + bc)
    d = orc.ndof(p)
    for trial in range(3):
        ny, nx = rng.integers(4, 9, size=2)
        mask = (rng.random((ny, nx)) < 0.35).astype(np.uint8)
        u = rng.standard_normal((ny, nx, 2, d))
        u[mask.astype(bool)] = 0.0
        h, D = 0.5 + rng.random(), 0.5 + 2 * rng.random()
        ref = (O2.assemble(p, h, D, mask, bc) @ u.reshape(-1)).reshape(u.shape)
        got = orc.apply_L(p, h, D, mask, u, bc)
        tol = 1e-12 if p < 3 else 1e-11
        assert np.linalg.norm(got - ref) <= tol * np.linalg.norm(ref)


@pytest.mark.parametrize("p", [1, 2])
def test_ssprk3_steps_match_dense(orc, p):
    """Full scheme (Dirac data, SSP-RK3, moments) vs dense stepping."""
    rng = np.random.default_rng(7 + p)
    mask = (rng.random((8, 7)) < 0.3).astype(np.uint8)
    mask[4, 3] = 0
    dt = (1 / 32) if p == 1 else (1 / 128)
    mom, dens = orc.solve(p, 1.0, 1.0, mask, [(3, 4)], dt, 40, keep_density=True)
    u0 = O2.delta(p, 1.0, 7, 8, (3, 4))
    assert np.allclose(orc.project_delta(p, 1.0, 7, 8, (3, 4)), u0, atol=1e-13)
    u = O2.ssprk3(O2.assemble(p, 1.0, 1.0, mask), u0, dt, 40).reshape(dens[0].shape)
    assert np.linalg.norm(dens[0] - u) <= 1e-12 * np.linalg.norm(u)
    assert np.allclose(mom[0], O2.moments(p, 1.0, u, (3, 4)), rtol=1e-12, atol=1e-13)


def test_composite_operator_is_5_point(orc):
    """After eliminating q, a pixel couples only to its 4 face neighbours
    (SURVEY F3); the P1 all-open self block is the dyadic table of App. A.11."""
    blocks, stray = O2.composite_blocks(1, 15)
    assert stray == 0.0
    self_row0 = [-53 / 2, 1, -9 / 2, 9 / 2, 9 / 2, 9]
    assert np.allclose(blocks[(0, 0)][0], self_row0, atol=1e-13)
    # every row sums to zero across the 5 blocks (constants in the interior)
    tot = sum(blocks.values())
    assert np.abs(tot.sum(axis=1)).max() < 1e-12


# ---------------------------------------------------------------- invariants
def test_initial_data_closed_form(orc):
    """P1 split-delta coefficients are +3/h^2 at the two diagonal vertices and
    -3/h^2 at the right-angle vertex (1/2 M^-1 N(x_c), by hand)."""
    h = 0.5
    u = orc.project_delta(1, h, 3, 3, (1, 1))
    assert np.allclose(u[1, 1, 0], np.array([3, -3, 3]) / h ** 2, rtol=1e-14)
    assert np.allclose(u[1, 1, 1], np.array([3, 3, -3]) / h ** 2, rtol=1e-14)
    assert np.count_nonzero(u) == 6


@pytest.mark.parametrize("p,expect", [(1, [[1 / 20, 1 / 10], [1 / 10, 1 / 20]]), (2, [[0, 0], [0, 0]])])
def test_initial_sigma_closed_form(orc, p, expect):
    """Sigma(0) of the projected Dirac: P1 h^2[[1/20,1/10],[1/10,1/20]]; P2 0
    (P2 integrates quadratics exactly, so the projection keeps the Dirac's
    zero second moments).  Mass 1, mean at the source."""
    h = 0.5
    mask = np.zeros((5, 5), np.uint8)
    mom = orc.solve(p, h, 1.0, mask, [(2, 2)], 0.01, 0)
    S, mu = orc.sigma(mom)
    assert abs(mom[0, 0] - 1) < 1e-14
    assert np.allclose(mu, 0, atol=1e-15)
    assert np.allclose(S, h * h * np.array(expect), atol=1e-15)


def test_mass_conserved_and_axons_static(orc):
    """REFLECT: total mass exact (P:204 no flow through axon walls; F2) and
    masked dofs identically zero for all t."""
    rng = np.random.default_rng(3)
    mask = (rng.random((20, 20)) < 0.45).astype(np.uint8)
    free = np.argwhere(mask == 0)
    src = [tuple(free[k][::-1]) for k in (0, len(free) // 2, len(free) - 1)]
    mom, dens = orc.solve(1, 1.0, 1.0, mask, src, 1 / 32, 500, keep_density=True)
    assert np.abs(mom[:, 0] - 1).max() < 1e-12
    assert np.abs(dens[:, mask.astype(bool)]).max() == 0.0


def test_absorbing_boundary_loses_mass(orc):
    """Eq. (4) u = 0 on the outer square: mass leaves once the density reaches it."""
    mask = np.zeros((10, 10), np.uint8)
    m_ref = orc.solve(1, 1.0, 1.0, mask, [(5, 5)], 1 / 32, 300, outer_bc=0)
    m_abs = orc.solve(1, 1.0, 1.0, mask, [(5, 5)], 1 / 32, 300, outer_bc=1)
    assert abs(m_ref[0, 0] - 1) < 1e-12
    assert m_abs[0, 0] < 0.9


@pytest.mark.parametrize("h,D", [(1.0, 1.0), (0.5, 2.0)])
def test_free_space_sigma_p1_closed_form(orc, h, D):
    """P1 free space: Sigma(Delta) = 2 D Delta I + h^2 [[1/20,1/15],[1/15,1/20]]
    once the ~0.25 h^2/D transient has passed; sharpens the
    paper's Sigma = 2Tk I.  Catches a wrong D/h scaling, a
    missing flux half, a wrong RK weight."""
    dt = h * h / D / 32
    nsteps = 64
    delta = nsteps * dt
    n = 72
    mask = np.zeros((n, n), np.uint8)
    mom = orc.solve(1, h, D, mask, [(36, 36)], dt, nsteps)
    S, mu = orc.sigma(mom)
    expect = 2 * D * delta * np.eye(2) + h * h * np.array([[1 / 20, 1 / 15], [1 / 15, 1 / 20]])
    assert np.allclose(S, expect, rtol=1e-12, atol=1e-13 * expect[0, 0])
    assert np.allclose(mu, 0, atol=1e-13 * h)


def test_free_space_sigma_p2_closed_form(orc):
    """P2 free space: Sigma(Delta) = 2 D Delta I exactly, also fully discrete
    (the moment ODE is linear in t, which SSP-RK3 integrates exactly)."""
    h, D = 1.0, 1.0
    dt = 1 / 128
    nsteps = 256
    n = 104
    mask = np.zeros((n, n), np.uint8)
    mom = orc.solve(2, h, D, mask, [(52, 52)], dt, nsteps)
    S, _ = orc.sigma(mom)
    assert np.allclose(S, 2 * D * nsteps * dt * np.eye(2), rtol=0, atol=2e-12)


def test_free_space_sigma_p3_closed_form(orc):
    """P3 reproduces quadratics, so like P2 the projected Dirac has Sigma(0) = 0
    and free-space Sigma = 2 D Delta I (walls 32 sigma away: 5e-13).  Catches
    a P3 basis / quadrature / face-node error that P1/P2 pins cannot see."""
    m = np.zeros((64, 64), np.uint8)
    S, mu = orc.sigma(orc.solve(3, 1.0, 1.0, m, [(32, 32)], 1 / 256, 128))
    assert np.abs(S - 1.0 * np.eye(2)).max() <= 2e-12
    assert np.abs(mu).max() <= 1e-13


def test_paper_analytic_value(orc):
    """k = 450 um^2/s, T = 0.036 s gives 2Tk = 32.4.  The same
    physics in grid units (h = 0.125 um) on a smaller free grid: P2 gives
    exactly 2 D Delta, i.e. 32.4 um^2 at T = 0.036 s."""
    paper = json.load(open(os.path.join(GOLD, "paper_values.json")))["free_diffusion_analytic"]
    k, T = paper["k0_um2_per_s"], paper["T_s"]
    assert abs(2 * T * k - paper["sigma_diag"]) < 1e-12
    # physical units h = 0.125 um, D = 450 um^2/s, over T' = T/1024 so that a
    # small grid keeps the walls >= 25 sigma away (P2 tails):
    # Sigma' = 32.4/1024 um^2 exactly; dt chosen stable (D dt/h^2 <= 0.013).
    h, scale = 0.125, 1024
    nsteps = 128
    dt = (T / scale) / nsteps
    assert k * dt / h ** 2 < 0.013
    n = 80
    mom = orc.solve(2, h, k, np.zeros((n, n), np.uint8), [(40, 40)], dt, nsteps)
    S, _ = orc.sigma(mom)
    assert np.allclose(S * scale, np.diag([32.4, 32.4]), rtol=0, atol=1e-10)


# ---------------------------------------------------------------- symmetries (F8)
def _case(seed):
    rng = np.random.default_rng(seed)
    mask = (rng.random((18, 18)) < 0.4).astype(np.uint8)
    free = np.argwhere(mask[5:13, 5:13] == 0) + 5
    src = [(int(f[1]), int(f[0])) for f in free[:4]]
    return mask, src


def test_transpose_symmetry_exact(orc):
    """x <-> y swaps L and U of every pixel (the diagonal is its own mirror),
    so Sigma' = P Sigma P^T exactly (catches an x/y or L/U asymmetry)."""
    mask, src = _case(11)
    S, mu = orc.sigma(orc.solve(1, 1.0, 1.0, mask, src, 1 / 32, 96))
    St, mut = orc.sigma(orc.solve(1, 1.0, 1.0, mask.T.copy(), [(j, i) for i, j in src], 1 / 32, 96))
    assert np.allclose(St, S[::-1, ::-1], rtol=1e-13, atol=1e-14)
    assert np.allclose(mut, mu[::-1], atol=1e-14)


def test_rotation_180_symmetry_exact(orc):
    """180 degrees maps the mesh onto itself: Sigma' = Sigma, mu' = -mu."""
    mask, src = _case(12)
    n = mask.shape[0]
    S, mu = orc.sigma(orc.solve(1, 1.0, 1.0, mask, src, 1 / 32, 96))
    Sr, mur = orc.sigma(orc.solve(1, 1.0, 1.0, mask[::-1, ::-1].copy(),
                                  [(n - 1 - i, n - 1 - j) for i, j in src], 1 / 32, 96))
    assert np.allclose(Sr, S, rtol=1e-13, atol=1e-14)
    assert np.allclose(mur, -mu, atol=1e-14)


def _disks_mask(k, L=12.0):
    """Fixed disk geometry on [0, L]^2 rasterised at h = 1/k (pixel centre in
    a closed disk, reading R16)."""
    n = int(L * k)
    c = (np.arange(n) + 0.5) / k
    X, Y = np.meshgrid(c, c)
    m = np.zeros((n, n), np.uint8)
    for cx, cy, r in [(3.1, 3.4, 1.6), (8.7, 4.2, 2.1), (4.6, 8.9, 1.9), (9.3, 9.6, 1.4)]:
        m |= ((X - cx) ** 2 + (Y - cy) ** 2 <= r * r).astype(np.uint8)
    return m


def test_rotation_90_eigenvalues_converge(orc):
    """90 degrees maps the LL->UR diagonals onto LR->UL ones, so the mesh is not
    invariant and Sigma' = R Sigma R^T holds only to discretisation order
    (north star: '90-degree-rotation invariance of Sigma's eigenvalues on
    rotated substrates').  Free space: Sigma = 2 D Delta I + h^2[[1/20, 1/15],
    [1/15, 1/20]] does not depend on where the source sits, so it is invariant
    (to rounding).  Walled substrate at h = 1/2 and 1/4 (same disks, same
    physical time): the eigenvalue mismatch shrinks with h (catches an
    orientation-dependent flux or wall term that does not vanish)."""
    def eig(mask, src, k, nsteps):
        n = mask.shape[0]
        S, _ = orc.sigma(orc.solve(1, 1.0 / k, 1.0, mask, src, 1 / 32 / k ** 2, nsteps))
        Sr, _ = orc.sigma(orc.solve(1, 1.0 / k, 1.0, np.rot90(mask).copy(),
                                    [(j, n - 1 - i) for i, j in src], 1 / 32 / k ** 2, nsteps))
        return np.linalg.eigvalsh(S), np.linalg.eigvalsh(Sr)
    # free space (walls >= 15 sigma away): Sigma itself is unchanged
    free = np.zeros((64, 64), np.uint8)
    e, er = eig(free, [(32, 32), (30, 33)], 1, 48)
    assert np.allclose(e, er, rtol=1e-12, atol=0)
    # walled: convergence in h
    diffs = []
    for k in (2, 4):
        m = _disks_mask(k)
        pts = [(6.1, 6.3), (5.9, 2.2), (2.6, 6.4)]          # physical source points (extracellular)
        src = [(int(x * k), int(y * k)) for x, y in pts]
        assert all(m[j, i] == 0 for i, j in src)
        e, er = eig(m, src, k, 32 * k * k)                   # physical time 1.0
        diffs.append(np.abs(e - er).max() / e.max())
    assert diffs[1] < 0.75 * diffs[0], diffs
    assert diffs[1] < 0.02, diffs


def test_sigma_symmetric_psd_and_hindered(orc):
    """Sigma stored symmetric; eigenvalues > 0; walls hinder: Sigma_ii < 2 D Delta
    (the paper's case study 19.50 < 32.4)."""
    mask, src = _case(13)
    S, _ = orc.sigma(orc.solve(1, 1.0, 1.0, mask, src, 1 / 32, 96))
    assert S[0, 1] == S[1, 0]
    assert np.linalg.eigvalsh(S).min() > 0
    assert S[0, 0] < 2 * 3.0 and S[1, 1] < 2 * 3.0


# ---------------------------------------------------------------- stability (F5)
def test_spectral_radius_and_rk3_stability(orc):
    """rho(L) <= 60 D/h^2 (P1 Bloch bound): SSP-RK3 is stable at
    0.98 dt_max and blows up at 1.05 dt_max on a free grid."""
    L = O2.assemble(1, 1.0, 1.0, np.zeros((10, 10), np.uint8))
    lam = np.linalg.eigvals(L)
    assert np.abs(lam).max() <= 60.0 + 1e-9
    assert lam.real.max() < 1e-10
    rho = 60.0
    dtmax = 2.5127453 / rho
    rng = np.random.default_rng(5)
    mask = np.zeros((24, 24), np.uint8)
    u0 = rng.standard_normal((24, 24, 2, 3))
    ok = orc.advance(1, 1.0, 1.0, mask, u0, 0.98 * dtmax, 300)
    bad = orc.advance(1, 1.0, 1.0, mask, u0, 1.05 * dtmax, 300)
    assert np.linalg.norm(ok) <= np.linalg.norm(u0)
    assert np.linalg.norm(bad) > 1e6 * np.linalg.norm(u0)


# ---------------------------------------------------------------- independent implementation
def test_config1_matches_independent_implementation(orc):
    """SURVEY App. A.10 (independent scratch implementation) config-1 values."""
    g = json.load(open(os.path.join(GOLD, "c1_independent_A10.json")))
    tol = g["tolerance_rel"]
    mask = c1_mask()
    assert mask.sum() == 208
    m1 = orc.solve(1, 1.0, 1.0, mask, [(4, 16)], 1 / 32, 1)[0]
    assert np.allclose(m1[[0, 3, 4, 5]], np.array(g["reflect_1"]["m"])[[0, 3, 4, 5]], rtol=tol)
    mom, dens = orc.solve(1, 1.0, 1.0, mask, [(4, 16)], 1 / 32, 200, keep_density=True)
    r = g["reflect_200"]
    assert np.allclose(mom[0], r["m"], rtol=tol, atol=tol)
    S, _ = orc.sigma(mom)
    assert np.allclose([S[0, 0], S[0, 1], S[1, 1]], r["sigma"], rtol=tol)
    assert abs(np.linalg.norm(dens) - r["l2_norm"]) <= 1e-12 * r["l2_norm"]
    assert np.abs(dens[0][mask.astype(bool)]).max() == 0.0
    ma = orc.solve(1, 1.0, 1.0, mask, [(4, 16)], 1 / 32, 200, outer_bc=1)
    a = g["absorb_200"]
    assert abs(ma[0, 0] - a["m00"]) <= tol
    Sa, _ = orc.sigma(ma)
    assert np.allclose([Sa[0, 0], Sa[0, 1], Sa[1, 1]], a["sigma"], rtol=tol)


def test_errors(orc):
    from oracle.oracle import OracleError
    mask = c1_mask()
    with pytest.raises(OracleError) as e:
        orc.solve(1, 1.0, 1.0, mask, [(16, 16)], 1 / 32, 1)     # source inside the axon
    assert e.value.code == 2
    with pytest.raises(OracleError):
        orc.solve(1, 1.0, 1.0, mask, [(40, 1)], 1 / 32, 1)      # out of grid
    with pytest.raises(OracleError) as e:
        orc.sigma(np.array([[0.0, 0, 0, 1, 0, 1]]))             # m00 <= 0
    assert e.value.code == 6


def test_own_mean_centering_gaussian_mixture_closed_form(orc):
    """centering=1 (reading R12): each density is shifted by its OWN
    mean, so Sigma is the mean of the per-source covariances; centering=0
    adds the spread of the per-source means (law of total covariance).
    Pinned on moment rows of Gaussians built from the textbook moments of
    N(m_s, C_s) scaled by a mass c_s (m00 = c, m10 = c m_x, m20 = c (C_xx +
    m_x^2), m11 = c (C_xy + m_x m_y), ...): the expected values are mean C_s
    and mean C_s + Cov(m_s), not a re-typed orc_sigma.  A dropped
    normalisation (c != 1), a sign slip in the own-mean subtraction or a
    leftover mixture mean term fails here."""
    rng = np.random.default_rng(7)
    n = 9
    c = rng.uniform(0.5, 2.0, n)
    mm = rng.normal(0.0, 1.5, (n, 2))
    C = []
    for _ in range(n):
        a = rng.normal(size=(2, 2))
        C.append(a @ a.T + 0.3 * np.eye(2))
    C = np.array(C)
    mom = np.stack([c, c * mm[:, 0], c * mm[:, 1], c * (C[:, 0, 0] + mm[:, 0] ** 2),
                    c * (C[:, 0, 1] + mm[:, 0] * mm[:, 1]), c * (C[:, 1, 1] + mm[:, 1] ** 2)], 1)
    S1, mu1 = orc.sigma(mom, centering=1)
    assert np.allclose(S1, C.mean(0), rtol=1e-13, atol=1e-14)
    assert np.allclose(mu1, 0)
    S0, mu0 = orc.sigma(mom, centering=0)
    spread = np.cov(mm.T, bias=True)                   # population covariance of the means
    assert np.allclose(S0, C.mean(0) + spread, rtol=1e-13, atol=1e-14)
    assert np.allclose(mu0, mm.mean(0), rtol=1e-13, atol=1e-14)


def test_own_mean_centering_invariant_under_reference_shift(orc):
    """The own-mean covariance of a density does not depend on the point its
    moments are taken about, so orc_sigma(centering=1) is unchanged when each
    source's moments are re-taken about a different pixel (a different shift
    per source) and each density is rescaled -- while the source-point
    reading (centering=0) changes.  Walled substrate, real DG densities."""
    mask, src = _case(14)
    mom, dens = orc.solve(1, 1.0, 1.0, mask, src, 1 / 32, 64, keep_density=True)
    rng = np.random.default_rng(3)
    shifted = []
    for k, (i, j) in enumerate(src):
        di, dj = rng.integers(-4, 5, 2)
        scale = rng.uniform(0.5, 3.0)
        shifted.append(orc.moments(1, 1.0, dens[k] * scale, (int(i + di), int(j + dj))))
    shifted = np.array(shifted)
    assert np.allclose(orc.moments(1, 1.0, dens[0], src[0]), mom[0], rtol=0, atol=1e-13)
    S1, _ = orc.sigma(mom, centering=1)
    S1s, _ = orc.sigma(shifted, centering=1)
    assert np.abs(S1s - S1).max() <= 1e-11 * S1.max()
    S0, _ = orc.sigma(mom, centering=0)
    S0s, _ = orc.sigma(shifted, centering=0)
    assert np.abs(S0s - S0).max() > 1e-2 * S0.max()
    # on walls the two readings differ (a few %)
    assert np.abs(S1 - S0).max() > 1e-3 * S0.max()


def test_own_mean_centering_free_space_p2_off_centre(orc):
    """Free space, P2, sources at arbitrary sub-pixel points: every density
    keeps its mean at the point and reproduces quadratics, so the own-mean
    Sigma is 2 D Delta I exactly for any mix of points."""
    m = np.zeros((76, 76), np.uint8)
    pts = [(37.31, 37.77), (38.9, 36.2), (36.05, 38.61)]
    mom = orc.solve_points(2, 1.0, 1.0, m, pts, 1 / 128, 128)
    S1, mu1 = orc.sigma(mom, centering=1)
    assert np.abs(S1 - 2.0 * np.eye(2)).max() <= 1e-12
    assert np.abs(mu1).max() == 0.0


@pytest.mark.parametrize("p,ns,dtf,lo_,hi_", [(1, (24, 48, 96), 64, 1.8, 2.3), (2, (16, 32), 128, 2.6, 3.5)])
def test_convergence_order_smooth_gaussian(orc, p, ns, dtf, lo_, hi_):
    """Textbook convergence: free diffusion of a smooth Gaussian (variance
    s2 -> s2 + 2 D t) in a box whose walls are > 6 sigma away; the L2 error
    of the fully discrete solution (dt = h^2/dtf, SSP-RK3 error O(h^6)) falls
    like h^(p+1) (measured 1.97 for P1, 3.04 for P2).  Catches any
    consistency error (a wrong flux weight or sign leaves the scheme
    conservative but drops the order)."""
    L, D, T, s2 = 8.0, 1.0, 0.0625, 0.25
    errs = []
    for n in ns:
        h = L / n
        dt = h * h / dtf
        nsteps = int(round(T / dt))
        dt = T / nsteps
        u0 = orc.project_gaussian(p, h, n, n, L / 2, L / 2, s2)
        u = orc.advance(p, h, D, np.zeros((n, n), np.uint8), u0, dt, nsteps)
        errs.append(orc.l2_err_gaussian(p, h, u, L / 2, L / 2, s2 + 2 * D * T))
    orders = [np.log2(errs[k] / errs[k + 1]) for k in range(len(errs) - 1)]
    assert all(lo_ <= o <= hi_ for o in orders), (errs, orders)


# ---------------------------------------------------------------- mixture + Eq. (9) residual (N2)
def test_mixture_dirac_node_value(orc):
    """At t = 0 the P1 projected Dirac is +-3/h^2 on the source pixel; its
    centre value (mean of the L and U traces at the diagonal midpoint) is
    (3 + 3)/2 = 3/h^2 (R20), and every other node is 0."""
    h = 0.5
    mom, dens = orc.solve(1, h, 1.0, np.zeros((9, 9), np.uint8), [(4, 4)], 0.01, 0, keep_density=True)
    g = orc.mixture(1, dens, [(4, 4)], mom, 3)
    assert abs(g[3, 3] - 3 / h ** 2) <= 1e-14 * 12
    g[3, 3] = 0
    assert np.abs(g).max() == 0.0


def test_mixture_free_space_is_gaussian(orc):
    """Free space, P2 (Sigma = 2 D Delta I exactly): the mixture nodes integrate
    to 1 and carry the second moment 2 D Delta by the midpoint rule (O(h^2/sigma^2)),
    and the Eq. (9) residual is small against sum N^2.  (P2 tails reach ~23
    sigma, so sources at different wall distances agree only to
    ~1e-6 here; exact translation invariance is pinned with P1 below.)"""
    n = 72
    mask = np.zeros((n, n), np.uint8)
    src = [(36, 36), (34, 37), (38, 35)]
    mom, dens = orc.solve(2, 1.0, 1.0, mask, src, 1 / 128, 512, keep_density=True)   # Delta = 4, sigma = 2.8
    R = 20
    g = orc.mixture(2, dens, src, mom, R)
    g1 = orc.mixture(2, dens[:1], src[:1], mom[:1], R)
    assert np.abs(g - g1).max() <= 1e-5 * g1.max()
    assert abs(g.sum() - 1.0) < 2e-3
    x = np.arange(-R, R + 1)
    assert abs((g.sum(axis=0) * x ** 2).sum() - 8.0) < 0.02 * 8.0   # midpoint rule on node values, O(h^2/sigma^2)
    S, mu = orc.sigma(mom)
    res = orc.residual(g, 1.0, S, mu)
    X, Y = np.meshgrid(x, x)
    gauss = np.exp(-(X ** 2 + Y ** 2) / 16.0) / (2 * np.pi * 8.0)
    assert res < 1e-3 * (gauss ** 2).sum()
    # Eq. (9) itself: the fitted Gaussian sampled at the nodes has zero residual
    Si = np.linalg.inv(S)
    dX, dY = X - mu[0], Y - mu[1]
    fit = np.exp(-0.5 * (Si[0, 0] * dX ** 2 + 2 * Si[0, 1] * dX * dY + Si[1, 1] * dY ** 2)) / (
        2 * np.pi * np.sqrt(np.linalg.det(S)))
    assert orc.residual(fit, 1.0, S, mu) < 1e-28


def test_mixture_translation_invariance_p1(orc):
    """P1, Delta = 2 (sigma = 2), walls > 15 sigma away: the mixture of shifted
    sources equals the single-source grid to rounding (catches a source/offset
    index mix-up in the centring)."""
    n = 80
    mask = np.zeros((n, n), np.uint8)
    src = [(40, 40), (37, 43), (44, 38)]
    mom, dens = orc.solve(1, 1.0, 1.0, mask, src, 1 / 32, 64, keep_density=True)
    g = orc.mixture(1, dens, src, mom, 10)
    g1 = orc.mixture(1, dens[:1], src[:1], mom[:1], 10)
    assert np.abs(g - g1).max() <= 1e-12 * g1.max()


# ---------------------------------------------------------------- N4 sub-pixel point sources
def test_points_reduce_to_pixel_centres(orc):
    """A point at a pixel centre is the pixel source of P:241 (bitwise)."""
    mask, src = _case(31)
    pts = [(i + 0.5, j + 0.5) for i, j in src]
    assert np.array_equal(orc.solve_points(1, 1.0, 1.0, mask, pts, 1 / 32, 20), orc.solve(1, 1.0, 1.0, mask, src, 1 / 32, 20))


@pytest.mark.parametrize("p", [1, 2, 3])
def test_point_projection_moments_exact(orc, p):
    """The L2 projection onto P_p reproduces every moment of degree <= p:
    mass 1 and first moments 0 about the point for any p, and (p >= 2) the
    second moments 0 too.  Points inside L, inside U, on the diagonal and on
    the pixel's lower-left edges (R21).  Catches a wrong triangle choice, a
    basis evaluated at the wrong local point, or moments about the pixel
    centre instead of the point."""
    m = np.zeros((6, 6), np.uint8)
    h = 0.7
    pts = [(2.71 * h, 3.22 * h), (2.23 * h, 3.64 * h), (2.4 * h, 3.4 * h), (2.0 * h, 3.3 * h), (2.6 * h, 3.0 * h)]
    mom = orc.solve_points(p, h, 1.0, m, pts, 1e-3, 0)
    assert np.allclose(mom[:, 0], 1.0, rtol=0, atol=1e-13)
    assert np.abs(mom[:, 1:3]).max() <= 1e-13
    if p >= 2:
        assert np.abs(mom[:, 3:]).max() <= 1e-13
    else:
        assert np.abs(mom[:, 3:]).max() > 1e-4          # P1 cannot hold x^2: a real test above


def test_point_free_space_p2_closed_form_and_translation(orc):
    """Free space, P2: Sigma = 2 D Delta I for a source anywhere in a pixel
    (the closed form does not depend on where the Dirac sits), and a shift by
    one whole pixel leaves every moment unchanged (the mesh is translation
    invariant by whole pixels)."""
    m = np.zeros((76, 76), np.uint8)                      # walls >= 25 sigma away
    pts = [(37.31, 37.77), (38.31, 37.77)]
    mom = orc.solve_points(2, 1.0, 1.0, m, pts, 1 / 128, 128)
    S, _ = orc.sigma(mom[:1])
    assert np.abs(S - 2.0 * np.eye(2)).max() <= 1e-12
    assert np.allclose(mom[0], mom[1], rtol=0, atol=1e-12)


# ---------------------------------------------------------------- N4 quadrilateral Q_p elements
def test_quad_q1_mass_matrix_closed_form(orc):
    """Q1 mass matrix = (h^2/36) [[4,2,2,1],[2,4,1,2],[2,1,4,2],[1,2,2,4]] (nodes
    (0,0),(1,0),(0,1),(1,1)); catches a wrong node order or quadrature."""
    h = 0.6
    R = orc.q_reference(1, h)
    ref = h * h / 36 * np.array([[4, 2, 2, 1], [2, 4, 1, 2], [2, 1, 4, 2], [1, 2, 2, 4]])
    assert np.allclose(R["M"], ref, rtol=0, atol=1e-15)


@pytest.mark.parametrize("p", [1, 2, 3])
def test_quad_apply_L_and_steps_match_dense(orc, p):
    """O1's element-loop Q_p operator == O2q's dense global assembly (Vandermonde
    basis, exact integrals) on random walled masks, and SSP-RK3 steps agree;
    masked rows are exactly zero and 1^T M L u = 0 (no flux through walls)."""
    from oracle import dense_quad as Q
    rng = np.random.default_rng(70 + p)
    d = (p + 1) ** 2
    for _ in range(2):
        mask = (rng.random((6, 7)) < 0.35).astype(np.uint8)
        u = rng.standard_normal((6, 7, d))
        u[mask.astype(bool)] = 0
        h, D = 0.7, 1.3
        L = Q.assemble(p, h, D, mask)
        ref = (L @ u.reshape(-1)).reshape(u.shape)
        got = orc.q_apply_L(p, h, D, mask, u)
        tol = 1e-12 if p <= 2 else 1e-9          # O2q's Q3 monomial Vandermonde: cond ~1e5
        assert np.linalg.norm(got - ref) <= tol * np.linalg.norm(ref)
        assert np.abs(got[mask.astype(bool)]).max() == 0.0
        M, _, _ = Q.local(p, h)
        assert abs(np.einsum("ij,yxj->", M, got)) <= 1e-12 * np.abs(got).sum()
    dt = 1e-3
    steps = Q.ssprk3(L, u.reshape(-1), dt, 5).reshape(u.shape)
    src_free = np.argwhere(mask == 0)[0][::-1]
    mom, dens = orc.q_solve(p, h, D, mask, [tuple(src_free)], dt, 5, keep_density=True)
    u0 = np.zeros_like(u)
    u0[src_free[1], src_free[0]] = np.linalg.solve(Q.local(p, h)[0], _q_basis_at_centre(p))
    assert np.allclose(dens[0], Q.ssprk3(L, u0.reshape(-1), dt, 5).reshape(u.shape), rtol=0,
                       atol=(1e-12 if p <= 2 else 1e-9) * np.abs(dens[0]).max())
    assert steps.shape == u.shape


def _q_basis_at_centre(p):
    from oracle import dense_quad as Q
    C = Q.coeffs(p)
    mons = [(a, b) for b in range(p + 1) for a in range(p + 1)]
    return np.array([sum(C[m, k] * 0.5 ** (a + b) for m, (a, b) in enumerate(mons)) for k in range(len(mons))])


def test_quad_free_space_closed_forms(orc):
    """Free space, walls >= 48 sigma away: Q1's projected central Dirac is the
    uniform density on the source pixel (M^-1 of N(1/2,1/2) = 1 since the Q1
    row sums of M are 1/4), so Sigma = 2 D Delta I + (h^2/12) I; Q2 holds
    x^2, y^2, so Sigma = 2 D Delta I exactly."""
    m = np.zeros((96, 96), np.uint8)
    S1, _ = orc.sigma(orc.q_solve(1, 1.0, 1.0, m, [(48, 48)], 1 / 32, 16))
    assert np.abs(S1 - (1.0 + 1 / 12) * np.eye(2)).max() <= 1e-12
    S2, mu2 = orc.sigma(orc.q_solve(2, 1.0, 1.0, m, [(48, 48)], 1 / 128, 64))
    assert np.abs(S2 - 1.0 * np.eye(2)).max() <= 1e-12
    assert np.abs(mu2).max() <= 1e-13


def test_quad_rotation_90_and_transpose_exact(orc):
    """Quads are D4-symmetric (no diagonal): a 90-degree rotation of a walled
    substrate gives Sigma' = R Sigma R^T to rounding (the triangles only
    converge in h), and the transpose swaps x and y exactly."""
    mask, src = _case(41)
    n = mask.shape[0]
    S, _ = orc.sigma(orc.q_solve(2, 1.0, 1.0, mask, src, 1 / 128, 120))
    Sr, _ = orc.sigma(orc.q_solve(2, 1.0, 1.0, np.rot90(mask).copy(), [(j, n - 1 - i) for i, j in src],
                                  1 / 128, 120))
    Rm = np.array([[0, -1], [1, 0]])
    assert np.allclose(Sr, Rm @ S @ Rm.T, rtol=1e-12, atol=1e-14)
    St, _ = orc.sigma(orc.q_solve(2, 1.0, 1.0, mask.T.copy(), [(j, i) for i, j in src], 1 / 128, 120))
    assert np.allclose(St, S[::-1, ::-1], rtol=1e-12, atol=1e-14)
    assert np.linalg.eigvalsh(S).min() > 0


@pytest.mark.parametrize("p,rho", [(1, 60.0), (2, 192.7953), (3, 462.37)])
def test_spectral_radius_bounds_pin_dt_max(orc, p, rho):
    """The library's dt limits are 2.5127453 / rho_p.  Pin rho_p
    against the assembled operator: the Bloch symbol of the all-open
    composite blocks (interior modes), a free grid with walls on all four
    sides (wall modes reach slightly above the interior sup for P2/P3) and
    random masks all stay inside rho_p, and rho_p is within 1 % of the
    largest of them (a constant far too large would waste steps, one too
    small would make dt_max unstable)."""
    blocks, stray = O2.composite_blocks(p, 15)
    assert stray < 1e-10
    seen = 0.0
    for tx in np.linspace(0, np.pi, 41):
        for ty in np.linspace(0, np.pi, 41):
            S = sum(B * np.exp(1j * (tx * o[0] + ty * o[1])) for o, B in blocks.items())
            seen = max(seen, np.abs(np.linalg.eigvals(S)).max())
    rng = np.random.default_rng(3)
    for n, f in ((12, 0.0), (7, 0.2), (7, 0.4)):
        mask = (rng.random((n, n)) < f).astype(np.uint8)
        lam = np.linalg.eigvals(O2.assemble(p, 1.0, 1.0, mask))
        assert lam.real.max() < 1e-9
        seen = max(seen, np.abs(lam).max())
    assert seen <= rho * (1 + 1e-9), seen
    assert rho <= 1.01 * seen, seen


@pytest.mark.parametrize("p,rho", [(1, 32.0), (2, 130.7)])
def test_quad_spectral_radius_pins_dt_max(orc, p, rho):
    """Quads (R22): the library's Q_p dt limit 2.5127453 / rho uses the Bloch
    radius of the 9-point-cross symbol; walled and random-mask operators stay
    inside it and rho is within 1 % of what is seen."""
    from oracle import dense_quad as Q
    B = Q.composite_blocks(p, 15)
    offs = [k for k, v in B.items() if np.abs(v).max() > 1e-12]
    seen = 0.0
    for tx in np.linspace(0, np.pi, 61):
        for ty in np.linspace(0, np.pi, 61):
            S = sum(B[o] * np.exp(1j * (tx * o[0] + ty * o[1])) for o in offs)
            seen = max(seen, np.abs(np.linalg.eigvals(S)).max())
    rng = np.random.default_rng(4)
    for n, f in ((10, 0.0), (7, 0.3)):
        lam = np.linalg.eigvals(Q.assemble(p, 1.0, 1.0, (rng.random((n, n)) < f).astype(np.uint8)))
        assert lam.real.max() < 1e-9
        seen = max(seen, np.abs(lam).max())
    assert seen <= rho and rho <= 1.01 * seen, seen


@pytest.mark.parametrize("p", [1, 2])
def test_quad_points(orc, p):
    """Quads with sub-pixel points (R21): a centre point is the pixel source
    (bitwise); the projection reproduces the moments the tensor space holds
    (mass 1 and first moments 0 for Q1 and Q2; second moments 0 for Q2);
    whole-pixel translation in free space changes no moment."""
    mask, src = _case(51)
    pts = [(i + 0.5, j + 0.5) for i, j in src]
    assert np.array_equal(orc.q_solve_points(p, 1.0, 1.0, mask, pts, 1 / 64, 10), orc.q_solve(p, 1.0, 1.0, mask, src, 1 / 64, 10))
    m = np.zeros((6, 6), np.uint8)
    h = 0.7
    P0 = [(2.71 * h, 3.22 * h), (2.0 * h, 3.3 * h), (2.6 * h, 3.0 * h)]
    mom = orc.q_solve_points(p, h, 1.0, m, P0, 1e-3, 0)
    assert np.allclose(mom[:, 0], 1.0, rtol=0, atol=1e-13)
    assert np.abs(mom[:, 1:3]).max() <= 1e-13
    if p == 2:
        assert np.abs(mom[:, 3:]).max() <= 1e-13
    f = np.zeros((96, 96), np.uint8)                   # walls >= 45 sigma (Q2 tails are long)
    a = orc.q_solve_points(p, 1.0, 1.0, f, [(47.3, 48.6), (48.3, 48.6)], 1 / 64, 32)
    assert np.allclose(a[0], a[1], rtol=0, atol=1e-12)


@pytest.mark.parametrize("p", [1, 2])
def test_quad_absorb_matches_dense_and_loses_mass(orc, p):
    """Quads under ABSORB (Eq. (4): h_u = 0 and h_q = k q- . n on the outer
    square): O1q == O2q on random masks touching every edge, and mass leaves
    through the outer square (it is conserved under REFLECT)."""
    from oracle import dense_quad as Q
    rng = np.random.default_rng(90 + p)
    d = (p + 1) ** 2
    mask = (rng.random((6, 7)) < 0.3).astype(np.uint8)
    u = rng.standard_normal((6, 7, d))
    u[mask.astype(bool)] = 0
    ref = (Q.assemble(p, 0.7, 1.3, mask, 1) @ u.reshape(-1)).reshape(u.shape)
    got = orc.q_apply_L(p, 0.7, 1.3, mask, u, outer_bc=1)
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)
    m = np.zeros((10, 10), np.uint8)
    mr = orc.q_solve(p, 1.0, 1.0, m, [(1, 1)], 1 / 64, 100)
    ma = orc.q_solve(p, 1.0, 1.0, m, [(1, 1)], 1 / 64, 100, outer_bc=1)
    assert abs(mr[0, 0] - 1) < 1e-13 and ma[0, 0] < 0.9
