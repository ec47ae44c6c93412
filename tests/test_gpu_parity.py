"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle O1,
element by element on the same seeded inputs, plus the closed forms.

Tolerances (BASELINE.json north_star): fp64 densities <= 1e-12 relative L2,
Sigma <= 1e-10; fp32 densities <= 1e-5, Sigma <= 1e-4 (relative to the
diagonal scale, SURVEY §8d "parity norms").
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = {64: dict(dens=1e-12, sig=1e-10, mom=1e-10), 32: dict(dens=1e-5, sig=1e-4, mom=1e-4)}


@pytest.fixture(scope="module")
def dg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1907_06191_b200 import build
    build.build_all()
    from paper_1907_06191_b200 import dgdiff
    return dgdiff


@pytest.fixture(scope="module")
def cfg():
    from paper_1907_06191_b200 import configs
    return configs


def rel_l2(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def sig_err(S, R):
    return np.abs(S - R).max() / max(R[0, 0], R[1, 1])


def mom_err(m, r):
    scale = np.array([1, 1, 1, 1, 1, 1.0]) * np.maximum(np.abs(r[:, :1]), 1e-300)
    scale[:, 3:] = np.maximum(np.abs(r[:, 3:4]) + np.abs(r[:, 5:6]), 1e-300)
    scale[:, 1:3] = np.sqrt(scale[:, 3:4])
    return (np.abs(m - r) / scale).max()


@pytest.mark.parametrize("kernel", [0, 1])
@pytest.mark.parametrize("prec", [64, 32])
def test_c1_densities_moments_sigma(dg, orc, cfg, prec, kernel):
    """Config c1 (BASELINE configs[0]): full density parity vs O1."""
    m = cfg.mask("c1")
    src = cfg.sources("c1")
    c = cfg.CONFIGS["c1"]
    ref_m, ref_d = orc.solve(1, 1.0, 1.0, m, src, c.dt, c.nsteps, keep_density=True)
    with dg.Solver(m, 1.0, 1.0, 1, precision=prec, keep_density=1, kernel=kernel) as s:
        s.solve(src, c.dt, c.nsteps)
        S, mu = s.covariance()
        got = s.density(0)
        mom = s.moments()
    t = TOL[prec]
    assert rel_l2(got, ref_d[0]) <= t["dens"]
    assert np.all(got[m.astype(bool)] == 0)                    # axon stasis
    R, rmu = orc.sigma(ref_m)
    assert sig_err(S, R) <= t["sig"]
    assert mom_err(mom, ref_m) <= t["mom"]
    assert abs(mom[0, 0] - 1) <= (1e-12 if prec == 64 else 2e-6)  # mass


@pytest.mark.parametrize("kernel", [0, 1])
@pytest.mark.parametrize("p,prec", [(1, 64), (1, 32), (2, 64), (2, 32)])
def test_random_masks_ragged_batches(dg, orc, p, prec, kernel):
    """Random masks (all 16 face codes, walls at the grid edge), a ragged
    number of sources (not a multiple of the 64/128-source group), several
    chunks, P1 and P2."""
    rng = np.random.default_rng(100 + p * 7 + prec)
    ny, nx = 23, 29
    m = (rng.random((ny, nx)) < 0.4).astype(np.uint8)
    free = np.argwhere(m == 0)
    G = 64 if prec == 64 else 128                             # sources per warp group
    n = G + 13                                                # ragged: 2 chunks, 13 in the last
    pick = free[rng.integers(0, len(free), n)]
    src = np.stack([pick[:, 1], pick[:, 0]], 1).astype(np.int32)
    dt = (1 / 32 if p == 1 else 1 / 128) * 0.64 / 1.7         # h = 0.8, D = 1.7
    nsteps = 60
    ref_m, ref_d = orc.solve(p, 0.8, 1.7, m, src, dt, nsteps, keep_density=True)
    with dg.Solver(m, 0.8, 1.7, p, precision=prec, keep_density=1, max_chunk=G, kernel=kernel) as s:
        s.solve(src, dt, nsteps)
        S, mu = s.covariance()
        mom = s.moments()
        st = s.stats()
        last = range(G, n)                                    # the last chunk is kept
        dens = [s.density(k) for k in last]
    t = TOL[prec]
    assert st["chunk"] == G
    for k, dk in zip(last, dens):
        assert rel_l2(dk, ref_d[k]) <= t["dens"], k
    R, rmu = orc.sigma(ref_m)
    assert sig_err(S, R) <= t["sig"]
    assert np.allclose(mu, rmu, atol=t["sig"] * np.sqrt(R[0, 0]))
    assert mom_err(mom, ref_m) <= t["mom"]


def test_chunking_is_bitwise_invariant(dg, cfg):
    """Per-source moments do not depend on how sources are chunked, so Sigma
    is bitwise identical (the property the multi-GPU all-reduce relies on)."""
    m = cfg.mask("c1")
    rng = np.random.default_rng(9)
    free = np.argwhere(m == 0)
    pick = free[rng.integers(0, len(free), 300)]
    src = np.stack([pick[:, 1], pick[:, 0]], 1).astype(np.int32)
    out = []
    for mc in (0, 64, 128):
        with dg.Solver(m, 1.0, 1.0, 1, max_chunk=mc) as s:
            s.solve(src, 1 / 32, 40)
            out.append((s.covariance()[0], s.moments()))
    for S, mom in out[1:]:
        assert np.array_equal(S, out[0][0])
        assert np.array_equal(mom, out[0][1])


@pytest.mark.parametrize("prec", [64, 32])
def test_c2_free_space_closed_form(dg, orc, cfg, prec):
    """Config c2 at full size (256^2, 1024 sources, 512 steps): Sigma =
    2 D Delta I + h^2 [[1/20, 1/15], [1/15, 1/20]] (sharpening
    P:286-299), and O1 parity on a source subset over 64 steps."""
    m = cfg.mask("c2")
    src = cfg.sources("c2")
    c = cfg.CONFIGS["c2"]
    with dg.Solver(m, 1.0, 1.0, 1, precision=prec) as s:
        s.solve(src, c.dt, c.nsteps)
        S, mu = s.covariance()
    delta = c.nsteps * c.dt
    expect = 2 * delta * np.eye(2) + np.array([[1 / 20, 1 / 15], [1 / 15, 1 / 20]])
    tol = 1e-12 if prec == 64 else 1e-4
    assert np.abs(S - expect).max() <= tol * expect[0, 0]
    assert np.abs(mu).max() <= tol * 10
    sub = src[::128]
    ref_m, ref_d = orc.solve(1, 1.0, 1.0, m, sub, c.dt, 64, keep_density=True)
    with dg.Solver(m, 1.0, 1.0, 1, precision=prec, keep_density=1) as s:
        s.solve(sub, c.dt, 64)
        for k in range(len(sub)):
            assert rel_l2(s.density(k), ref_d[k]) <= TOL[prec]["dens"]


def test_c2_p2_closed_form(dg, cfg):
    """P2 variant of c2: Sigma = 2 D Delta I exactly (dt = 1/128, 512 steps)."""
    m = cfg.mask("c2")
    src = cfg.sources("c2")[::4]
    with dg.Solver(m, 1.0, 1.0, 2) as s:
        s.solve(src, 1 / 128, 512)
        S, mu = s.covariance()
    assert np.abs(S - 8.0 * np.eye(2)).max() <= 1e-11 * 8


def test_errors_on_gpu(dg, cfg):
    m = cfg.mask("c1")
    with dg.Solver(m, 1.0, 1.0, 1) as s:
        with pytest.raises(dg.DGDiffError) as e:
            s.solve([[16, 16]], 1 / 32, 1)                  # axon pixel
        assert e.value.status == dg.E_SOURCE
        with pytest.raises(dg.DGDiffError) as e:
            s.solve([[4, 16]], 0.05, 1)                      # dt > 2.5127/60
        assert e.value.status == dg.E_UNSTABLE
        with pytest.raises(dg.DGDiffError) as e:
            s.covariance(1.0)                                # no solve yet
        assert e.value.status == dg.E_STATE
        s.solve([[4, 16]], 1 / 32, 10)
        with pytest.raises(dg.DGDiffError) as e:
            s.covariance(1.0)                                # delta != nsteps dt
        assert e.value.status == dg.E_STATE
        S, _ = s.covariance(10 / 32)
        assert S[0, 1] == S[1, 0]


# ---------------------------------------------------------------- K3 fused step
@pytest.mark.parametrize("prec", [64, 32])
def test_fused_step_c1_and_ragged(dg, orc, cfg, prec):
    """K3 (one SSP-RK3 step per pass, temporal_steps=2) vs O1: c1 densities and
    a ragged multi-chunk batch on a random mask (walls, all face codes)."""
    m = cfg.mask("c1")
    src = cfg.sources("c1")
    c = cfg.CONFIGS["c1"]
    ref_m, ref_d = orc.solve(1, 1.0, 1.0, m, src, c.dt, c.nsteps, keep_density=True)
    with dg.Solver(m, 1.0, 1.0, 1, precision=prec, keep_density=1, temporal_steps=2) as s:
        s.solve(src, c.dt, c.nsteps)
        S, _ = s.covariance()
        got = s.density(0)
    t = TOL[prec]
    assert rel_l2(got, ref_d[0]) <= t["dens"]
    R, _ = orc.sigma(ref_m)
    assert sig_err(S, R) <= t["sig"]
    rng = np.random.default_rng(300 + prec)
    mk = (rng.random((37, 41)) < 0.4).astype(np.uint8)
    free = np.argwhere(mk == 0)
    n = 32 + 9
    pick = free[rng.integers(0, len(free), n)]
    srcs = np.stack([pick[:, 1], pick[:, 0]], 1).astype(np.int32)
    dt = 1 / 32 * 0.49 / 1.3
    ref_m, ref_d = orc.solve(1, 0.7, 1.3, mk, srcs, dt, 45, keep_density=True)
    with dg.Solver(mk, 0.7, 1.3, 1, precision=prec, keep_density=1, max_chunk=32, temporal_steps=2) as s:
        s.solve(srcs, dt, 45)
        S, _ = s.covariance()
        mom = s.moments()
        dens = [s.density(k) for k in range(32, n)]
    for k, dk in zip(range(32, n), dens):
        assert rel_l2(dk, ref_d[k]) <= t["dens"], k
    assert mom_err(mom, ref_m) <= t["mom"]
    assert sig_err(S, orc.sigma(ref_m)[0]) <= t["sig"]


@pytest.mark.parametrize("nsteps", [1, 2, 7])
def test_fused_step_equals_per_stage(dg, cfg, nsteps):
    """K3 performs the per-stage kernel's arithmetic in the same order per
    pixel; on the c3 substrate (several bands and strips) the moments agree to
    rounding (odd and even step counts exercise the ping-pong buffers)."""
    m = cfg.mask("c3")
    src = cfg.sources("c3", 96)
    out = {}
    for ts in (1, 2):
        with dg.Solver(m, 1.0, 1.0, 1, temporal_steps=ts) as s:
            s.solve(src, 1 / 32, nsteps)
            out[ts] = (s.moments(), s.covariance()[0])
    assert mom_err(out[2][0], out[1][0]) <= 1e-13
    assert np.abs(out[2][1] - out[1][1]).max() <= 1e-13 * out[1][1].max()


@pytest.mark.parametrize("prec,p", [(64, 1), (32, 1), (64, 2)])
def test_mixture_grid_and_residual(dg, orc, prec, p):
    """N2: the mixture grid and Eq. (9) residual vs the
    oracle on a random mask with walls, several chunks, ragged batch."""
    rng = np.random.default_rng(500 + prec + p)
    mk = (rng.random((48, 44)) < 0.35).astype(np.uint8)
    free = np.argwhere(mk[12:36, 12:32] == 0) + 12
    G = 64 if p == 1 and prec == 64 else (128 if p == 1 else 32)
    n = G + 5
    pick = free[rng.integers(0, len(free), n)]
    src = np.stack([pick[:, 1], pick[:, 0]], 1).astype(np.int32)
    dt = 1 / 32 if p == 1 else 1 / 128
    R = 12
    ref_m, ref_d = orc.solve(p, 1.0, 1.0, mk, src, dt, 50, keep_density=True)
    ref_g = orc.mixture(p, ref_d, src, ref_m, R)
    S_ref, mu_ref = orc.sigma(ref_m)
    ref_res = orc.residual(ref_g, 1.0, S_ref, mu_ref)
    with dg.Solver(mk, 1.0, 1.0, p, precision=prec, mixture_radius=R, max_chunk=G) as s:
        s.solve(src, dt, 50)
        S, mu = s.covariance()
        g, res = s.mixture()
    tol = 1e-12 if prec == 64 else 1e-5
    assert rel_l2(g, ref_g) <= tol
    assert abs(res - ref_res) <= (1e-10 if prec == 64 else 1e-3) * ref_res


def test_nccl_one_rank_world(dg, cfg):
    """The multi-GPU code path on one device: a one-rank NCCL communicator
    (dlopen, ncclCommInitRank, the moment-table and mixture all-reduces) gives
    bitwise the same Sigma and mixture as the communicator-free path."""
    import torch
    m = cfg.mask("c1")
    rng = np.random.default_rng(11)
    free = np.argwhere(m == 0)
    pick = free[rng.integers(0, len(free), 70)]
    src = np.stack([pick[:, 1], pick[:, 0]], 1).astype(np.int32)
    out = []
    for nid in (None, torch.cuda.nccl.unique_id()):
        with dg.Solver(m, 1.0, 1.0, 1, nccl_id=nid, mixture_radius=6) as s:
            s.solve(src, 1 / 32, 30)
            S, mu = s.covariance()
            g, res = s.mixture()
            out.append((S, mu, g, res))
    for a, b in zip(out[0], out[1]):
        assert np.array_equal(a, b)


# ---------------------------------------------------------------- ABSORB outer boundary (Eq. (4))
@pytest.mark.parametrize("prec", [64, 32])
def test_absorb_c1_golden_and_oracle(dg, orc, cfg, prec):
    """outer_bc = ABSORB (Eq. (4)) on c1: densities vs O1 and the
    independent implementation's m00 / Sigma after 200 steps."""
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "c1_independent_A10.json")))["absorb_200"]
    m = cfg.mask("c1")
    src = cfg.sources("c1")
    ref_m, ref_d = orc.solve(1, 1.0, 1.0, m, src, 1 / 32, 200, outer_bc=1, keep_density=True)
    with dg.Solver(m, 1.0, 1.0, 1, precision=prec, outer_bc=1, keep_density=1) as s:
        s.solve(src, 1 / 32, 200)
        S, _ = s.covariance()
        mom = s.moments()
        dens = s.density(0)
    t = TOL[prec]
    assert rel_l2(dens, ref_d[0]) <= t["dens"]
    assert abs(mom[0, 0] - g["m00"]) <= (1e-12 if prec == 64 else 1e-5)
    assert np.allclose([S[0, 0], S[0, 1], S[1, 1]], g["sigma"], rtol=t["sig"], atol=t["sig"])


@pytest.mark.parametrize("p,prec", [(1, 64), (1, 32), (2, 64), (3, 64)])
def test_absorb_random_masks(dg, orc, p, prec):
    """ABSORB on random masks touching every grid edge (all (code, outer)
    combinations occur), ragged two-chunk batch, vs O1."""
    rng = np.random.default_rng(700 + p * 3 + prec)
    mk = (rng.random((21, 26)) < 0.3).astype(np.uint8)
    free = np.argwhere(mk == 0)
    G = 64 if p == 1 and prec == 64 else (128 if p == 1 else 32)
    n = G + 7
    pick = free[rng.integers(0, len(free), n)]
    src = np.stack([pick[:, 1], pick[:, 0]], 1).astype(np.int32)
    dt = {1: 1 / 32, 2: 1 / 128, 3: 1 / 256}[p]
    ref_m, ref_d = orc.solve(p, 1.0, 1.0, mk, src, dt, 80, outer_bc=1, keep_density=True)
    with dg.Solver(mk, 1.0, 1.0, p, precision=prec, outer_bc=1, keep_density=1, max_chunk=G) as s:
        s.solve(src, dt, 80)
        S, _ = s.covariance()
        mom = s.moments()
        dens = [s.density(k) for k in range(G, n)]
    t = TOL[prec]
    for k, dk in zip(range(G, n), dens):
        assert rel_l2(dk, ref_d[k]) <= t["dens"], k
    assert mom_err(mom, ref_m) <= t["mom"]
    assert sig_err(S, orc.sigma(ref_m)[0]) <= t["sig"]
    assert mom[:, 0].min() < 1.0                                  # mass leaves through the outer square


# ---------------------------------------------------------------- edge cases
def test_zero_steps_is_projected_dirac(dg, cfg):
    """nsteps = 0: moments of the projected Dirac itself, P1 Sigma(0) =
    h^2 [[1/20, 1/10], [1/10, 1/20]] (closed form) and mass 1."""
    m = np.zeros((9, 9), np.uint8)
    with dg.Solver(m, 0.5, 1.0, 1) as s:
        s.solve([[4, 4], [2, 6]], 0.001, 0)
        S, mu = s.covariance(0.0)
        mom = s.moments()
    assert np.allclose(mom[:, 0], 1.0, atol=1e-14)
    assert np.allclose(S, 0.25 * np.array([[1 / 20, 1 / 10], [1 / 10, 1 / 20]]), atol=1e-15)
    assert np.allclose(mu, 0, atol=1e-15)


@pytest.mark.parametrize("prec", [64, 32])
def test_trapped_pocket_and_enclosure(dg, orc, prec):
    """A source in a one-pixel pocket never leaves it (all four faces closed:
    its operator is the code-0 block) and keeps mass 1; a source inside a
    closed 5x5 room of axons conserves mass and matches O1."""
    m = np.ones((16, 16), np.uint8)
    m[3, 3] = 0                                   # isolated pixel
    m[8:13, 6:11] = 0                             # closed room
    src = np.array([[3, 3], [8, 10], [6, 12]], np.int32)
    ref_m, ref_d = orc.solve(1, 1.0, 1.0, m, src, 1 / 32, 300, keep_density=True)
    with dg.Solver(m, 1.0, 1.0, 1, precision=prec, keep_density=1) as s:
        s.solve(src, 1 / 32, 300)
        mom = s.moments()
        d = [s.density(k) for k in range(3)]
    t = TOL[prec]
    for k in range(3):
        assert rel_l2(d[k], ref_d[k]) <= t["dens"]
    assert np.abs(mom[:, 0] - 1).max() <= (1e-12 if prec == 64 else 2e-6)
    assert np.abs(d[0]).sum() == np.abs(d[0][3, 3]).sum()    # nothing outside the pocket


def test_argument_and_state_errors(dg, cfg):
    m = cfg.mask("c1")
    with pytest.raises(dg.DGDiffError) as e:
        dg.Solver(m, 1.0, 1.0, 1).solve(np.zeros((0, 2), np.int32), 1 / 32, 1)
    assert e.value.status == dg.E_ARG
    with dg.Solver(m, 1.0, 1.0, 1) as s:
        s.solve([[4, 16]], 1 / 32, 2)
        with pytest.raises(dg.DGDiffError) as e:
            s.density(0)                                          # keep_density off
        assert e.value.status == dg.E_STATE
        with pytest.raises(dg.DGDiffError) as e:
            s.mixture()                                           # mixture_radius 0
        assert e.value.status == dg.E_STATE
        with pytest.raises(dg.DGDiffError) as e:
            s.solve([[-1, 3]], 1 / 32, 1)
        assert e.value.status == dg.E_SOURCE
    dtm = dg.dgdiff_dt_max(1, 1.0, 1.0)
    with dg.Solver(m, 1.0, 1.0, 1) as s:
        s.solve([[4, 16]], dtm, 10)                               # the limit itself is allowed
        S, _ = s.covariance()
        assert np.all(np.isfinite(S))
    with pytest.raises(dg.DGDiffError) as e:
        dg.Solver(m, 1.0, 1.0, 1, outer_bc=1, temporal_steps=2)
    assert e.value.status == dg.E_ARG


# ---------------------------------------------------------------- N3 Monte-Carlo cross-check
def test_mc_matches_reference_bitwise(dg):
    """GPU walkers == the numpy reference (same Philox stream, same rules):
    displacements bit for bit on a random mask with walls."""
    from oracle import mc
    rng = np.random.default_rng(17)
    m = (rng.random((24, 24)) < 0.35).astype(np.uint8)
    free = np.argwhere(m[6:18, 6:18] == 0) + 6
    src = np.stack([free[:5, 1], free[:5, 0]], 1).astype(np.int32)
    K, T, delta = 40, 150, 3.0
    with dg.Solver(m, 1.0, 1.0, 1) as s:
        S, mu, se, disp = s.mc_covariance(src, K, T, delta, seed=99, want_disp=True)
    l = np.sqrt(4 * 1.0 * delta / T)
    ref = mc.walk(m, src, K, T, l, 99)
    assert np.array_equal(disp, ref)


def test_mc_free_space_sigma(dg):
    """Free space: MC Sigma = 2 D Delta I within 4 standard errors (2D walk of
    step l: E[dx^2] = T l^2 / 2 = 2 D Delta)."""
    m = np.zeros((256, 256), np.uint8)
    src = np.array([[128, 128], [120, 131]], np.int32)
    with dg.Solver(m, 0.5, 2.0, 1) as s:
        S, mu, se = s.mc_covariance(src, 200000, 400, 1.5, seed=5)
    want = 2 * 2.0 * 1.5
    assert abs(S[0, 0] - want) < 4 * se[0] and abs(S[1, 1] - want) < 4 * se[2]
    assert abs(S[0, 1]) < 4 * se[1]


def test_dg_vs_mc_gamma_substrate_refinement(dg, cfg):
    """Physics cross-check (the paper's DG-vs-MC comparison) on the
    c3 Gamma substrate, 64 sources, Delta = 8: MC with reflecting (rejecting)
    walls on the pixel mask vs DG on the SAME staircase geometry at h and h/2
    (each pixel split 2 x 2; the sources are the same physical points).  The
    P1 gap is the O(h) wall error of the paper's u+ = 0 wall flux (reading
    R6): it must shrink like h (measured 5.7 % -> 2.9 % -> 1.1 % at h, h/2,
    h/4, profiles/r02_dg_mc_refine.jsonl); P2 is within ~1.2 % at h.  Both
    hindered well below 2 D Delta."""
    m = cfg.mask("c3")
    src = cfg.sources("c3", 64)
    pts = src.astype(np.float64) + 0.5
    with dg.Solver(m, 1.0, 1.0, 1) as s:
        Sm, _, se = s.mc_covariance(src, 20000, 8192, 8.0, seed=2024)
    gaps = {}
    for p, f in ((1, 1), (1, 2), (2, 1)):
        h = 1.0 / f
        dt = h * h / (32 if p == 1 else 128)
        with dg.Solver(np.kron(m, np.ones((f, f), np.uint8)), h, 1.0, p, windows=1) as s:
            s.solve_points(pts, dt, int(round(8.0 / dt)))
            S, _ = s.covariance()
        gaps[p, f] = np.mean([abs(S[k, k] - Sm[k, k]) / Sm[k, k] for k in (0, 1)])
        assert S[0, 0] < 0.7 * 16.0 and S[1, 1] < 0.7 * 16.0
    assert Sm[0, 0] < 0.7 * 16.0 and Sm[1, 1] < 0.7 * 16.0
    assert gaps[1, 1] <= 0.08 and gaps[2, 1] <= 0.025
    assert gaps[1, 2] <= 0.6 * gaps[1, 1], gaps          # O(h): halves per refinement
    assert gaps[1, 2] <= 0.04, gaps


@pytest.mark.parametrize("p,prec,outer", [(1, 64, 0), (1, 32, 0), (2, 64, 0), (1, 64, 1)])
def test_windows_bitwise_equal_whole_grid(dg, cfg, p, prec, outer):
    """N1 active windows: Morton-sorted source groups, stages clipped to each
    group's source box grown by one pixel per stage.  Every source's arithmetic
    inside its support is unchanged and everything outside is exactly zero, so
    moments and densities equal the whole-grid solve bit for bit -- across
    several ragged chunks, sources near the grid edge (ABSORB boundary blocks)
    and a box that outgrows the grid."""
    m = cfg.mask("c3")
    rng = np.random.default_rng(21)
    free = np.argwhere(m == 0)
    src = free[rng.choice(len(free), 300, replace=False)][:, ::-1].astype(np.int32)
    edge = free[(free[:, 0] < 3) | (free[:, 1] > 508)][:4][:, ::-1].astype(np.int32)
    src = np.concatenate([src, edge])
    dt = 1 / 32 if p == 1 else 1 / 128
    out = {}
    for w in (0, 1):
        with dg.Solver(m, 1.0, 1.0, p, precision=prec, keep_density=1, max_chunk=128, outer_bc=outer,
                       mixture_radius=6, windows=w) as s:
            s.solve(src, dt, 40)
            S, mu = s.covariance()
            n = len(src)
            dens = {k: s.density(k) for k in range(n - 300, n, 37) if _in_last_chunk(s, k)}
            out[w] = (s.moments(), S, mu, s.mixture(), dens, s.stats())
    m0, m1 = out[0][0], out[1][0]
    assert np.array_equal(m0, m1)
    assert np.array_equal(out[0][1], out[1][1]) and np.array_equal(out[0][2], out[1][2])
    g0, g1 = out[0][3][0], out[1][3][0]
    assert np.abs(g0 - g1).max() <= 1e-13 * np.abs(g0).max()
    common = set(out[0][4]) & set(out[1][4])
    for k in common:
        assert np.array_equal(out[0][4][k], out[1][4][k]), k
    # the windowed solve moves fewer bytes
    assert out[1][5]["stage_bytes"] < out[0][5]["stage_bytes"]


def _in_last_chunk(s, k):
    try:
        s.density(k)
        return True
    except Exception:
        return False


def test_windows_c1_oracle(dg, orc, cfg):
    """N1 windows on config c1 (one source next to the disk, 200 steps: the
    box outgrows the 32^2 grid) against O1."""
    m = cfg.mask("c1")
    src = cfg.sources("c1")
    c = cfg.CONFIGS["c1"]
    ref_m, ref_d = orc.solve(1, 1.0, 1.0, m, src, c.dt, c.nsteps, keep_density=True)
    for nst in (3, c.nsteps):
        r_m, r_d = orc.solve(1, 1.0, 1.0, m, src, c.dt, nst, keep_density=True)
        with dg.Solver(m, 1.0, 1.0, 1, keep_density=1, windows=1) as s:
            s.solve(src, c.dt, nst)
            got = s.density(0)
            mom = s.moments()
        assert rel_l2(got, r_d[0]) <= 1e-12
        assert mom_err(mom, r_m) <= 1e-10
        if nst == 3:   # after 3 steps = 9 stages the support is within 9 pixels (L1)
            i0, j0 = src[0]
            jj, ii = np.nonzero(np.abs(got).sum(axis=(2, 3)))
            assert (np.abs(ii - i0) + np.abs(jj - j0)).max() <= 9


@pytest.mark.parametrize("prec", [64, 32])
def test_p3_random_masks_and_free_space(dg, orc, prec):
    """N4: P3 on the ring kernel (V + sum F_f self blocks, non-dyadic
    coefficients rounded to the state precision) against O1 on a random mask
    with a ragged two-chunk batch, and the free-space closed form
    Sigma = 2 D Delta I (P3 reproduces quadratics)."""
    rng = np.random.default_rng(300 + prec)
    ny, nx = 21, 27
    m = (rng.random((ny, nx)) < 0.4).astype(np.uint8)
    free = np.argwhere(m == 0)
    G = 32 if prec == 64 else 64
    n = G + 7
    pick = free[rng.integers(0, len(free), n)]
    src = np.stack([pick[:, 1], pick[:, 0]], 1).astype(np.int32)
    dt = 1 / 256 * 0.64 / 1.7
    ref_m, ref_d = orc.solve(3, 0.8, 1.7, m, src, dt, 50, keep_density=True)
    with dg.Solver(m, 0.8, 1.7, 3, precision=prec, keep_density=1, max_chunk=G) as s:
        s.solve(src, dt, 50)
        S, mu = s.covariance()
        mom = s.moments()
        dens = [s.density(k) for k in range(G, n)]
    t = TOL[prec]
    for k, dk in zip(range(G, n), dens):
        assert rel_l2(dk, ref_d[k]) <= t["dens"], k
    assert mom_err(mom, ref_m) <= t["mom"]
    R, _ = orc.sigma(ref_m)
    assert sig_err(S, R) <= t["sig"]
    fm = np.zeros((96, 96), np.uint8)
    with dg.Solver(fm, 1.0, 1.0, 3, precision=prec) as s:
        s.solve(np.array([[48, 48], [47, 49], [49, 47]], np.int32), 1 / 256, 256)
        S, mu = s.covariance()
    assert np.abs(S - 2.0 * np.eye(2)).max() <= (1e-11 if prec == 64 else 2e-4)


@pytest.mark.parametrize("p,prec,windows,element", [(1, 64, 0, 0), (1, 32, 0, 0), (2, 64, 0, 0), (1, 64, 1, 0),
                                                    (3, 64, 0, 0), (1, 64, 0, 1), (2, 64, 1, 1), (2, 32, 0, 1)])
def test_subpixel_points_vs_oracle(dg, orc, p, prec, windows, element):
    """N4 sub-pixel sources: points inside L, inside U, on the diagonal and on
    pixel edges (R21), a ragged two-chunk batch, against O1's solve_points
    (densities of the kept chunk, per-source moments about the point, Sigma)."""
    rng = np.random.default_rng(500 + 10 * p + prec + windows)
    ny, nx = 22, 26
    m = (rng.random((ny, nx)) < 0.35).astype(np.uint8)
    free = np.argwhere(m == 0)
    G = ({1: 64, 2: 32, 3: 32}[p] if element == 0 else 32) * (2 if prec == 32 else 1)
    n = G + 9
    pick = free[rng.integers(0, len(free), n)]
    loc = rng.random((n, 2))
    loc[0] = (0.3, 0.3)        # diagonal
    loc[1] = (0.0, 0.6)        # left edge
    loc[2] = (0.45, 0.0)       # bottom edge
    loc[3] = (0.5, 0.5)        # centre
    h = 0.8
    pts = (np.stack([pick[:, 1], pick[:, 0]], 1) + loc) * h
    dt = ({1: 1 / 32, 2: 1 / 128, 3: 1 / 256} if element == 0 else {1: 1 / 16, 2: 1 / 64})[p] * h * h / 1.3
    osolve = orc.solve_points if element == 0 else orc.q_solve_points
    ref_m, ref_d = osolve(p, h, 1.3, m, pts, dt, 30, keep_density=True)
    with dg.Solver(m, h, 1.3, p, precision=prec, keep_density=1, max_chunk=G, windows=windows,
                   element=element) as s:
        s.solve_points(pts, dt, 30)
        S, mu = s.covariance()
        mom = s.moments()
        dens = {k: s.density(k) for k in range(n) if _in_last_chunk(s, k)}
    t = TOL[prec]
    assert len(dens) == n - G
    for k, dk in dens.items():
        assert rel_l2(dk, ref_d[k]) <= t["dens"], k
    assert mom_err(mom, ref_m) <= t["mom"]
    R, _ = orc.sigma(ref_m)
    assert sig_err(S, R) <= t["sig"]


def test_points_at_centres_equal_pixel_sources(dg, cfg):
    """dgdiff_solve_batch_points at pixel centres == dgdiff_solve_batch, bitwise;
    out-of-grid / axon points are E_SOURCE; the mixture is refused."""
    m = cfg.mask("c3")
    src = cfg.sources("c3")[:100]
    with dg.Solver(m, 1.0, 1.0, 1, mixture_radius=4) as s:
        s.solve(src, 1 / 32, 20)
        a = s.moments()
        s.solve_points(src + 0.5, 1 / 32, 20)
        b = s.moments()
        s.covariance()
        with pytest.raises(dg.DGDiffError) as e:
            s.mixture()
        assert e.value.status == dg.E_STATE
        axon = np.argwhere(m == 1)[0][::-1] + 0.5
        for bad in ([[-0.1, 3.0]], [[512.0, 3.0]], [axon], [[np.nan, 1.0]]):
            with pytest.raises(dg.DGDiffError) as e:
                s.solve_points(np.array(bad, float), 1 / 32, 2)
            assert e.value.status == dg.E_SOURCE
    assert np.array_equal(a, b)


@pytest.mark.parametrize("p,prec", [(1, 64), (2, 64), (1, 32), (2, 32)])
def test_quads_random_masks_vs_oracle(dg, orc, p, prec):
    """N4 Q_p quadrilaterals (9-point-cross ring kernel: 2-column strip halo,
    rows j-2..j+2, 8 neighbour indices) against O1's element-loop quad path
    on a random walled mask with a ragged two-chunk batch."""
    rng = np.random.default_rng(700 + 10 * p + prec)
    ny, nx = 21, 25
    m = (rng.random((ny, nx)) < 0.35).astype(np.uint8)
    free = np.argwhere(m == 0)
    G = 32 if prec == 64 else 64
    n = G + 11
    pick = free[rng.integers(0, len(free), n)]
    src = np.stack([pick[:, 1], pick[:, 0]], 1).astype(np.int32)
    h, D = 0.8, 1.4
    dt = (1 / 16 if p == 1 else 1 / 64) * h * h / D
    ref_m, ref_d = orc.q_solve(p, h, D, m, src, dt, 40, keep_density=True)
    with dg.Solver(m, h, D, p, precision=prec, keep_density=1, max_chunk=G, element=1) as s:
        s.solve(src, dt, 40)
        S, mu = s.covariance()
        mom = s.moments()
        dens = {k: s.density(k) for k in range(G, n)}
    t = TOL[prec]
    for k, dk in dens.items():
        assert rel_l2(dk, ref_d[k]) <= t["dens"], k
    assert mom_err(mom, ref_m) <= t["mom"]
    R, _ = orc.sigma(ref_m)
    assert sig_err(S, R) <= t["sig"]


def test_quads_closed_forms_rotation_and_windows(dg):
    """Q1 / Q2 free space: Sigma = 2 D Delta I + h^2/12 I (Q1) and 2 D Delta I
    (Q2); on a walled substrate a 90-degree rotation gives R Sigma R^T exactly
    (quads are D4-symmetric); N1 windows are bitwise equal for quads too (the
    support grows by two pixels per stage)."""
    fm = np.zeros((96, 96), np.uint8)
    src = np.array([[48, 48], [47, 49], [49, 46]], np.int32)
    with dg.Solver(fm, 1.0, 1.0, 1, element=1) as s:
        s.solve(src, 1 / 32, 16)
        S1, _ = s.covariance()
    assert np.abs(S1 - (1.0 + 1 / 12) * np.eye(2)).max() <= 1e-11
    with dg.Solver(fm, 1.0, 1.0, 2, element=1) as s:
        s.solve(src, 1 / 128, 64)
        S2, _ = s.covariance()
    assert np.abs(S2 - 1.0 * np.eye(2)).max() <= 1e-11
    rng = np.random.default_rng(9)
    m = (rng.random((40, 40)) < 0.4).astype(np.uint8)
    free = np.argwhere(m[12:28, 12:28] == 0) + 12
    ps = np.array([(f[1], f[0]) for f in free[:20]], np.int32)
    n = m.shape[0]
    with dg.Solver(m, 1.0, 1.0, 2, element=1) as s:
        s.solve(ps, 1 / 128, 100)
        S, _ = s.covariance()
        mom0 = s.moments()
    with dg.Solver(np.rot90(m).copy(), 1.0, 1.0, 2, element=1) as s:
        s.solve(np.array([(j, n - 1 - i) for i, j in ps], np.int32), 1 / 128, 100)
        Sr, _ = s.covariance()
    Rm = np.array([[0, -1], [1, 0]])
    assert np.allclose(Sr, Rm @ S @ Rm.T, rtol=1e-12, atol=1e-14)
    with dg.Solver(m, 1.0, 1.0, 2, element=1, windows=1, max_chunk=32) as s:
        s.solve(ps, 1 / 128, 100)
        mom1 = s.moments()
    assert np.array_equal(mom0, mom1)


def test_handles_are_independent(dg, cfg):
    """Handles of different degree / element type alive at once give exactly
    the moments each gives alone (no process-wide tables: the moment and
    mixture weights travel with the handle)."""
    m = cfg.mask("c1")
    src = cfg.sources("c1")
    alone = {}
    for key in ((1, 0), (2, 0), (2, 1)):
        with dg.Solver(m, 1.0, 1.0, key[0], element=key[1], mixture_radius=3) as s:
            s.solve(src, 1 / 256, 20)
            s.covariance()
            alone[key] = (s.moments(), s.mixture()[0])
    hs = {key: dg.Solver(m, 1.0, 1.0, key[0], element=key[1], mixture_radius=3) for key in alone}
    try:
        for key in ((2, 1), (1, 0), (2, 0)):      # created in one order, solved in another
            hs[key].solve(src, 1 / 256, 20)
        for key, h in hs.items():
            h.covariance()
            assert np.array_equal(h.moments(), alone[key][0]), key
            assert np.array_equal(h.mixture()[0], alone[key][1]), key
    finally:
        for h in hs.values():
            h.close()


@pytest.mark.parametrize("p,element", [(1, 0), (2, 0), (3, 0), (1, 1), (2, 1)])
def test_degenerate_grids(dg, orc, p, element):
    """Edge cases of the substrate shape: a single pixel (no open face: the
    density must not move), a one-pixel-high strip (1-D diffusion; the ring
    kernel's bands and halos collapse), every source on the same pixel, and
    zero steps -- against the oracle (triangles or quads), with and without
    N1 windows."""
    solve = orc.solve if element == 0 else orc.q_solve
    dt = {1: 1 / 32, 2: 1 / 128, 3: 1 / 256}[p] if element == 0 else {1: 1 / 16, 2: 1 / 64}[p]
    for shape, src in (((1, 1), [(0, 0)]), ((1, 37), [(5, 0), (5, 0), (36, 0)]), ((29, 2), [(1, 28), (0, 0)])):
        m = np.zeros(shape, np.uint8)
        for nsteps in (0, 7):
            ref = solve(p, 1.0, 1.0, m, src, dt, nsteps)
            for w in (0, 1):
                with dg.Solver(m, 1.0, 1.0, p, element=element, windows=w) as s:
                    s.solve(np.array(src, np.int32), dt, nsteps)
                    mom = s.moments()
                # (absolute: the P2+ second moments of the projected Dirac are 0)
                assert np.abs(mom - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max()), (shape, nsteps, w)
                assert np.abs(mom[:, 0] - 1).max() <= 1e-13


def test_c4_device_filling_chunk_and_ragged_tail(dg, orc, cfg):
    """Maximum size: the c4 substrate with the chunk sized by free device
    memory (~640 sources, ~155 GB of RK registers on a B200) and a ragged
    second chunk; sources sampled in both chunks against O1 (2 steps)."""
    m = cfg.mask("c4")
    src = cfg.sources("c4", 1000)[:700]
    with dg.Solver(m, 1.0, 1.0, 1) as s:
        s.solve(src, 1 / 32, 2)
        mom = s.moments()
        st = s.stats()
    assert 256 < st["chunk"] < 700                    # memory-limited chunk, so there is a tail
    pick = np.array([1, st["chunk"] + 3])
    ref = orc.solve(1, 1.0, 1.0, m, src[pick], 1 / 32, 2)
    assert mom_err(mom[pick], ref) <= 1e-10
    assert np.abs(mom[:, 0] - 1).max() <= 1e-13


@pytest.mark.parametrize("p,element", [(1, 0), (2, 0), (3, 0), (1, 1), (2, 1)])
def test_windows_sigma_clip(dg, cfg, p, element):
    """N1 approximate windows (windows = 2, reading R23): the box growth is
    capped at K sigma (K = 20 / 30 / 45 for P1 / P2 / P3, 25 / 40 for Q1 /
    Q2), where the DG tails are below rounding: moments and Sigma agree with
    the whole-grid solve to 1e-12 although far fewer bytes move."""
    m = cfg.mask("c3")
    src = cfg.sources("c3")[:300]
    dt = ({1: 1 / 32, 2: 1 / 128, 3: 1 / 256} if element == 0 else {1: 1 / 16, 2: 1 / 64})[p]
    nst = 300
    res = {}
    for w in (0, 2):
        with dg.Solver(m, 1.0, 1.0, p, windows=w, element=element) as s:
            s.solve(src, dt, nst)
            S, mu = s.covariance()
            res[w] = (s.moments(), S, s.stats()["stage_bytes"])
    assert mom_err(res[2][0], res[0][0]) <= 1e-12
    assert np.abs(res[2][1] - res[0][1]).max() <= 1e-12 * res[0][1].max()
    assert res[2][2] < res[0][2]


@pytest.mark.parametrize("p,prec,windows", [(1, 64, 0), (2, 64, 0), (2, 32, 0), (2, 64, 1)])
def test_quads_absorb_vs_oracle(dg, orc, p, prec, windows):
    """Quads under ABSORB (Eq. (4)): pixels within two of the outer square use
    K0's runtime blocks (self by (code, outer), neighbour by opposite-face
    state and far-face-outer); sources next to every edge, against O1q."""
    rng = np.random.default_rng(800 + 10 * p + prec + windows)
    ny, nx = 19, 23
    m = (rng.random((ny, nx)) < 0.3).astype(np.uint8)
    free = np.argwhere(m == 0)
    edge = free[(free[:, 0] <= 1) | (free[:, 0] >= ny - 2) | (free[:, 1] <= 1) | (free[:, 1] >= nx - 2)]
    G = 32 if prec == 64 else 64
    pick = np.concatenate([edge[:G // 2], free[rng.integers(0, len(free), G // 2 + 5)]])
    src = np.stack([pick[:, 1], pick[:, 0]], 1).astype(np.int32)
    n = len(src)
    dt = (1 / 16 if p == 1 else 1 / 64) * 0.64 / 1.2
    ref_m, ref_d = orc.q_solve(p, 0.8, 1.2, m, src, dt, 40, keep_density=True, outer_bc=1)
    with dg.Solver(m, 0.8, 1.2, p, precision=prec, keep_density=1, max_chunk=G, element=1, outer_bc=1,
                   windows=windows) as s:
        s.solve(src, dt, 40)
        S, mu = s.covariance()
        mom = s.moments()
        dens = {k: s.density(k) for k in range(n) if _in_last_chunk(s, k)}
    t = TOL[prec]
    assert len(dens) > 0
    for k, dk in dens.items():
        assert rel_l2(dk, ref_d[k]) <= t["dens"], k
    assert mom_err(mom, ref_m) <= t["mom"]
    assert (ref_m[:, 0] < 1 - 1e-6).any()          # mass really leaves through the outer square


@pytest.mark.parametrize("nsteps", [1, 2, 7])
def test_k3b_decoupled_step_bitwise_equals_per_stage(dg, orc, cfg, nsteps):
    """K3b (temporal_steps = 3: the fused step with decoupled producer / U1 /
    U2 / u' warp roles handing rows on through mbarriers) performs each
    pixel's arithmetic in the per-stage kernel's order: moments and densities
    are bit-identical to K2 on the c3 substrate (several bands and strips,
    ragged two-chunk batch), and c1 matches O1 at 1e-12."""
    m = cfg.mask("c3")
    src = cfg.sources("c3", 96)[:77]
    out = {}
    for ts in (0, 3):
        with dg.Solver(m, 1.0, 1.0, 1, temporal_steps=ts, keep_density=1, max_chunk=64) as s:
            s.solve(src, 1 / 32, nsteps)
            out[ts] = (s.moments(), s.density(76))
    assert np.array_equal(out[3][0], out[0][0]) and np.array_equal(out[3][1], out[0][1])
    if nsteps == 7:
        c = cfg.CONFIGS["c1"]
        ref_m, ref_d = orc.solve(1, 1.0, 1.0, cfg.mask("c1"), cfg.sources("c1"), c.dt, c.nsteps, keep_density=True)
        with dg.Solver(cfg.mask("c1"), 1.0, 1.0, 1, temporal_steps=3, keep_density=1) as s:
            s.solve(cfg.sources("c1"), c.dt, c.nsteps)
            assert rel_l2(s.density(0), ref_d[0]) <= 1e-12


@pytest.mark.parametrize("degree,prec", [(1, 64), (1, 32), (2, 64), (2, 32)])
def test_k3c_wavefront_step_bitwise_equals_per_stage(dg, cfg, degree, prec):
    """K3c (temporal_steps = 4: one launch per SSP-RK3 step, the ring kernel's
    items of all three stages in wavefront order with per-item completion
    counters) does each pixel's arithmetic exactly as K2: moments and
    densities bit-identical on the c3 substrate (32 strips, several bands,
    two source groups in a chunk and a ragged second chunk), several steps."""
    m = cfg.mask("c3")
    src = cfg.sources("c3", 200)[:150]
    dt = 1 / 32 if degree == 1 else 1 / 128
    out = {}
    for ts in (0, 4):
        with dg.Solver(m, 1.0, 1.0, degree, precision=prec, temporal_steps=ts, keep_density=1, max_chunk=128) as s:
            s.solve(src, dt, 5)
            out[ts] = (s.moments(), s.density(149), s.density(129))   # densities: last chunk only
    for a, b in zip(out[4], out[0]):
        assert np.array_equal(a, b)


# ---------------------------------------------------------------- round 2: parity gaps closed
def test_centering_own_mean_vs_oracle(dg, orc, cfg):
    """opts.centering = 1 (own-mean centering, reading R12) on a walled
    Gamma substrate where the two readings differ by a few %: the GPU's K5
    branch against O1's orc_sigma(centering = 1), on the oracle's own moments
    (covariance_table) and on a live solve of sampled sources vs O1."""
    from paper_1907_06191_b200 import substrate as S
    m = S.gen_substrate(128, 128, 0.60, 41).mask
    src = S.sample_sources(m, 40, 42)
    nsteps = 100
    ref_m = orc.solve(1, 1.0, 1.0, m, src, 1 / 32, nsteps)
    R1, rmu1 = orc.sigma(ref_m, centering=1)
    R0, _ = orc.sigma(ref_m, centering=0)
    assert np.abs(R1 - R0).max() > 1e-3 * R0.max()          # the readings really differ here
    with dg.Solver(m, 1.0, 1.0, 1, centering=1) as s:
        s.solve(src, 1 / 32, nsteps)
        S1, mu1 = s.covariance()
        T1, tmu1 = s.covariance_table(ref_m)
        mom = s.moments()
    assert sig_err(T1, R1) <= 1e-13 and np.abs(tmu1).max() == 0.0
    assert sig_err(S1, R1) <= 1e-10
    assert np.abs(mu1).max() == 0.0
    assert mom_err(mom, ref_m) <= 1e-10
    with dg.Solver(m, 1.0, 1.0, 1, precision=32, centering=1) as s:
        s.solve(src, 1 / 32, nsteps)
        S1f, _ = s.covariance()
    assert sig_err(S1f, R1) <= 1e-4


@pytest.mark.parametrize("windows", [0, 1])
def test_logical_ranks_bitwise(dg, cfg, windows):
    """Multi-GPU readiness on one device: nranks = R handles
    without a communicator ("logical ranks") each solve their contiguous shard
    [r n/R, (r+1) n/R) into a zero-padded [n][6] table; the host sums the R
    tables (what ncclAllReduce does: disjoint rows plus zeros, exact) and K5
    reduces it in source order, so moments and Sigma are BITWISE those of one
    rank, for R = 2, 4, 8 -- with and without N1 windows (the batch is
    Morton-sorted before sharding, and the perm scatter puts each rank's rows
    back in input order)."""
    m = cfg.mask("c3")
    src = cfg.sources("c3", 1000)
    nsteps = 24
    with dg.Solver(m, 1.0, 1.0, 1, windows=windows) as s:
        s.solve(src, 1 / 32, nsteps)
        S1, mu1 = s.covariance()
        M1 = s.moments()
    for R in (2, 4, 8):
        tab = np.zeros_like(M1)
        owner = np.full(len(src), -1)
        for r in range(R):
            with dg.Solver(m, 1.0, 1.0, 1, windows=windows, rank=r, nranks=R) as s:
                s.solve(src, 1 / 32, nsteps)
                Mr = s.moments()
                b, e = dg.dgdiff_shard(len(src), r, R)
                mine = np.flatnonzero(np.any(Mr != 0, axis=1))
                if windows:
                    # the shard [b, e) of the batch in Morton order: e - b rows,
                    # disjoint from the other ranks'
                    assert len(mine) == e - b and np.all(owner[mine] == -1)
                else:
                    assert np.all(Mr[:b] == 0) and np.all(Mr[e:] == 0)
                owner[mine] = r
                with pytest.raises(dg.DGDiffError):
                    s.covariance()                               # a logical rank holds only its shard
                tab += Mr
                if r == R - 1:
                    SR, muR = s.covariance_table(tab)
        assert np.all(owner >= 0)
        assert np.array_equal(tab, M1), R
        assert np.array_equal(SR, S1) and np.array_equal(muR, mu1), R


@pytest.mark.parametrize("prec", [64, 32])
def test_k3c_wavefront_c1_vs_oracle(dg, orc, cfg, prec):
    """K3c (temporal_steps = 4) on config c1 against O1 directly (not only
    against K2): densities, moments, Sigma."""
    m = cfg.mask("c1")
    src = cfg.sources("c1")
    c = cfg.CONFIGS["c1"]
    ref_m, ref_d = orc.solve(1, 1.0, 1.0, m, src, c.dt, c.nsteps, keep_density=True)
    with dg.Solver(m, 1.0, 1.0, 1, precision=prec, temporal_steps=4, keep_density=1) as s:
        s.solve(src, c.dt, c.nsteps)
        S, _ = s.covariance()
        got = s.density(0)
        mom = s.moments()
    t = TOL[prec]
    assert rel_l2(got, ref_d[0]) <= t["dens"]
    assert mom_err(mom, ref_m) <= t["mom"]
    assert sig_err(S, orc.sigma(ref_m)[0]) <= t["sig"]


def test_windows_density_after_longer_solve(dg, orc, cfg):
    """N1 windows keep only each group's reachable rows; after a long solve the
    registers hold stale values outside a later short solve's range, and
    dgdiff_get_density must report exact zeros there: long
    windowed solve, then a 3-step one on the 512^2 grid, density vs O1."""
    m = cfg.mask("c3")
    src_long = cfg.sources("c3", 64)
    src = cfg.sources("c3", 130)[66:130]
    with dg.Solver(m, 1.0, 1.0, 1, windows=1, keep_density=1) as s:
        s.solve(src_long, 1 / 32, 60)
        s.solve(src, 1 / 32, 3)
        got = [s.density(k) for k in (0, 63)]
    ref_m, ref_d = orc.solve(1, 1.0, 1.0, m, src[[0, 63]], 1 / 32, 3, keep_density=True)
    for r in range(2):
        assert rel_l2(got[r], ref_d[r]) <= 1e-12
        assert np.array_equal(got[r] == 0, ref_d[r] == 0)


def test_kernel_option_range_checked(dg, cfg):
    """opts.kernel outside 0..3 is rejected (an undocumented value
    once selected a diagnostic path that skipped the arithmetic)."""
    for k in (-1, 4, 9):
        with pytest.raises(dg.DGDiffError):
            dg.Solver(cfg.mask("c1"), 1.0, 1.0, 1, kernel=k)


def test_product_library_ignores_environment(dg, cfg):
    """The product library reads no tuning knob from the environment."""
    with dg.Solver(cfg.mask("c1"), 1.0, 1.0, 1) as s:
        s.solve(cfg.sources("c1"), 1 / 32, 2)
        st = s.stats()
    assert st["tuning_build"] == 0 and st["env_overrides"] == 0


# ---------------------------------------------------------------- K3d: fused stages 2 + 3
@pytest.mark.parametrize("degree,prec", [(1, 64), (1, 32), (2, 64), (2, 32)])
def test_k3d_stage_pair_bitwise_equals_per_stage(dg, cfg, degree, prec):
    """K3d (temporal_steps = 5: stage 1 on K2, stages 2 + 3 in one launch with
    U2 in shared memory) does each pixel's arithmetic exactly as K2: moments
    and densities bit-identical on the c3 substrate (64 strips of 8 columns,
    several bands, two source groups and a ragged second chunk), over an even
    and an odd number of steps (the u / u' registers trade places each step)."""
    m = cfg.mask("c3")
    G = {(1, 64): 64, (1, 32): 128, (2, 64): 32, (2, 32): 64}[(degree, prec)]
    src = cfg.sources("c3", 400)[:2 * G + 7]
    dt = 1 / 32 if degree == 1 else 1 / 128
    for nsteps in (4, 5):
        out = {}
        for ts in (0, 5):
            with dg.Solver(m, 1.0, 1.0, degree, precision=prec, temporal_steps=ts, keep_density=1,
                           max_chunk=2 * G) as s:
                s.solve(src, dt, nsteps)
                S, mu = s.covariance()
                n = len(src)
                out[ts] = (s.moments(), S, mu, s.density(n - 1), s.density(2 * G))
        for a, b in zip(out[5], out[0]):
            assert np.array_equal(a, b), (degree, prec, nsteps)


@pytest.mark.parametrize("prec", [64, 32])
def test_k3d_c1_and_random_masks_vs_oracle(dg, orc, cfg, prec):
    """K3d against O1 directly: config c1 (full density, 200 steps) and a
    random mask with every face code, walls on the grid edge and a ragged
    batch (P1 and P2)."""
    m = cfg.mask("c1")
    c = cfg.CONFIGS["c1"]
    ref_m, ref_d = orc.solve(1, 1.0, 1.0, m, cfg.sources("c1"), c.dt, c.nsteps, keep_density=True)
    with dg.Solver(m, 1.0, 1.0, 1, precision=prec, temporal_steps=5, keep_density=1) as s:
        s.solve(cfg.sources("c1"), c.dt, c.nsteps)
        S, _ = s.covariance()
        got = s.density(0)
    t = TOL[prec]
    assert rel_l2(got, ref_d[0]) <= t["dens"]
    assert sig_err(S, orc.sigma(ref_m)[0]) <= t["sig"]
    rng = np.random.default_rng(77)
    mm = (rng.random((21, 37)) < 0.4).astype(np.uint8)
    free = np.argwhere(mm == 0)
    src = free[rng.integers(0, len(free), 45)][:, ::-1].astype(np.int32)
    for p in (1, 2):
        dt = (1 / 32 if p == 1 else 1 / 128)
        rm, rd = orc.solve(p, 1.0, 1.0, mm, src, dt, 13, keep_density=True)
        with dg.Solver(mm, 1.0, 1.0, p, precision=prec, temporal_steps=5, keep_density=1) as s:
            s.solve(src, dt, 13)
            mom = s.moments()
            for k in (0, 44):
                assert rel_l2(s.density(k), rd[k]) <= t["dens"], (p, k)
        assert mom_err(mom, rm) <= t["mom"], p


_P3CROP = {}


def _p3crop(orc, cfg):
    """77 sources (the fp32 batch; fp64 takes the first 45) on the crop, O1 once."""
    if not _P3CROP:
        m = np.ascontiguousarray(cfg.mask("c5")[384:640, 384:640])
        rng = np.random.default_rng(77)
        free = np.argwhere(m[64:192, 64:192] == 0) + 64
        pick = free[rng.choice(len(free), 77, replace=False)]
        src = np.stack([pick[:, 1], pick[:, 0]], 1).astype(np.int32)
        ref_m, ref_d = orc.solve(3, 1.0, 1.0, m, src, 1 / 256, 16, keep_density=True)
        _P3CROP.update(m=m, src=src, ref_m=ref_m, ref_d=ref_d)
    return _P3CROP


@pytest.mark.parametrize("prec", [64, 32])
def test_p3_gamma_crop_vs_oracle(dg, orc, cfg, prec):
    """N4 P3 on a 256^2 crop of the c5 Gamma substrate (round 2: the fp64
    kernel applies the column-form operator to pixel pairs): one chunk of two
    source groups (the second ragged), 16 steps, every density, moment and
    Sigma against O1.  Dense rows fill the ring to its minimum, pairs straddle
    open and closed faces, single pixels end odd rows."""
    d = _p3crop(orc, cfg)
    G = 32 if prec == 64 else 64
    n = G + 13
    src, ref_m, ref_d = d["src"][:n], d["ref_m"][:n], d["ref_d"][:n]
    with dg.Solver(d["m"], 1.0, 1.0, 3, precision=prec, keep_density=1, max_chunk=2 * G) as s:
        s.solve(src, 1 / 256, 16)
        S, mu = s.covariance()
        mom = s.moments()
        dens = [s.density(k) for k in range(n)]
    t = TOL[prec]
    assert max(rel_l2(dens[k], ref_d[k]) for k in range(n)) <= t["dens"]
    assert mom_err(mom, ref_m) <= t["mom"]
    R, _ = orc.sigma(ref_m)
    assert sig_err(S, R) <= t["sig"]


def test_q2_gamma_crop_full_bands_vs_oracle(dg, orc, cfg):
    """N4 Q2 on a 512 x 600 crop of the c5 Gamma substrate: 75 strips x 2
    source groups put the ring kernel at its 64-row band cap, so the item
    neighbour buffers (one bulk copy per item from the strip-major table)
    run full; one chunk of 37 sources (the second group ragged), 8 steps,
    every density, moment and Sigma against O1's quad path."""
    m = np.ascontiguousarray(cfg.mask("c5")[256:768, 200:800])
    rng = np.random.default_rng(45)
    free = np.argwhere(m[176:336, 220:380] == 0) + (176, 220)
    pick = free[rng.choice(len(free), 37, replace=False)]
    src = np.stack([pick[:, 1], pick[:, 0]], 1).astype(np.int32)
    dt, nst = 1 / 64, 8
    ref_m, ref_d = orc.q_solve(2, 1.0, 1.0, m, src, dt, nst, keep_density=True)
    with dg.Solver(m, 1.0, 1.0, 2, keep_density=1, max_chunk=64, element=1) as s:
        s.solve(src, dt, nst)
        S, mu = s.covariance()
        mom = s.moments()
        err = max(rel_l2(s.density(k), ref_d[k]) for k in range(37))
    t = TOL[64]
    assert err <= t["dens"]
    assert mom_err(mom, ref_m) <= t["mom"]
    R, _ = orc.sigma(ref_m)
    assert sig_err(S, R) <= t["sig"]


@pytest.mark.parametrize("windows", [0, 1])
def test_logical_ranks_more_ranks_than_sources(dg, cfg, windows):
    """R = 8 logical ranks for 3 sources: five ranks get an empty shard (a
    zero table, no kept chunk: get_density refuses instead of returning an
    earlier solve's state); the summed tables give one rank's Sigma bitwise."""
    m = cfg.mask("c1")
    src = np.array([[4, 16], [5, 16], [4, 17]], np.int32)
    with dg.Solver(m, 1.0, 1.0, 1, windows=windows) as s:
        s.solve(src, 1 / 32, 20)
        S1, mu1 = s.covariance()
        M1 = s.moments()
    tab = np.zeros_like(M1)
    for r in range(8):
        with dg.Solver(m, 1.0, 1.0, 1, windows=windows, rank=r, nranks=8, keep_density=1) as s:
            s.solve(np.repeat(src, 6, axis=0)[:16], 1 / 32, 4)   # earlier: every rank keeps a chunk
            s.solve(src, 1 / 32, 20)
            Mr = s.moments()
            b, e = dg.dgdiff_shard(len(src), r, 8)
            if e == b:
                assert np.all(Mr == 0)
                with pytest.raises(dg.DGDiffError):
                    s.density(0)
            tab += Mr
            if r == 7:
                SR, muR = s.covariance_table(tab)
    assert np.array_equal(tab, M1)
    assert np.array_equal(SR, S1) and np.array_equal(muR, mu1)


@pytest.mark.parametrize("p,kernel", [(1, 0), (2, 0), (1, 1), (2, 1)])
def test_adjoint_moments_vs_oracle_and_forward(dg, orc, cfg, p, kernel):
    """opts.adjoint = 1 (round 2): every source's moments from ONE group of
    weight fields stepped with the transposed operator (m_s = (P(dt L^T)^N
    w_s)^T u0_s), on the ring kernel with transposed tables and the sources'
    domain of dependence (kernel 0) or the v1 table kernel (kernel 1).
    Against O1 on c1 and a random walled mask (all sources), and against the
    per-source GPU solve on the c3 substrate (128 sources): per-source moments
    and Sigma within the fp64 tolerances."""
    t = TOL[64]
    m = cfg.mask("c1")
    src = cfg.sources("c1")
    c = cfg.CONFIGS["c1"]
    dt = c.dt if p == 1 else 1 / 128
    ref = orc.solve(p, 1.0, 1.0, m, src, dt, c.nsteps)
    with dg.Solver(m, 1.0, 1.0, p, adjoint=1, kernel=kernel) as s:
        s.solve(src, dt, c.nsteps)
        S, mu = s.covariance()
        mom = s.moments()
    assert mom_err(mom, ref) <= t["mom"]
    rng = np.random.default_rng(90 + p)
    mk = (rng.random((30, 34)) < 0.35).astype(np.uint8)
    free = np.argwhere(mk == 0)
    pick = free[rng.integers(0, len(free), 70)]
    srcs = np.stack([pick[:, 1], pick[:, 0]], 1).astype(np.int32)
    ref = orc.solve(p, 0.8, 1.3, mk, srcs, dt * 0.64 / 1.3, 60)
    with dg.Solver(mk, 0.8, 1.3, p, adjoint=1, kernel=kernel) as s:
        s.solve(srcs, dt * 0.64 / 1.3, 60)
        S, mu = s.covariance()
        mom = s.moments()
    assert mom_err(mom, ref) <= t["mom"]
    R, _ = orc.sigma(ref)
    assert sig_err(S, R) <= t["sig"]
    m3 = cfg.mask("c3")
    src3 = cfg.sources("c3")[:128]
    with dg.Solver(m3, 1.0, 1.0, p) as s:
        s.solve(src3, dt, 100)
        S0, _ = s.covariance()
        M0 = s.moments()
    with dg.Solver(m3, 1.0, 1.0, p, adjoint=1, kernel=kernel) as s:
        s.solve(src3, dt, 100)
        S1, _ = s.covariance()
        M1 = s.moments()
    assert mom_err(M1, M0) <= t["mom"]
    assert sig_err(S1, S0) <= t["sig"]


@pytest.mark.parametrize("p", [1, 2])
def test_adjoint_moments_subpixel_points_vs_oracle(dg, orc, p):
    """opts.adjoint with N4 sub-pixel point sources (R21): each point's
    moments are its evolved weight fields read against the point's
    projected-Dirac row, re-centred on the point; against O1's
    solve_points."""
    rng = np.random.default_rng(610 + p)
    ny, nx = 26, 30
    m = (rng.random((ny, nx)) < 0.3).astype(np.uint8)
    free = np.argwhere(m == 0)
    pick = free[rng.integers(0, len(free), 40)]
    loc = rng.random((40, 2))
    loc[0] = (0.3, 0.3)
    loc[1] = (0.0, 0.6)
    h = 0.8
    pts = (np.stack([pick[:, 1], pick[:, 0]], 1) + loc) * h
    dt = (1 / 32 if p == 1 else 1 / 128) * h * h
    ref = orc.solve_points(p, h, 1.0, m, pts, dt, 40)
    with dg.Solver(m, h, 1.0, p, adjoint=1) as s:
        s.solve_points(pts, dt, 40)
        S, mu = s.covariance()
        mom = s.moments()
    t = TOL[64]
    assert mom_err(mom, ref) <= t["mom"]
    R, _ = orc.sigma(ref)
    assert sig_err(S, R) <= t["sig"]


def test_adjoint_logical_ranks_bitwise(dg, cfg):
    """Adjoint moments under logical ranks: the origin lattice spans the whole
    batch, so the summed R-rank tables and Sigma equal one rank bit for bit."""
    m = cfg.mask("c3")
    src = cfg.sources("c3")[:300]
    with dg.Solver(m, 1.0, 1.0, 1, adjoint=1) as s:
        s.solve(src, 1 / 32, 24)
        S1, mu1 = s.covariance()
        M1 = s.moments()
    for R in (2, 4):
        tab = np.zeros_like(M1)
        for r in range(R):
            with dg.Solver(m, 1.0, 1.0, 1, adjoint=1, rank=r, nranks=R) as s:
                s.solve(src, 1 / 32, 24)
                tab += s.moments()
                if r == R - 1:
                    SR, muR = s.covariance_table(tab)
        assert np.array_equal(tab, M1), R
        assert np.array_equal(SR, S1) and np.array_equal(muR, mu1), R


def test_adjoint_on_fp32_handle_is_fp64_accurate(dg, orc, cfg):
    """An fp32 handle with adjoint = 1 steps the (fp64) weight fields: its
    moments meet the fp64 tolerance against O1, not only the fp32 one."""
    rng = np.random.default_rng(77)
    mk = (rng.random((28, 31)) < 0.35).astype(np.uint8)
    free = np.argwhere(mk == 0)
    pick = free[rng.integers(0, len(free), 50)]
    srcs = np.stack([pick[:, 1], pick[:, 0]], 1).astype(np.int32)
    for p, dt in ((1, 1 / 32), (2, 1 / 128)):
        ref = orc.solve(p, 1.0, 1.0, mk, srcs, dt, 50)
        with dg.Solver(mk, 1.0, 1.0, p, precision=32, adjoint=1) as s:
            s.solve(srcs, dt, 50)
            S, mu = s.covariance()
            mom = s.moments()
        assert mom_err(mom, ref) <= TOL[64]["mom"], p
        R, _ = orc.sigma(ref)
        assert sig_err(S, R) <= TOL[64]["sig"], p


@pytest.mark.parametrize("p", [1, 2])
def test_adjoint_moments_quads_vs_oracle(dg, orc, p):
    """opts.adjoint for N4 quadrilaterals: the transposed 9-point cross (the
    face block's variant follows the pixel two steps on) on the ring kernel,
    against O1's quad path on a random walled mask."""
    rng = np.random.default_rng(820 + p)
    mk = (rng.random((27, 31)) < 0.35).astype(np.uint8)
    free = np.argwhere(mk == 0)
    pick = free[rng.integers(0, len(free), 45)]
    srcs = np.stack([pick[:, 1], pick[:, 0]], 1).astype(np.int32)
    h, D = 0.8, 1.4
    dt = (1 / 16 if p == 1 else 1 / 64) * h * h / D
    ref = orc.q_solve(p, h, D, mk, srcs, dt, 40)
    with dg.Solver(mk, h, D, p, element=1, adjoint=1) as s:
        s.solve(srcs, dt, 40)
        S, mu = s.covariance()
        mom = s.moments()
    t = TOL[64]
    assert mom_err(mom, ref) <= t["mom"]
    R, _ = orc.sigma(ref)
    assert sig_err(S, R) <= t["sig"]
