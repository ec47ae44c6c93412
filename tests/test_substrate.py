"""Row a0 (G1): the seeded Gamma-axon substrate and source generators
(readings R11, R16, R17).

Checked against brute force and the definitions, not against the generator:
non-overlap of every disk pair, radius bounds, the rasterisation rule
re-derived pixel by pixel from the circle list, the target fraction, seed
determinism, the source box and its extracellular-only support, and the
SPEC text-format round trip.
"""
import math

import numpy as np
import pytest

from paper_1907_06191_b200 import configs, substrate as G


@pytest.fixture(scope="module")
def sub():
    return G.gen_substrate(160, 144, 0.55, seed=17)


def test_disks_do_not_overlap_and_radii_are_bounded(sub):
    c = sub.circles
    assert len(c) > 50
    assert (c[:, 2] >= G.RMIN_UM - 1e-15).all() and (c[:, 2] <= G.RMAX_UM + 1e-15).all()
    d = np.hypot(c[:, None, 0] - c[None, :, 0], c[:, None, 1] - c[None, :, 1])
    rr = c[:, None, 2] + c[None, :, 2]
    iu = np.triu_indices(len(c), 1)
    assert (d[iu] >= rr[iu] - 1e-12).all()          # brute force over all pairs
    L = np.array([160, 144]) * sub.h_um
    assert (c[:, 0] >= 0).all() and (c[:, 0] < L[0]).all() and (c[:, 1] >= 0).all() and (c[:, 1] < L[1]).all()


def test_mask_is_the_pixel_centre_rasterisation(sub):
    """R16: pixel (i, j) is axon iff its centre lies in some closed disk."""
    ny, nx = sub.mask.shape
    h = sub.h_um
    X, Y = np.meshgrid((np.arange(nx) + 0.5) * h, (np.arange(ny) + 0.5) * h)
    ref = np.zeros((ny, nx), bool)
    for x, y, r in sub.circles:
        ref |= (X - x) ** 2 + (Y - y) ** 2 <= r * r
    assert np.array_equal(sub.mask.astype(bool), ref)


def test_fraction_reaches_target_and_seeded(sub):
    assert 0.55 <= sub.fraction < 0.55 + 0.02       # stops at the first disk past the target
    again = G.gen_substrate(160, 144, 0.55, seed=17)
    assert np.array_equal(again.mask, sub.mask) and np.array_equal(again.circles, sub.circles)
    other = G.gen_substrate(160, 144, 0.55, seed=18)
    assert not np.array_equal(other.mask, sub.mask)


def test_largest_first_within_each_batch(sub):
    """RSA places radii largest first: the first batch is non-increasing."""
    r = sub.circles[:, 2]
    n0 = max(1, int(0.5 * len(r)))
    assert (np.diff(r[:n0]) <= 1e-15).all()


def test_gamma_radii_fit_the_paper_extremes():
    """R17: shape 11.27, scale 0.0446 um make 0.150 / 1.141 um the expected
    min / max of 1901 draws, to within sampling noise."""
    mins, maxs = [], []
    for s in range(40):
        r = np.random.default_rng(s).gamma(G.GAMMA_SHAPE, G.GAMMA_SCALE_UM, size=1901)
        mins.append(r.min())
        maxs.append(r.max())
    assert abs(np.mean(mins) - 0.150) < 0.02 and abs(np.mean(maxs) - 1.141) < 0.08
    r = G.sample_radii(10000, 3)
    assert r.min() >= G.RMIN_UM and r.max() <= G.RMAX_UM
    assert abs(r.mean() - G.GAMMA_SHAPE * G.GAMMA_SCALE_UM) < 0.01


def test_sources_uniform_in_the_centred_box_and_extracellular(sub):
    """R11: pixel-centre sources, uniform over the unmasked pixels of the
    centred box of side ceil(0.4 n), with replacement."""
    m = sub.mask
    ny, nx = m.shape
    src = G.sample_sources(m, 20000, seed=5)
    bx, by = math.ceil(0.4 * nx), math.ceil(0.4 * ny)
    x0, y0 = (nx - bx) // 2, (ny - by) // 2
    assert (src[:, 0] >= x0).all() and (src[:, 0] < x0 + bx).all()
    assert (src[:, 1] >= y0).all() and (src[:, 1] < y0 + by).all()
    assert not m[src[:, 1], src[:, 0]].any()
    free = np.count_nonzero(m[y0:y0 + by, x0:x0 + bx] == 0)
    counts = np.bincount(src[:, 1] * nx + src[:, 0], minlength=nx * ny)
    hit = counts[counts > 0]
    assert len(hit) == free or len(hit) > 0.98 * free        # every free pixel is reachable
    assert abs(hit.mean() - 20000 / free) < 1e-9 * 20000     # mean count = n / free pixels
    assert np.array_equal(G.sample_sources(m, 100, seed=5), src[:100])


def test_text_format_round_trip(sub, tmp_path):
    p = tmp_path / "sub.txt"
    G.save_substrate(p, sub)
    c = G.load_circles(p)
    assert np.array_equal(c, sub.circles)
    assert p.read_text().startswith("# substrate side=")


def test_configs_c1_c2_shapes():
    m1 = configs.mask("c1")
    assert m1.shape == (32, 32) and m1[16, 16] == 1 and m1[16, 4] == 0
    c = (np.arange(32) + 0.5)
    X, Y = np.meshgrid(c, c)
    assert np.array_equal(m1, (((X - 16) ** 2 + (Y - 16) ** 2) <= 64).astype(np.uint8))
    m2 = configs.mask("c2")
    assert m2.shape == (256, 256) and not m2.any()
    s2 = configs.sources("c2")
    assert len(s2) == 1024 and s2.min() == 97 and s2.max() == 159
