"""Pins of the Monte-Carlo reference walk (oracle/mc.py): the generator's
known-answer vectors, exact step lengths, no walker ever inside an axon, and
the free-space mean-square displacement T l^2 (l = sqrt(4 D t_s / T))."""
import numpy as np
import pytest

from oracle import mc


@pytest.mark.parametrize("ctr,key,out", [
    ((0, 0, 0, 0), (0, 0), (0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8)),
    ((0xffffffff,) * 4, (0xffffffff, 0xffffffff), (0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd)),
    ((0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344), (0xa4093822, 0x299f31d0),
     (0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1)),
])
def test_philox_known_answers(ctr, key, out):
    """Philox4x32-10 known-answer vectors (Salmon et al., SC'11 / Random123)."""
    c = mc.philox4x32_10(*[np.array([v], np.uint32) for v in ctr], np.array([key[0]], np.uint32),
                         np.array([key[1]], np.uint32))
    assert tuple(int(v[0]) for v in c) == out


def test_one_free_step_has_length_l():
    d = mc.walk(np.zeros((10, 10), np.uint8), [(5, 5)], 300, 1, 0.7, 3)
    assert np.allclose(np.hypot(d[:, 0], d[:, 1]), 0.7, rtol=0, atol=1e-14)


def test_free_msd_and_walls():
    T, l = 60, 0.5
    d = mc.walk(np.zeros((40, 40), np.uint8), [(20, 20)], 4000, T, l, 11)
    msd = (d ** 2).sum(axis=1)
    se = msd.std() / np.sqrt(len(msd))
    assert abs(msd.mean() - T * l * l) < 4 * se
    rng = np.random.default_rng(2)
    mask = (rng.random((20, 20)) < 0.4).astype(np.uint8)
    mask[10, 10] = 0
    d = mc.walk(mask, [(10, 10)], 300, 80, 0.6, 5)
    fx, fy = np.floor(10.5 + d[:, 0]).astype(int), np.floor(10.5 + d[:, 1]).astype(int)
    assert not mask[fy, fx].any()
