"""The stored oracle answers (tests/golden/<cfg>_o1.npz, written by
tests/golden/gen_golden.py from oracle/ only) are consistent with their
inputs and with the oracle as it stands: seeded sources, pixel samples inside
the grid (axon pixels of the window hold exact zeros), exact mass, sample
coverage, and one c2 source recomputed by O1 bit for bit."""
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
NAMES = ["c2", "c3", "c4", "c5"]


def load(name):
    z = np.load(os.path.join(HERE, "golden", f"{name}_o1.npz"))
    return {k: z[k] for k in z.files}


@pytest.mark.parametrize("name", NAMES)
def test_fixture_inputs_and_invariants(name):
    from paper_1907_06191_b200 import configs
    g = load(name)
    batch = int(g["batch"])
    src = configs.sources(name, None if batch < 0 else batch)
    assert np.array_equal(src[g["idx"]], g["sources"])
    m = configs.mask(name)
    ny, nx = m.shape
    for r in range(len(g["idx"])):
        p = g["pix"][r]
        ok = p[:, 0] >= 0
        p, v = p[ok], g["dens"][r][ok]
        assert np.all((p[:, 0] < nx) & (p[:, 1] < ny))
        axon = m[p[:, 1], p[:, 0]] == 1                           # the window includes axon pixels:
        assert np.all(v[axon] == 0)                               # stasis, exact zeros
        assert np.abs(v[~axon]).max() > 0
        s = g["sources"][r]
        assert any((p[:, 0] == s[0]) & (p[:, 1] == s[1]))         # the source pixel is in the window
    assert np.abs(g["mom"][:, 0] - 1.0).max() <= 1e-12            # REFLECT: exact mass
    assert g["norm_frac"].min() >= 0.99
    assert int(g["degree"]) == configs.CONFIGS[name].degree
    assert float(g["dt"]) == configs.CONFIGS[name].dt


def test_fixture_reproduced_by_oracle(orc):
    """One c2 source (free space, 512 steps) recomputed now equals the stored
    moments and sampled coefficients exactly (the fixture is O1's output)."""
    from paper_1907_06191_b200 import configs
    g = load("c2")
    m = configs.mask("c2")
    mom, dens = orc.solve(1, 1.0, 1.0, m, g["sources"][:1], float(g["dt"]), int(g["nsteps"]), keep_density=True)
    assert np.array_equal(mom[0], g["mom"][0])
    p = g["pix"][0]
    p = p[p[:, 0] >= 0]
    assert np.array_equal(dens[0][p[:, 1], p[:, 0]].reshape(len(p), -1), g["dens"][0][:len(p)])
