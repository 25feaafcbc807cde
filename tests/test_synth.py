"""Synthetic Fe3O4 generator (G0): geometry, grid rule, basis, inputs."""
import numpy as np
import pytest

from paper_1402_4247_b200 import _abi
from paper_1402_4247_b200.system import Fe3O4, good_size, radial_table

BOHR = 0.529177210903


def test_grid_rule(built):
    assert good_size(44) == 45 and good_size(71) == 72 and good_size(143) == 144 and good_size(7) == 8
    assert Fe3O4.config("cubic56_200Ry").system.grid == (72, 72, 72)
    assert Fe3O4.config("sweep56_250Ry").system.npts == 512_000  # the paper's 512,000
    assert Fe3O4.config("sweep56_100Ry").system.grid == (54, 54, 54)


def test_magnetite_geometry(built):
    s = Fe3O4.config("cubic56_200Ry").system
    assert s.natom == 56 and (s.species_of_atom == 0).sum() == 24
    L = s.lattice[0, 0]
    fe, ox = s.tau[s.species_of_atom == 0], s.tau[s.species_of_atom == 1]
    d = fe[:, None, :] - ox[None, :, :]
    d -= L * np.round(d / L)
    r = np.sqrt((d ** 2).sum(-1)) * BOHR
    near = np.sort(r, axis=1)
    tet, octa = near[:8], near[8:]  # 8a sites first in canonical order
    assert np.allclose(tet[:, :4], 1.889, atol=2e-3) and np.all(tet[:, 4] > 3.0)
    assert np.allclose(octa[:, :6], 2.059, atol=2e-3)


def test_primitive_cell(built):
    s = Fe3O4.config("primitive14_150Ry").system
    assert s.natom == 14 and s.nbasis == 142
    assert abs(abs(np.linalg.det(s.lattice)) - (8.396 / BOHR) ** 3 / 4) < 1e-9


def test_radial_normalisation(built):
    tab = radial_table(1, 0.6, 6.0, 4001)
    r = np.linspace(0, 6.0, 4001)
    R = tab[:, 0] * r  # l = 1
    f = R * R * r * r
    h = r[1] - r[0]
    integral = h / 3 * (f[0] + f[-1] + 4 * f[1:-1:2].sum() + 2 * f[2:-1:2].sum())
    assert abs(integral - 1.0) < 1e-9
    # derivative column is du/dr
    assert np.allclose(np.gradient(tab[:, 0], h)[5:-5], tab[5:-5, 1], rtol=0, atol=1e-5)


def test_inputs_deterministic_and_symmetric(built):
    from oracle.oracle import Oracle

    f1 = Fe3O4.config("primitive14_150Ry")
    f2 = Fe3O4.config("primitive14_150Ry")
    ix = Oracle(f1.system).build_index()
    d1, d2 = f1.dm(ix, nspin=2), f2.dm(ix, nspin=2)
    assert np.array_equal(d1, d2)
    assert not np.array_equal(d1[0], d1[1])
    assert np.array_equal(f1.veff(2), f2.veff(2))
    norb = f1.system.norb_of_atom()
    off = ix["pair_off"]
    for p, q in enumerate(ix["pair_mirror"]):
        na, nb = norb[ix["pair_a"][p]], norb[ix["pair_b"][p]]
        assert np.array_equal(d1[0, off[p]:off[p + 1]].reshape(na, nb), d1[0, off[q]:off[q + 1]].reshape(nb, na).T)


def test_bad_config(built):
    from paper_1402_4247_b200.errors import ConfigError

    with pytest.raises(ConfigError):
        Fe3O4(_abi.KBG_CELL_PRIMITIVE, 2, 150.0)
    with pytest.raises(ConfigError):
        Fe3O4(_abi.KBG_CELL_CUBIC, 1, -1.0)
