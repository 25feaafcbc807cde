"""GPU V_eff from rho (kb_veff.cu) vs the numpy restatement (oracle/veff.py): the rho of
the GPU grid pass, nspin 1 and 2, with V_loc; V_eff within 1e-12 of max|V|, energies within 1e-12
relative; plus the plane-wave Hartree case on the Fe3O4 lattice."""
import numpy as np
import pytest

from oracle import veff as V
from paper_1402_4247_b200.grid import GridPass
from paper_1402_4247_b200.system import Fe3O4

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def setup(built):
    f = Fe3O4.config("primitive14_150Ry")
    gp = GridPass(f.system)
    ix = gp.build_index()
    dm = f.dm(ix)
    rho = gp.density(dm)
    lat = np.asarray(f.system.lattice).reshape(3, 3)
    return f, gp, rho, lat, tuple(f.system.grid)


def test_veff_parity_unpolarized(setup):
    f, gp, rho, lat, N = setup
    rho = np.abs(rho)  # a physical (non-negative) density of the grid-pass shape
    vloc = f.veff()[0]
    v, e = gp.veff(rho, vloc)
    rv, re = V.veff(rho, lat, N, vloc)
    assert np.abs(v - rv).max() <= 1e-12 * np.abs(rv).max()
    assert abs(e[0] - re[0]) <= 1e-12 * abs(re[0]) and abs(e[1] - re[1]) <= 1e-12 * abs(re[1])


def test_veff_parity_spin(setup):
    f, gp, rho, lat, N = setup
    r2 = np.concatenate([0.6 * np.abs(rho), 0.4 * np.abs(rho)])
    v, e = gp.veff(r2)
    rv, re = V.veff(r2, lat, N)
    assert np.abs(v - rv).max() <= 1e-12 * np.abs(rv).max()
    assert abs(e[1] - re[1]) <= 1e-12 * abs(re[1])


def test_plane_wave_hartree_on_the_cell(setup):
    f, gp, rho, lat, N = setup
    B = V.reciprocal(lat)
    G = 2 * np.pi * (1 * B[0] + 2 * B[1] - 1 * B[2])
    fr = np.stack(np.meshgrid(*[np.arange(n) / n for n in N], indexing="ij"), -1).reshape(-1, 3) @ lat
    cosg = np.cos(fr @ G)
    test = (0.05 + 0.01 * cosg)[None]
    v, _ = gp.veff(test)
    vx = -(3 * test[0] / np.pi) ** (1 / 3)
    assert np.abs(v[0] - vx - 4 * np.pi * 0.01 * cosg / (G @ G)).max() <= 1e-12


@pytest.mark.parametrize("nspin", [1, 2])
def test_lda_pw92_parity(setup, nspin):
    """KBG_OPT_XC = 1: exchange + Perdew-Wang 1992 correlation, nspin 1 and 2 (polarized split)."""
    from paper_1402_4247_b200 import _abi

    f, gp, rho, lat, N = setup
    r = np.abs(rho) if nspin == 1 else np.concatenate([0.7 * np.abs(rho), 0.3 * np.abs(rho)])
    gp.set_option(_abi.KBG_OPT_XC, 1)
    try:
        v, e = gp.veff(r)
    finally:
        gp.set_option(_abi.KBG_OPT_XC, 0)
    rv, re = V.veff(r, lat, N, xc=1)
    assert np.abs(v - rv).max() <= 1e-12 * np.abs(rv).max()
    assert abs(e[1] - re[1]) <= 1e-12 * abs(re[1])
    vx, ex = V.veff(r, lat, N)  # correlation lowers V and E_xc
    assert (v <= vx + 1e-15).all() and e[1] < ex[1]
