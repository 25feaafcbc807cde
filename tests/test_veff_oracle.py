"""CPU: the numpy V_eff restatement (oracle/veff.py) against analytic cases."""
import numpy as np
import pytest

from oracle import veff as V

LAT = np.array([[6.0, 0.0, 0.0], [1.0, 5.0, 0.0], [0.5, 0.7, 7.0]])
N = (12, 10, 14)


def grid_points():
    f = np.stack(np.meshgrid(*[np.arange(n) / n for n in N], indexing="ij"), -1)
    return f @ LAT


@pytest.mark.parametrize("m", [(1, 0, 0), (0, 2, 1), (1, -1, 3)])
def test_hartree_of_a_plane_wave(m):
    """rho = rho0 + A cos(G.r) -> V_H = 4 pi A cos(G.r) / |G|^2 (the constant is the neutralized G = 0)."""
    B = V.reciprocal(LAT)
    G = 2 * np.pi * (m[0] * B[0] + m[1] * B[1] + m[2] * B[2])
    r = grid_points()
    rho = 0.3 + 0.1 * np.cos(r @ G)
    vh = V.hartree(rho, LAT)
    assert np.abs(vh - 4 * np.pi * 0.1 * np.cos(r @ G) / (G @ G)).max() <= 1e-13


def test_uniform_density_exchange():
    rho = np.full((1, int(np.prod(N))), 0.02)
    v, (eh, ex) = V.veff(rho, LAT, N)
    assert np.abs(v + (3 * 0.02 / np.pi) ** (1 / 3)).max() <= 1e-15
    vol = abs(np.linalg.det(LAT))
    assert abs(eh) <= 1e-14
    assert abs(ex - (-0.75 * (3 / np.pi) ** (1 / 3) * 0.02 ** (4 / 3) * vol)) <= 1e-12 * abs(ex)


def test_spin_split_equals_unpolarized():
    rng = np.random.default_rng(3)
    rho = rng.uniform(0.0, 0.1, (1, int(np.prod(N))))
    v1, e1 = V.veff(rho, LAT, N)
    v2, e2 = V.veff(np.concatenate([rho / 2, rho / 2]), LAT, N)
    assert np.abs(v2[0] - v1[0]).max() <= 1e-14 and np.abs(v2[1] - v1[0]).max() <= 1e-14
    assert np.allclose(e1, e2, rtol=1e-13)


def test_pw92_published_value():
    """PW92 paramagnetic correlation at rs = 1 and 2 (Hartree): -0.0598 and -0.0448."""
    for rs, ref in ((1.0, -0.0598), (2.0, -0.0448)):
        n = 3.0 / (4.0 * np.pi * rs ** 3)
        eps, vu, vd = V.pw92(n, 0.0)
        assert abs(eps - ref) <= 5e-4, (rs, eps)
        assert vu == vd


@pytest.mark.parametrize("zeta", [0.0, 0.3, -0.7, 1.0])
def test_pw92_potential_is_the_derivative(zeta):
    """v_c,s = d(n eps_c)/d rho_s, central finite differences in rho_up and rho_down."""
    n = 0.037
    up, dn = n * (1 + zeta) / 2, n * (1 - zeta) / 2

    def energy(u, d):
        t = u + d
        return t * V.pw92(t, (u - d) / t)[0]

    _, vu, vd = V.pw92(n, zeta)
    h = 1e-6 * n
    fu = (energy(up + h, dn) - energy(up - h, dn)) / (2 * h)
    assert abs(fu - vu) <= 1e-7 * abs(vu)
    if zeta < 1.0:
        fd = (energy(up, dn + h) - energy(up, dn - h)) / (2 * h)
        assert abs(fd - vd) <= 1e-7 * abs(vd)


def test_lda_spin_split_equals_unpolarized():
    rng = np.random.default_rng(5)
    rho = rng.uniform(0.0, 0.1, (1, int(np.prod(N))))
    v1, e1 = V.veff(rho, LAT, N, xc=1)
    v2, e2 = V.veff(np.concatenate([rho / 2, rho / 2]), LAT, N, xc=1)
    assert np.abs(v2[0] - v1[0]).max() <= 1e-13 and np.abs(v2[1] - v1[0]).max() <= 1e-13
    assert np.allclose(e1, e2, rtol=1e-13)
