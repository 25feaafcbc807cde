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
