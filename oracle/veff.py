"""numpy restatement of V_eff from rho (kb_veff.cu) -- TEST INFRASTRUCTURE.

Only tests/ and tools/ reference legs use it. The reference has no code for this step (SPEC.md:9 puts
V_eff construction out of its scope); the formulas are the standard ones, pinned by analytic cases in
tests/test_veff_oracle.py: V_H(G) = 4 pi rho(G)/|G|^2 (G = 0 dropped), V_x,s = -(6 rho_s/pi)^(1/3).
"""
from __future__ import annotations

import numpy as np


def reciprocal(lattice) -> np.ndarray:
    """Rows b_i with a_i . b_j = delta_ij (lattice rows a_i)."""
    return np.linalg.inv(np.asarray(lattice, dtype=np.float64).reshape(3, 3)).T


def hartree(rho_tot: np.ndarray, lattice) -> np.ndarray:
    N = rho_tot.shape
    B = reciprocal(lattice)
    f = np.fft.rfftn(rho_tot)
    m = [np.fft.fftfreq(N[0], 1.0 / N[0]), np.fft.fftfreq(N[1], 1.0 / N[1]), np.arange(N[2] // 2 + 1)]
    M0, M1, M2 = np.meshgrid(*m, indexing="ij")
    G = 2 * np.pi * (M0[..., None] * B[0] + M1[..., None] * B[1] + M2[..., None] * B[2])
    g2 = (G ** 2).sum(-1)
    g2[0, 0, 0] = 1.0
    v = 4 * np.pi * f / g2
    v[0, 0, 0] = 0.0
    return np.fft.irfftn(v, s=N, axes=(0, 1, 2))


def veff(rho: np.ndarray, lattice, N, vloc=None, dV=None):
    """rho [nspin][npts] -> (veff [nspin][npts], (E_H, E_x))."""
    rho = np.asarray(rho, dtype=np.float64)
    nspin = rho.shape[0]
    rt = rho.sum(0).reshape(N)
    vh = hartree(rt, lattice).ravel()
    rs = np.maximum(rho, 0.0) if nspin == 2 else np.maximum(rho, 0.0) * 0.5
    vx = -np.cbrt(6.0 / np.pi) * np.cbrt(rs)
    v = vh[None, :] + vx + (0.0 if vloc is None else np.asarray(vloc)[None, :])
    ex_sum = (rs * np.cbrt(rs)).sum() * (1.0 if nspin == 2 else 2.0)
    if dV is None:
        dV = abs(np.linalg.det(np.asarray(lattice).reshape(3, 3))) / np.prod(N)
    e = (0.5 * (vh * rho.sum(0)).sum() * dV, -0.75 * np.cbrt(6.0 / np.pi) * ex_sum * dV)
    return v, e
