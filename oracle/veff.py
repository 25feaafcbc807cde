"""numpy restatement of V_eff from rho (kb_veff.cu) -- TEST INFRASTRUCTURE.

Only tests/ and tools/ reference legs use it. The reference has no code for this step (SPEC.md:9 puts
V_eff construction out of its scope); the formulas are the standard ones, pinned by analytic cases in
tests/test_veff_oracle.py: V_H(G) = 4 pi rho(G)/|G|^2 (G = 0 dropped), V_x,s = -(6 rho_s/pi)^(1/3);
xc=1 adds the Perdew-Wang 1992 LSDA correlation (Phys. Rev. B 45, 13244, Table I parameters, Hartree),
pinned by its published value at rs = 1 and by v_c,s = d(n eps_c)/d rho_s (finite differences).
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


# PW92 G(rs; A, alpha1, beta1..beta4), p = 1: eps_c(rs, 0), eps_c(rs, 1), -alpha_c(rs)
PW92 = ((0.031091, 0.21370, 7.5957, 3.5876, 1.6382, 0.49294),
        (0.015545, 0.20548, 14.1189, 6.1977, 3.3662, 0.62517),
        (0.016887, 0.11125, 10.357, 3.6231, 0.88026, 0.49671))
FZ0 = 1.709921  # f''(0)


def _pw92_g(rs, A, a1, b1, b2, b3, b4):
    """G and dG/drs."""
    sr = np.sqrt(rs)
    q0 = -2.0 * A * (1.0 + a1 * rs)
    q1 = 2.0 * A * (b1 * sr + b2 * rs + b3 * rs * sr + b4 * rs * rs)
    q1p = A * (b1 / sr + 2.0 * b2 + 3.0 * b3 * sr + 4.0 * b4 * rs)
    lg = np.log1p(1.0 / q1)
    return q0 * lg, -2.0 * A * a1 * lg - q0 * q1p / (q1 * q1 + q1)


def pw92(n, zeta):
    """eps_c, v_c,up, v_c,down of the PW92 LSDA correlation (Hartree) at density n, polarization zeta."""
    n = np.asarray(n, dtype=np.float64)
    zeta = np.clip(np.asarray(zeta, dtype=np.float64), -1.0, 1.0)
    rs = np.cbrt(3.0 / (4.0 * np.pi * n))
    ec0, d0 = _pw92_g(rs, *PW92[0])
    ec1, d1 = _pw92_g(rs, *PW92[1])
    ma, dma = _pw92_g(rs, *PW92[2])  # -alpha_c
    ac, dac = -ma, -dma
    c43 = 2.0 ** (4.0 / 3.0) - 2.0
    f = ((1 + zeta) ** (4 / 3) + (1 - zeta) ** (4 / 3) - 2.0) / c43
    fp = (4.0 / 3.0) * (np.cbrt(1 + zeta) - np.cbrt(1 - zeta)) / c43
    z3 = zeta ** 3
    z4 = z3 * zeta
    eps = ec0 + ac * f / FZ0 * (1 - z4) + (ec1 - ec0) * f * z4
    deps_rs = d0 + dac * f / FZ0 * (1 - z4) + (d1 - d0) * f * z4
    deps_z = ac / FZ0 * (fp * (1 - z4) - 4 * z3 * f) + (ec1 - ec0) * (fp * z4 + 4 * z3 * f)
    common = eps - rs / 3.0 * deps_rs - zeta * deps_z
    return eps, common + deps_z, common - deps_z


def veff(rho: np.ndarray, lattice, N, vloc=None, dV=None, xc: int = 0):
    """rho [nspin][npts] -> (veff [nspin][npts], (E_H, E_xc)); xc 0: Slater exchange only, 1: + PW92."""
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
    exc = -0.75 * np.cbrt(6.0 / np.pi) * ex_sum * dV
    if xc == 1:
        up, dn = (rs[0], rs[1]) if nspin == 2 else (rs[0], rs[0])
        n = up + dn
        live = n > 1e-30
        ns = np.where(live, n, 1.0)
        eps, vu, vd = pw92(ns, np.where(live, (up - dn) / ns, 0.0))
        eps, vu, vd = (np.where(live, x, 0.0) for x in (eps, vu, vd))
        v = v + (np.stack([vu, vd]) if nspin == 2 else vu[None, :])
        exc += (n * eps).sum() * dV
    e = (0.5 * (vh * rho.sum(0)).sum() * dV, exc)
    return v, e
