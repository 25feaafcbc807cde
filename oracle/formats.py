"""numpy restatement of the format converters -- TEST INFRASTRUCTURE.

Only tests/ may use this module, as the checker of libkbgrid's kb_formats.cu.
The reference's band pipeline is SPEC-only (no code in /root/reference/proj),
so these follow the SPEC text directly; its worked examples are the known
answers (tests/test_formats_oracle.py):

* RealSpaceOperator: dense n x n block per R.
* bloch_transform: M(k) = sum_R exp(+2 pi i k.R) M_R.
* density_matrices folding: rho(R) = sum_k w_k exp(-2 pi i k.R) rho_k
  (SPEC.md:275-283).

Pair lists are generic: (pair_a, pair_b, pair_R, pair_off) plus the orbital
count of every atom; pair p's block is row-major norb[a] x norb[b] at
pair_off[p]. Sums run in pair order (over R) and k order, like the GPU.
"""
from __future__ import annotations

import numpy as np


def orbital_offsets(norb) -> np.ndarray:
    return np.concatenate([[0], np.cumsum(np.asarray(norb, dtype=np.int64))])


def offsets(pair_R) -> np.ndarray:
    """Distinct R, sorted lexicographically (kbg_offsets)."""
    R = np.asarray(pair_R, dtype=np.int64).reshape(-1, 3)
    return np.array(sorted({tuple(r) for r in R}), dtype=np.int64).reshape(-1, 3)


def _blocks(pairs, pair_a, pair_b, pair_off, norb):
    for p in range(len(pair_a)):
        na, nb = norb[pair_a[p]], norb[pair_b[p]]
        yield p, pairs[pair_off[p]:pair_off[p + 1]].reshape(na, nb)


def to_realspace(pairs, pair_a, pair_b, pair_R, pair_off, norb) -> np.ndarray:
    off = orbital_offsets(norb)
    Rs = [tuple(r) for r in offsets(pair_R)]
    rid = {r: i for i, r in enumerate(Rs)}
    R = np.asarray(pair_R).reshape(-1, 3)
    out = np.zeros((len(Rs), off[-1], off[-1]))
    for p, blk in _blocks(pairs, pair_a, pair_b, pair_off, norb):
        a, b = pair_a[p], pair_b[p]
        out[rid[tuple(R[p])], off[a]:off[a + 1], off[b]:off[b + 1]] = blk
    return out


def bloch(pairs, pair_a, pair_b, pair_R, pair_off, norb, k) -> np.ndarray:
    """M(k) = sum_R exp(+2 pi i k.R) M_R, one k (fractional)."""
    off = orbital_offsets(norb)
    R = np.asarray(pair_R, dtype=np.float64).reshape(-1, 3)
    k = np.asarray(k, dtype=np.float64)
    out = np.zeros((off[-1], off[-1]), dtype=np.complex128)
    for p, blk in _blocks(pairs, pair_a, pair_b, pair_off, norb):
        a, b = pair_a[p], pair_b[p]
        th = 2.0 * np.pi * (k[0] * R[p, 0] + k[1] * R[p, 1] + k[2] * R[p, 2])
        out[off[a]:off[a + 1], off[b]:off[b + 1]] += (np.cos(th) + 1j * np.sin(th)) * blk
    return out


def fold(rho_k, kpts, w, pair_a, pair_b, pair_R, pair_off, norb):
    """rho(R) = sum_k w_k exp(-2 pi i k.R) rho_k, restricted to the pair list.
    Returns (real part as pair values, max |imaginary part|)."""
    off = orbital_offsets(norb)
    R = np.asarray(pair_R, dtype=np.float64).reshape(-1, 3)
    kpts = np.asarray(kpts, dtype=np.float64).reshape(-1, 3)
    re = np.zeros(pair_off[-1])
    im = np.zeros(pair_off[-1])
    for p in range(len(pair_a)):
        a, b = pair_a[p], pair_b[p]
        acc = np.zeros((off[a + 1] - off[a], off[b + 1] - off[b]), dtype=np.complex128)
        for k in range(len(kpts)):
            th = 2.0 * np.pi * (kpts[k] @ R[p])
            acc += w[k] * (np.cos(th) - 1j * np.sin(th)) * rho_k[k, off[a]:off[a + 1], off[b]:off[b + 1]]
        re[pair_off[p]:pair_off[p + 1]] = acc.real.ravel()
        im[pair_off[p]:pair_off[p + 1]] = acc.imag.ravel()
    return re, float(np.abs(im).max()) if len(im) else 0.0
