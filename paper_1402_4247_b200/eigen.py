"""Eigen_HH on the GPU: the reference kband eigensolver's pieces, host-side mirror.

kband API (/root/reference/proj/include/kband/householder.hpp:56-82) -> this module:
  tridiagonalize(HermitianMatrix, plan)     -> tridiagonalize(a, fault_proc6_sign=False)   [GPU]
  back_transform(records, Y)                -> back_transform(records, y)                  [GPU]
  normalize_columns(C)                      -> normalize_columns(c)                         [GPU]
  eigen_hh(a, want_vectors)                 -> eigen_hh(a, want_vectors, solve_tridiag=...)
The tridiagonal QL solve between the GPU steps runs on the host, as in the paper (LAPACK
dstevx/dstegr/dstedc on the CPUs): the default is scipy's LAPACK stemr
(scipy.linalg.eigh_tridiagonal); callers inside kband pass kband::solve_tridiag.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _abi
from .errors import DimensionError, raise_for_status


@dataclass
class HouseholderRecords:
    """Stage records (householder.hpp:44-51), stacked: u (n-1, n) complex, h, s (n-1,), phase (n-1,) complex."""

    u: np.ndarray
    h: np.ndarray
    s: np.ndarray
    phase: np.ndarray


@dataclass
class TridiagReal:
    d: np.ndarray
    e: np.ndarray
    records: HouseholderRecords


def _lib():
    return _abi.kbgrid()


def _check(st: int, what: str) -> None:
    if st:
        raise_for_status(st, what, _lib().kbg_hh_last_error().decode())


def _cptr(a: np.ndarray):
    assert a.dtype == np.complex128 and a.flags.c_contiguous
    return a.ctypes.data_as(_abi._DP)


def tridiagonalize(a: np.ndarray, fault_proc6_sign: bool = False) -> TridiagReal:
    a = np.ascontiguousarray(a, dtype=np.complex128)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise DimensionError(f"tridiagonalize: matrix not square {a.shape}")
    n = a.shape[0]
    nr = max(n - 1, 0)
    d = np.empty(n)
    e = np.empty(max(nr, 1))
    u = np.empty((max(nr, 1), n), dtype=np.complex128)
    h = np.empty(max(nr, 1))
    s = np.empty(max(nr, 1))
    ph = np.empty(max(nr, 1), dtype=np.complex128)
    _check(_lib().kbg_hh_tridiagonalize(n, _cptr(a), int(fault_proc6_sign), _abi.dptr(d), _abi.dptr(e), _cptr(u),
                                        _abi.dptr(h), _abi.dptr(s), _cptr(ph)), "kbg_hh_tridiagonalize")
    return TridiagReal(d, e[:nr], HouseholderRecords(u[:nr], h[:nr], s[:nr], ph[:nr]))


def back_transform(records: HouseholderRecords, y: np.ndarray) -> np.ndarray:
    y = np.ascontiguousarray(y, dtype=np.float64)
    n, m = y.shape
    if records.u.shape != (max(n - 1, 0), n):
        raise DimensionError(f"back_transform: records {records.u.shape} do not match matrix dimension {n}")
    if n == 1:
        return y.astype(np.complex128)
    w = np.empty((n, m), dtype=np.complex128)
    u = np.ascontiguousarray(records.u, dtype=np.complex128)
    h = np.ascontiguousarray(records.h, dtype=np.float64)
    ph = np.ascontiguousarray(records.phase, dtype=np.complex128)
    _check(_lib().kbg_hh_back_transform(n, m, _cptr(u), _abi.dptr(h), _cptr(ph), _abi.dptr(y), _cptr(w)),
           "kbg_hh_back_transform")
    return w


def normalize_columns(c: np.ndarray) -> np.ndarray:
    c = np.array(c, dtype=np.complex128, order="C", copy=True)
    _check(_lib().kbg_hh_normalize_columns(c.shape[0], c.shape[1], _cptr(c)), "kbg_hh_normalize_columns")
    return c


def triple_product(t: np.ndarray, h: np.ndarray) -> np.ndarray:
    """kband::triple_product (Part 3): T^H H T, re-symmetrized and validated Hermitian (GPU ZGEMMs)."""
    t = np.ascontiguousarray(t, dtype=np.complex128)
    h = np.ascontiguousarray(h, dtype=np.complex128)
    n, m = t.shape
    if h.shape != (n, n):
        raise DimensionError("triple_product: T rows must match H dim")
    c = np.empty((m, m), dtype=np.complex128)
    _check(_lib().kbg_hh_triple_product(n, m, _cptr(t), _cptr(h), _cptr(c)), "kbg_hh_triple_product")
    return c


def lapack_solve_tridiag(d: np.ndarray, e: np.ndarray, want_vectors: bool):
    """Host tridiagonal eigensolver (LAPACK via scipy), the paper's CPU step."""
    from scipy.linalg import eigh_tridiagonal

    if len(d) == 1:
        return d.copy(), (np.ones((1, 1)) if want_vectors else None)
    if want_vectors:
        w, z = eigh_tridiagonal(d, e, lapack_driver="stemr")
        return w, z
    return eigh_tridiagonal(d, e, eigvals_only=True, lapack_driver="stemr"), None


def gpu_solve_tridiag(d: np.ndarray, e: np.ndarray, want_vectors: bool):
    """kband::solve_tridiag on the GPU (kbg_tridiag_solve: Sturm multisection + inverse iteration):
    (eigenvalues ascending, eigenvectors as columns or None)."""
    d = np.ascontiguousarray(d, dtype=np.float64)
    e = np.ascontiguousarray(e, dtype=np.float64)
    n = len(d)
    if len(e) + 1 != n:
        raise DimensionError("solve_tridiag: off-diagonal length must be n-1")
    w = np.empty(n)
    z = np.empty((n, n)) if want_vectors else None
    ee = e if n > 1 else np.zeros(1)
    _check(_lib().kbg_tridiag_solve(n, _abi.dptr(d), _abi.dptr(ee), int(want_vectors), _abi.dptr(w),
                                    _abi.dptr(z) if want_vectors else None), "kbg_tridiag_solve")
    return w, z


def eigen_hh(a: np.ndarray, want_vectors: bool = True, solve_tridiag=None):
    """kband::eigen_hh (householder.cpp:333-351). Default: the whole pipeline on the GPU, device-resident
    (kbg_hh_eigen: tridiagonalize -> GPU tridiagonal solve -> back transform -> normalization). With a host
    `solve_tridiag` (e.g. lapack_solve_tridiag, the paper's CPU step): GPU tridiagonalize -> that solver ->
    GPU back transform + normalization. Returns (eigenvalues ascending, eigenvectors as columns or None)."""
    if solve_tridiag is None:
        a = np.ascontiguousarray(a, dtype=np.complex128)
        n = a.shape[0]
        if a.ndim != 2 or a.shape[1] != n:
            raise DimensionError(f"eigen_hh: matrix not square {a.shape}")
        w = np.empty(n)
        c = np.empty((n, n), dtype=np.complex128) if want_vectors else None
        _check(_lib().kbg_hh_eigen(n, _cptr(a), int(want_vectors), _abi.dptr(w), _cptr(c) if want_vectors else None),
               "kbg_hh_eigen")
        return w, c
    t = tridiagonalize(a)
    w, z = solve_tridiag(t.d, t.e, want_vectors)
    if not want_vectors:
        return np.asarray(w), None
    return np.asarray(w), normalize_columns(back_transform(t.records, np.ascontiguousarray(z)))


__all__ = ["HouseholderRecords", "TridiagReal", "tridiagonalize", "back_transform", "normalize_columns", "triple_product",
           "lapack_solve_tridiag", "gpu_solve_tridiag", "eigen_hh"]
