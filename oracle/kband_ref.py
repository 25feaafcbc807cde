"""ctypes wrapper of oracle/_ref/libkband_ref.so -- TEST INFRASTRUCTURE.

The reference's own kband eigensolver (compiled from /root/reference/proj/src by `make -C oracle ref`,
see oracle/kband_ref_shim.cpp). Only tests/ and bench-style tools' reference legs use it, as the checker
and the timed CPU baseline of SURVEY.md 8(f1).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "_ref", "libkband_ref.so")

_I, _I64, _DP = C.c_int, C.c_int64, C.POINTER(C.c_double)
SYMBOLS = [
    ("kbr_last_error", C.c_char_p, []),
    ("kbr_tridiagonalize", _I, [_I64, _DP, _I, _DP, _DP, _DP, _DP, _DP, _DP]),
    ("kbr_back_transform", _I, [_I64, _I64, _DP, _DP, _DP, _DP, _DP, _DP, _I]),
    ("kbr_normalize_columns", _I, [_I64, _I64, _DP]),
    ("kbr_solve_tridiag", _I, [_I64, _DP, _DP, _I, _DP, _DP]),
    ("kbr_eigen_hh", _I, [_I64, _DP, _I, _I, _DP, _DP]),
    ("kbr_triple_product", _I, [_I64, _I64, _DP, _DP, _DP]),
]
_lib = None


def available() -> bool:
    if not os.path.exists(SO) and os.path.isdir("/root/reference/proj"):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=False)
    return os.path.exists(SO)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise OSError(f"{SO} missing (build with `make -C oracle ref` where /root/reference exists)")
        _lib = C.CDLL(SO)
        for name, res, args in SYMBOLS:
            fn = getattr(_lib, name)
            fn.restype, fn.argtypes = res, args
    return _lib


def _p(a):
    return a.ctypes.data_as(_DP)


def _call(st, what):
    if st:
        raise RuntimeError(f"{what}: status {st}: {lib().kbr_last_error().decode()}")


def tridiagonalize(a, fault_sign=False):
    a = np.ascontiguousarray(a, dtype=np.complex128)
    n = a.shape[0]
    nr = max(n - 1, 1)
    d, e, h, s = np.empty(n), np.empty(nr), np.empty(nr), np.empty(nr)
    u = np.empty((nr, n), dtype=np.complex128)
    ph = np.empty(nr, dtype=np.complex128)
    _call(lib().kbr_tridiagonalize(n, _p(a), int(fault_sign), _p(d), _p(e), _p(u), _p(h), _p(s), _p(ph)),
          "kbr_tridiagonalize")
    k = n - 1
    return d, e[:k], u[:k], h[:k], s[:k], ph[:k]


def back_transform(u, h, s, ph, y, threads=1):
    y = np.ascontiguousarray(y, dtype=np.float64)
    n, m = y.shape
    w = np.empty((n, m), dtype=np.complex128)
    u = np.ascontiguousarray(u, dtype=np.complex128)
    _call(lib().kbr_back_transform(n, m, _p(u), _p(np.ascontiguousarray(h)), _p(np.ascontiguousarray(s)),
                                   _p(np.ascontiguousarray(ph, dtype=np.complex128)), _p(y), _p(w), threads),
          "kbr_back_transform")
    return w


def normalize_columns(c):
    c = np.array(c, dtype=np.complex128, order="C", copy=True)
    _call(lib().kbr_normalize_columns(c.shape[0], c.shape[1], _p(c)), "kbr_normalize_columns")
    return c


def solve_tridiag(d, e, want_vectors=True):
    n = len(d)
    w = np.empty(n)
    z = np.empty((n, n)) if want_vectors else np.empty(1)
    _call(lib().kbr_solve_tridiag(n, _p(np.ascontiguousarray(d)), _p(np.ascontiguousarray(e) if n > 1 else
                                  np.zeros(1)), int(want_vectors), _p(w), _p(z)), "kbr_solve_tridiag")
    return w, (z if want_vectors else None)


def eigen_hh(a, want_vectors=True, threads=1):
    a = np.ascontiguousarray(a, dtype=np.complex128)
    n = a.shape[0]
    w = np.empty(n)
    v = np.empty((n, n), dtype=np.complex128) if want_vectors else np.empty(1, dtype=np.complex128)
    _call(lib().kbr_eigen_hh(n, _p(a), int(want_vectors), threads, _p(w), _p(v)), "kbr_eigen_hh")
    return w, (v if want_vectors else None)


def triple_product(t, h):
    t = np.ascontiguousarray(t, dtype=np.complex128)
    h = np.ascontiguousarray(h, dtype=np.complex128)
    n, m = t.shape
    c = np.empty((m, m), dtype=np.complex128)
    _call(lib().kbr_triple_product(n, m, _p(t), _p(h), _p(c)), "kbr_triple_product")
    return c
