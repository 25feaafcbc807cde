"""ctypes wrapper of oracle/liboracle.so -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke(), bench.py's CPU-baseline legs and offline
analysis tools (tools/padding_model.py, tools/crossover_model.py: index statistics)
use this module -- as the checker, the timed CPU baseline or an index source; never
the package. PARITY
UNPINNED: see oracle/oracle.h.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_1402_4247_b200 import _abi
from paper_1402_4247_b200.errors import raise_for_status

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "liboracle.so")

_P, _I, _I64, _D = C.c_void_p, C.c_int, C.c_int64, C.c_double
_DP = C.POINTER(C.c_double)
SYMBOLS = [
    ("kbo_create", _I, [C.POINTER(_abi.kbg_system), C.POINTER(_P)]),
    ("kbo_build_index", _I, [_P]),
    ("kbo_index_view", _I, [_P, C.POINTER(_abi.kbg_index)]),
    ("kbo_density", _I, [_P, _I, _DP, _DP, _I]),
    ("kbo_hamiltonian", _I, [_P, _I, _DP, _D, _DP, _I]),
    ("kbo_density_range", _I, [_P, _I, _DP, _DP, _I, _I64, _I64]),
    ("kbo_hamiltonian_range", _I, [_P, _I, _DP, _D, _DP, _I, _I64, _I64]),
    ("kbo_block_orbitals", _I, [_P, _I64, _DP, _I64, C.POINTER(_I)]),
    ("kbo_orbitals_at", _I, [_P, _I, _DP, _DP]),
    ("kbo_last_error", C.c_char_p, [_P]),
    ("kbo_normalize_rows", _I, [_DP, _I64, _I64, _I]),
    ("kbo_destroy", None, [_P]),
]


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    if not os.path.exists(SO):
        build()
    return _abi.load(SO, SYMBOLS)


class Oracle:
    def __init__(self, system):
        self._lib = lib()
        self.system = system
        self._csys = system.to_c()
        h = C.c_void_p()
        raise_for_status(self._lib.kbo_create(C.byref(self._csys), C.byref(h)), "kbo_create")
        self._h = h
        self._index = None

    def _check(self, st, what):
        if st:
            raise_for_status(st, what, self._lib.kbo_last_error(self._h).decode())

    def build_index(self) -> dict:
        self._check(self._lib.kbo_build_index(self._h), "kbo_build_index")
        ix = _abi.kbg_index()
        self._check(self._lib.kbo_index_view(self._h, C.byref(ix)), "kbo_index_view")
        self._index = _abi.index_to_numpy(ix)
        return self._index

    @property
    def index(self) -> dict:
        return self._index if self._index is not None else self.build_index()

    def density(self, dm: np.ndarray, threads: int = 0, blocks=None) -> np.ndarray:
        dm = np.ascontiguousarray(dm, dtype=np.float64)
        nspin = dm.shape[0]
        rho = np.zeros((nspin, self.system.npts))
        b0, b1 = blocks if blocks is not None else (0, self.index["nblock"])
        self._check(self._lib.kbo_density_range(self._h, nspin, _abi.dptr(dm), _abi.dptr(rho), threads, b0, b1),
                    "kbo_density")
        return rho

    def hamiltonian(self, veff: np.ndarray, dV: float, threads: int = 0, blocks=None) -> np.ndarray:
        veff = np.ascontiguousarray(veff, dtype=np.float64)
        nspin = veff.shape[0]
        h = np.zeros((nspin, self.index["nnz"]))
        b0, b1 = blocks if blocks is not None else (0, self.index["nblock"])
        self._check(self._lib.kbo_hamiltonian_range(self._h, nspin, _abi.dptr(veff), dV, _abi.dptr(h), threads,
                                                    b0, b1), "kbo_hamiltonian")
        return h

    def block_orbitals(self, block: int) -> np.ndarray:
        cap = 64 * 64 * 32
        out = np.zeros(cap)
        m = C.c_int()
        self._check(self._lib.kbo_block_orbitals(self._h, block, _abi.dptr(out), cap, C.byref(m)),
                    "kbo_block_orbitals")
        return out[: m.value * 64].reshape(m.value, 64)

    def orbitals_at(self, species: int, d) -> np.ndarray:
        d = np.ascontiguousarray(d, dtype=np.float64)
        out = np.zeros(32)
        self._check(self._lib.kbo_orbitals_at(self._h, species, _abi.dptr(d), _abi.dptr(out)), "kbo_orbitals_at")
        return out[: self.system.species[species].norb]

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._lib.kbo_destroy(h)
            self._h = None


def normalize_rows(x: np.ndarray, threads: int = 1) -> np.ndarray:
    """Host backend of the HBM probe (Table 2 normalization): rows of x divided by their norms."""
    x = np.array(x, dtype=np.float64, order="C", copy=True)
    nvec, n = (x.shape[0], x.shape[1]) if x.ndim == 2 else (1, x.shape[0])
    raise_for_status(lib().kbo_normalize_rows(_abi.dptr(x), nvec, n, threads), "kbo_normalize_rows")
    return x
