"""Host-side mirror of the grid-pass operator API over the C-ABI (libkbgrid.so).

Operators: build_index (A1), orbitals_on_grid (A2,
block_orbitals), density_grid (A3), hamiltonian_grid (A4). Signatures follow
the reference's style -- inputs by value, outputs returned, errors raised as
the kband taxonomy (/root/reference/proj/include/kband/linalg.hpp:75-80,
common.hpp:21-38). Every call goes through the CUDA library; there is no CPU
path here.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _abi
from .errors import raise_for_status
from .system import System


class GridPass:
    def __init__(self, system: System, device: int = 0, rank: int = 0, nranks: int = 1):
        self._lib = _abi.kbgrid()
        self.system = system
        self._csys = system.to_c()
        h = C.c_void_p()
        st = self._lib.kbg_create_sharded(C.byref(self._csys), device, rank, nranks, C.byref(h))
        raise_for_status(st, "kbg_create")
        self._h = h
        self.device = device
        self._index = None

    # -- helpers -------------------------------------------------------------
    def _check(self, st: int, what: str) -> None:
        if st:
            raise_for_status(st, what, self._lib.kbg_last_error(self._h).decode())

    @property
    def handle(self):
        return self._h

    def set_option(self, option: int, value: int) -> None:
        self._check(self._lib.kbg_set_option(self._h, option, value), "kbg_set_option")

    # -- G1 ------------------------------------------------------------------
    def build_index(self) -> dict:
        self._check(self._lib.kbg_build_index(self._h), "kbg_build_index")
        self._index = None
        return self.index

    @property
    def index(self) -> dict:
        if self._index is None:
            ix = _abi.kbg_index()
            self._check(self._lib.kbg_index_view(self._h, C.byref(ix)), "kbg_index_view")
            self._index = _abi.index_to_numpy(ix)
        return self._index

    def shard_range(self) -> tuple[int, int]:
        b0, b1 = C.c_int64(), C.c_int64()
        self._check(self._lib.kbg_shard_range(self._h, C.byref(b0), C.byref(b1)), "kbg_shard_range")
        return b0.value, b1.value

    # -- G2 ------------------------------------------------------------------
    def block_orbitals(self, block: int) -> np.ndarray:
        cap = 64 * 64 * 32
        out = np.zeros(cap)
        m = C.c_int()
        self._check(self._lib.kbg_block_orbitals(self._h, block, _abi.dptr(out), cap, C.byref(m)),
                    "kbg_block_orbitals")
        return out[: m.value * 64].reshape(m.value, 64)

    # -- G3 / G4, host buffers (drop-in) ---------------------------------------
    def density(self, dm: np.ndarray) -> np.ndarray:
        dm = np.ascontiguousarray(dm, dtype=np.float64)
        if dm.ndim == 1:
            dm = dm[None]
        rho = np.empty((dm.shape[0], self.system.npts))
        self._check(self._lib.kbg_density(self._h, dm.shape[0], _abi.dptr(dm), _abi.dptr(rho)), "kbg_density")
        return rho

    def hamiltonian(self, veff: np.ndarray, dV: float) -> np.ndarray:
        veff = np.ascontiguousarray(veff, dtype=np.float64)
        if veff.ndim == 1:
            veff = veff[None]
        nnz = self._nnz()
        h = np.empty((veff.shape[0], nnz))
        self._check(self._lib.kbg_hamiltonian(self._h, veff.shape[0], _abi.dptr(veff), dV, _abi.dptr(h)),
                    "kbg_hamiltonian")
        return h

    def _nnz(self) -> int:
        ix = _abi.kbg_index()
        self._check(self._lib.kbg_index_view(self._h, C.byref(ix)), "kbg_index_view")
        return int(ix.nnz)

    # -- G3 / G4, device buffers (timing path; torch CUDA tensors) -------------
    @staticmethod
    def _stream_ptr(stream) -> int:
        return 0 if stream is None else int(stream.cuda_stream)

    def density_dev(self, dm, rho, stream=None) -> None:
        self._check(self._lib.kbg_density_dev(self._h, dm.shape[0], dm.data_ptr(), rho.data_ptr(),
                                              self._stream_ptr(stream)), "kbg_density_dev")

    def hamiltonian_dev(self, veff, dV: float, h, stream=None) -> None:
        self._check(self._lib.kbg_hamiltonian_dev(self._h, veff.shape[0], veff.data_ptr(), dV, h.data_ptr(),
                                                  self._stream_ptr(stream)), "kbg_hamiltonian_dev")

    def hamiltonian_accumulate_dev(self, veff, dV: float, h, stream=None) -> None:
        self._check(self._lib.kbg_hamiltonian_accumulate_dev(self._h, veff.shape[0], veff.data_ptr(), dV,
                                                             h.data_ptr(), self._stream_ptr(stream)),
                    "kbg_hamiltonian_accumulate_dev")

    def hamiltonian_mirror_dev(self, h, stream=None) -> None:
        self._check(self._lib.kbg_hamiltonian_mirror_dev(self._h, h.shape[0], h.data_ptr(),
                                                         self._stream_ptr(stream)), "kbg_hamiltonian_mirror_dev")

    @property
    def last_launches(self) -> int:
        return int(self._lib.kbg_last_launches(self._h))

    @property
    def last_tally(self) -> tuple[float, float]:
        t = _abi.kbg_tally()
        self._check(self._lib.kbg_last_tally(self._h, C.byref(t)), "kbg_last_tally")
        return t.flops, t.bytes

    def close(self) -> None:
        h = getattr(self, "_h", None)
        if h:
            self._lib.kbg_destroy(h)
            self._h = None

    def __del__(self):
        self.close()
