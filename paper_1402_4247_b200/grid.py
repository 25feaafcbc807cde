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


def normalize_rows(x: np.ndarray) -> np.ndarray:
    """HBM probe (Table 2 of the paper): each row of x divided by its norm, on the GPU
    through the host C-ABI (transfers included)."""
    x = np.array(x, dtype=np.float64, order="C", copy=True)
    nvec, n = (x.shape[0], x.shape[1]) if x.ndim == 2 else (1, x.shape[0])
    raise_for_status(_abi.kbgrid().kbg_normalize_rows(_abi.dptr(x), nvec, n), "kbg_normalize_rows")
    return x


def normalize_rows_dev(x, stream=None) -> None:
    """In place on a CUDA tensor (nvec, n) float64."""
    st = 0 if stream is None else int(stream.cuda_stream)
    raise_for_status(_abi.kbgrid().kbg_normalize_rows_dev(x.data_ptr(), x.shape[0], x.shape[1], st),
                     "kbg_normalize_rows_dev")


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

    def plan_info(self) -> dict:
        """Execution plan kbg_build_index chose (persistent kernels, schedule, rho split, sizes)."""
        v = (C.c_int64 * 8)()
        self._check(self._lib.kbg_plan_info(self._h, v), "kbg_plan_info")
        keys = ("persist", "schedule", "rho_split", "max_rows", "max_htask", "max_rtask", "smem_h", "smem_rho")
        return dict(zip(keys, (int(x) for x in v)))

    # -- G2 ------------------------------------------------------------------
    def block_orbitals(self, block: int) -> np.ndarray:
        cap = 64 * 64 * 32
        out = np.zeros(cap)
        m = C.c_int()
        self._check(self._lib.kbg_block_orbitals(self._h, block, _abi.dptr(out), cap, C.byref(m)),
                    "kbg_block_orbitals")
        return out[: m.value * 64].reshape(m.value, 64)

    # -- input validation (the C-ABI reads nspin * n doubles from each pointer) --
    @staticmethod
    def _spin_array(x, n: int, what: str) -> np.ndarray:
        """(n,) or (nspin, n) float64, C-contiguous; a flat 2n array is rejected, not reinterpreted."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        if x.ndim == 1:
            x = x[None]
        if x.ndim != 2 or x.shape[1] != n:
            raise_for_status(_abi.KBG_ERR_DIMENSION, what, f"expected ({n},) or (nspin, {n}), got {x.shape}")
        if x.shape[0] not in (1, 2):
            raise_for_status(_abi.KBG_ERR_CONFIG, what, f"nspin must be 1 or 2, got {x.shape[0]}")
        return x

    @staticmethod
    def _spin_tensor(t, n: int, what: str) -> int:
        """CUDA float64 tensor (nspin, n), contiguous; returns nspin."""
        import torch

        if t.dtype != torch.float64:
            raise_for_status(_abi.KBG_ERR_DIMENSION, what, f"dtype {t.dtype} (float64 required)")
        if not t.is_cuda or not t.is_contiguous():
            raise_for_status(_abi.KBG_ERR_CONFIG, what, "a contiguous CUDA tensor is required")
        if t.dim() != 2 or t.shape[1] != n:
            raise_for_status(_abi.KBG_ERR_DIMENSION, what, f"expected (nspin, {n}), got {tuple(t.shape)}")
        if t.shape[0] not in (1, 2):
            raise_for_status(_abi.KBG_ERR_CONFIG, what, f"nspin must be 1 or 2, got {t.shape[0]}")
        return int(t.shape[0])

    # -- G3 / G4, host buffers (drop-in) ---------------------------------------
    def density(self, dm: np.ndarray) -> np.ndarray:
        dm = self._spin_array(dm, self._nnz(), "density: dm")
        rho = np.empty((dm.shape[0], self.system.npts))
        self._check(self._lib.kbg_density(self._h, dm.shape[0], _abi.dptr(dm), _abi.dptr(rho)), "kbg_density")
        return rho

    def hamiltonian(self, veff: np.ndarray, dV: float) -> np.ndarray:
        veff = self._spin_array(veff, self.system.npts, "hamiltonian: veff")
        nnz = self._nnz()
        h = np.empty((veff.shape[0], nnz))
        self._check(self._lib.kbg_hamiltonian(self._h, veff.shape[0], _abi.dptr(veff), dV, _abi.dptr(h)),
                    "kbg_hamiltonian")
        return h

    def grid_pass(self, dm: np.ndarray, veff: np.ndarray, dV: float,
                  out: tuple[np.ndarray, np.ndarray] | None = None) -> tuple[np.ndarray, np.ndarray]:
        """rho and H of one SCF iteration in one call (overlapped transfers): returns (rho, h).
        `out` = (rho, h): caller-owned C-contiguous float64 outputs (e.g. pinned, which the kernels write
        in place); a sharded context writes only its share of them (KBG_OPT_SHARD_IO)."""
        dm = self._spin_array(dm, self._nnz(), "grid_pass: dm")
        veff = self._spin_array(veff, self.system.npts, "grid_pass: veff")
        if dm.shape[0] != veff.shape[0]:
            raise_for_status(_abi.KBG_ERR_DIMENSION, "grid_pass", "dm and veff spin counts differ")
        if out is not None:
            rho, h = out
            for a, n, what in ((rho, self.system.npts, "rho"), (h, self._nnz(), "h")):
                if (not isinstance(a, np.ndarray) or a.dtype != np.float64 or not a.flags.c_contiguous
                        or a.shape != (dm.shape[0], n)):
                    raise_for_status(_abi.KBG_ERR_DIMENSION, "grid_pass", f"out {what}: C-contiguous float64 "
                                     f"({dm.shape[0]}, {n}) required")
        else:
            # sharded contexts write only their share of rho and H (KBG_OPT_SHARD_IO): zeros elsewhere
            rho = np.zeros((dm.shape[0], self.system.npts))
            h = np.zeros((dm.shape[0], self._nnz()))
        self._check(self._lib.kbg_grid_pass(self._h, dm.shape[0], _abi.dptr(dm), _abi.dptr(veff), dV, _abi.dptr(rho),
                                            _abi.dptr(h)), "kbg_grid_pass")
        return rho, h

    def _nnz(self) -> int:
        ix = _abi.kbg_index()
        self._check(self._lib.kbg_index_view(self._h, C.byref(ix)), "kbg_index_view")
        return int(ix.nnz)

    # -- G3 / G4, device buffers (timing path; torch CUDA tensors) -------------
    @staticmethod
    def _stream_ptr(stream) -> int:
        return 0 if stream is None else int(stream.cuda_stream)

    def density_dev(self, dm, rho, stream=None) -> None:
        ns = self._spin_tensor(dm, self._nnz(), "density_dev: dm")
        if self._spin_tensor(rho, self.system.npts, "density_dev: rho") != ns:
            raise_for_status(_abi.KBG_ERR_DIMENSION, "density_dev", "dm and rho spin counts differ")
        self._check(self._lib.kbg_density_dev(self._h, dm.shape[0], dm.data_ptr(), rho.data_ptr(),
                                              self._stream_ptr(stream)), "kbg_density_dev")

    def _check_h_args(self, veff, h, what: str) -> None:
        ns = self._spin_tensor(veff, self.system.npts, what + ": veff")
        if self._spin_tensor(h, self._nnz(), what + ": h") != ns:
            raise_for_status(_abi.KBG_ERR_DIMENSION, what, "veff and h spin counts differ")

    def hamiltonian_dev(self, veff, dV: float, h, stream=None) -> None:
        self._check_h_args(veff, h, "hamiltonian_dev")
        self._check(self._lib.kbg_hamiltonian_dev(self._h, veff.shape[0], veff.data_ptr(), dV, h.data_ptr(),
                                                  self._stream_ptr(stream)), "kbg_hamiltonian_dev")

    def hamiltonian_accumulate_dev(self, veff, dV: float, h, stream=None) -> None:
        self._check_h_args(veff, h, "hamiltonian_accumulate_dev")
        self._check(self._lib.kbg_hamiltonian_accumulate_dev(self._h, veff.shape[0], veff.data_ptr(), dV,
                                                             h.data_ptr(), self._stream_ptr(stream)),
                    "kbg_hamiltonian_accumulate_dev")

    def grid_pass_dev(self, dm, veff, dV: float, rho, h, stream=None) -> None:
        """rho and the mirrored H of one pass on device tensors (kbg_grid_pass_dev: one fused persistent
        kernel when possible)."""
        ns = self._spin_tensor(dm, self._nnz(), "grid_pass_dev: dm")
        for t, n, what in ((veff, self.system.npts, "veff"), (rho, self.system.npts, "rho"), (h, self._nnz(), "h")):
            if self._spin_tensor(t, n, "grid_pass_dev: " + what) != ns:
                raise_for_status(_abi.KBG_ERR_DIMENSION, "grid_pass_dev", f"{what} spin count differs from dm's")
        self._check(self._lib.kbg_grid_pass_dev(self._h, ns, dm.data_ptr(), veff.data_ptr(), dV, rho.data_ptr(),
                                                h.data_ptr(), self._stream_ptr(stream)), "kbg_grid_pass_dev")

    def hamiltonian_mirror_dev(self, h, stream=None) -> None:
        self._spin_tensor(h, self._nnz(), "hamiltonian_mirror_dev: h")
        self._check(self._lib.kbg_hamiltonian_mirror_dev(self._h, h.shape[0], h.data_ptr(),
                                                         self._stream_ptr(stream)), "kbg_hamiltonian_mirror_dev")

    # -- V_eff from rho (kb_veff.cu) -------------------------
    def veff(self, rho: np.ndarray, vloc: np.ndarray | None = None) -> tuple[np.ndarray, tuple[float, float]]:
        """V_eff,s = V_H + V_x,s (+ V_loc) on the grid and (E_H, E_x)."""
        rho = np.ascontiguousarray(rho, dtype=np.float64)
        if rho.ndim == 1:
            rho = rho[None]
        out = np.empty_like(rho)
        e = (C.c_double * 2)()
        vl = None if vloc is None else np.ascontiguousarray(vloc, dtype=np.float64)
        self._check(self._lib.kbg_veff(self._h, rho.shape[0], _abi.dptr(rho), None if vl is None else _abi.dptr(vl),
                                       _abi.dptr(out), e), "kbg_veff")
        return out, (e[0], e[1])

    def veff_dev(self, rho, veff, vloc=None, energy=None, stream=None) -> None:
        self._check(self._lib.kbg_veff_dev(self._h, rho.shape[0], rho.data_ptr(),
                                           None if vloc is None else vloc.data_ptr(), veff.data_ptr(),
                                           None if energy is None else energy.data_ptr(), self._stream_ptr(stream)),
                    "kbg_veff_dev")

    # -- multi-GPU H over peer memory (kb_comm.cu) ----------------------------
    def comm_handle(self) -> bytes:
        """This rank's exchange-buffer handle (all-gather it, then comm_open)."""
        buf = C.create_string_buffer(_abi.KBG_COMM_HANDLE_BYTES)
        self._check(self._lib.kbg_comm_handle(self._h, buf), "kbg_comm_handle")
        return buf.raw

    def comm_open(self, handles) -> None:
        blob = b"".join(handles)
        buf = C.create_string_buffer(blob, len(blob))
        self._check(self._lib.kbg_comm_open(self._h, buf), "kbg_comm_open")

    def hamiltonian_allreduce_dev(self, veff, dV: float, h, stream=None) -> None:
        """Sharded H pass whose result is the full, mirrored H on every rank (no NCCL)."""
        self._check_h_args(veff, h, "hamiltonian_allreduce_dev")
        self._check(self._lib.kbg_hamiltonian_allreduce_dev(self._h, veff.shape[0], veff.data_ptr(), dV, h.data_ptr(),
                                                            self._stream_ptr(stream)),
                    "kbg_hamiltonian_allreduce_dev")

    def shard_io(self) -> dict:
        """Shard-local I/O ranges of kbg_grid_pass on this sharded context (after comm_open)."""
        v = (C.c_int64 * 8)()
        self._check(self._lib.kbg_shard_io(self._h, v), "kbg_shard_io")
        keys = ("b0", "b1", "p0", "p1", "h0", "h1", "dm_read", "v_read")
        return dict(zip(keys, (int(x) for x in v)))

    def hamiltonian_partial_dev(self, veff, dV: float, stream=None) -> None:
        """First half of hamiltonian_allreduce_dev: this rank's partial H into its exchange buffer."""
        self._spin_tensor(veff, self.system.npts, "hamiltonian_partial_dev: veff")
        self._check(self._lib.kbg_hamiltonian_partial_dev(self._h, veff.shape[0], veff.data_ptr(), dV,
                                                          self._stream_ptr(stream)), "kbg_hamiltonian_partial_dev")

    def hamiltonian_exchange_dev(self, h, stream=None) -> None:
        """Second half: the fused reduce + mirror over peer memory -> the full H in h."""
        ns = self._spin_tensor(h, self._nnz(), "hamiltonian_exchange_dev: h")
        self._check(self._lib.kbg_hamiltonian_exchange_dev(self._h, ns, h.data_ptr(), self._stream_ptr(stream)),
                    "kbg_hamiltonian_exchange_dev")

    def comm_check(self) -> None:
        """After synchronizing a hamiltonian_allreduce_dev: raise if a peer never arrived."""
        self._check(self._lib.kbg_comm_check(self._h), "kbg_comm_check")

    # -- formats either side (see formats.py for the SPEC types) --
    def offsets(self) -> np.ndarray:
        """Distinct lattice offsets R of the pair list, sorted, shape (nR, 3)."""
        n = C.c_int()
        self._check(self._lib.kbg_offsets(self._h, C.byref(n), None), "kbg_offsets")
        R = np.empty((n.value, 3), dtype=np.int32)
        self._check(self._lib.kbg_offsets(self._h, C.byref(n), R.ctypes.data_as(C.POINTER(C.c_int32))),
                    "kbg_offsets")
        return R

    def nbasis(self) -> int:
        return int(self.system.nbasis)

    def _pairs(self, x) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        if x.shape != (self._nnz(),):
            raise_for_status(_abi.KBG_ERR_DIMENSION, "pairs", f"expected ({self._nnz()},) values, got {x.shape}")
        return x

    def to_realspace(self, pairs: np.ndarray) -> np.ndarray:
        """pair-sparse (nnz,) -> dense blocks (nR, n, n) in offsets() order."""
        pairs = self._pairs(pairs)
        n = self.nbasis()
        out = np.empty((len(self.offsets()), n, n))
        self._check(self._lib.kbg_to_realspace(self._h, _abi.dptr(pairs), _abi.dptr(out)), "kbg_to_realspace")
        return out

    def from_realspace(self, blocks: np.ndarray) -> np.ndarray:
        n = self.nbasis()
        blocks = np.ascontiguousarray(blocks, dtype=np.float64)
        if blocks.shape != (len(self.offsets()), n, n):
            raise_for_status(_abi.KBG_ERR_DIMENSION, "from_realspace", f"blocks shape {blocks.shape}")
        out = np.empty(self._nnz())
        self._check(self._lib.kbg_from_realspace(self._h, _abi.dptr(blocks), _abi.dptr(out)), "kbg_from_realspace")
        return out

    def bloch(self, pairs: np.ndarray, kpts) -> np.ndarray:
        """M(k) = sum_R exp(+2 pi i k.R) M_R for each k (fractional), (nk, n, n) complex."""
        pairs = self._pairs(pairs)
        k = np.ascontiguousarray(np.atleast_2d(kpts), dtype=np.float64)
        n = self.nbasis()
        out = np.empty((k.shape[0], n, n), dtype=np.complex128)
        self._check(self._lib.kbg_bloch(self._h, _abi.dptr(pairs), k.shape[0], _abi.dptr(k),
                                        out.ctypes.data_as(_abi._DP)), "kbg_bloch")
        return out

    def fold(self, rho_k: np.ndarray, kpts, weights) -> tuple[np.ndarray, float]:
        """DM_R = Re sum_k w_k exp(-2 pi i k.R) rho_k on the pair list; returns (pairs, max |imag|)."""
        k = np.ascontiguousarray(np.atleast_2d(kpts), dtype=np.float64)
        w = np.ascontiguousarray(weights, dtype=np.float64)
        n = self.nbasis()
        rho_k = np.ascontiguousarray(rho_k, dtype=np.complex128)
        if rho_k.shape != (k.shape[0], n, n) or w.shape != (k.shape[0],):
            raise_for_status(_abi.KBG_ERR_DIMENSION, "fold", f"rho_k {rho_k.shape}, weights {w.shape}, nk {k.shape[0]}")
        out = np.empty(self._nnz())
        mi = C.c_double()
        self._check(self._lib.kbg_fold(self._h, k.shape[0], _abi.dptr(k), _abi.dptr(w),
                                       rho_k.ctypes.data_as(_abi._DP), _abi.dptr(out), C.byref(mi)), "kbg_fold")
        return out, mi.value

    def density_matrix_k(self, C: np.ndarray, w) -> np.ndarray:
        """rho_k = sum_i w_i c_i c_i^H from states C (n, m) complex (columns = states)."""
        C = np.ascontiguousarray(C, dtype=np.complex128)
        w = np.ascontiguousarray(w, dtype=np.float64)
        n = self.nbasis()
        if C.ndim != 2 or C.shape[0] != n or w.shape != (C.shape[1],):
            raise_for_status(_abi.KBG_ERR_DIMENSION, "density_matrix_k", f"C {C.shape}, w {w.shape}, n {n}")
        out = np.empty((n, n), dtype=np.complex128)
        self._check(self._lib.kbg_density_matrix_k(self._h, C.shape[1], C.ctypes.data_as(_abi._DP), _abi.dptr(w),
                                                   out.ctypes.data_as(_abi._DP)), "kbg_density_matrix_k")
        return out

    def density_matrix_k_dev(self, C, w, out, stream=None) -> None:
        self._check(self._lib.kbg_density_matrix_k_dev(self._h, C.shape[1], C.data_ptr(), w.data_ptr(), out.data_ptr(),
                                                       self._stream_ptr(stream)), "kbg_density_matrix_k_dev")

    def bloch_dev(self, pairs, kpts, out, stream=None) -> None:
        k = np.ascontiguousarray(np.atleast_2d(kpts), dtype=np.float64)
        self._check(self._lib.kbg_bloch_dev(self._h, pairs.data_ptr(), k.shape[0], _abi.dptr(k), out.data_ptr(),
                                            self._stream_ptr(stream)), "kbg_bloch_dev")

    def fold_dev(self, rho_k, kpts, weights, out, stream=None) -> None:
        k = np.ascontiguousarray(np.atleast_2d(kpts), dtype=np.float64)
        w = np.ascontiguousarray(weights, dtype=np.float64)
        self._check(self._lib.kbg_fold_dev(self._h, k.shape[0], _abi.dptr(k), _abi.dptr(w), rho_k.data_ptr(),
                                           out.data_ptr(), self._stream_ptr(stream)), "kbg_fold_dev")

    def to_realspace_dev(self, pairs, blocks, stream=None) -> None:
        self._check(self._lib.kbg_to_realspace_dev(self._h, pairs.data_ptr(), blocks.data_ptr(),
                                                   self._stream_ptr(stream)), "kbg_to_realspace_dev")

    def from_realspace_dev(self, blocks, pairs, stream=None) -> None:
        self._check(self._lib.kbg_from_realspace_dev(self._h, blocks.data_ptr(), pairs.data_ptr(),
                                                     self._stream_ptr(stream)), "kbg_from_realspace_dev")

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
