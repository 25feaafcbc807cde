"""Structure / Species / GridSpec value types.

A `System` owns numpy copies of everything a `kbg_system` points to, so the
ctypes struct it hands to the C-ABI stays valid for the System's lifetime.
Invariants are checked here with the reference's error taxonomy
(/root/reference/proj/include/kband/common.hpp:21-38) before any call.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from .errors import ConfigError, DimensionError, raise_for_status

ORB_PER_L = (1, 3, 5)


@dataclass
class Species:
    l: list[int]
    rc: float
    table: np.ndarray  # [nrad, ntab, 2] (u, du/dr), u = R(r)/r^l on [0, rc]

    def __post_init__(self):
        self.table = np.ascontiguousarray(self.table, dtype=np.float64)
        if self.table.ndim != 3 or self.table.shape[2] != 2:
            raise DimensionError("Species.table must be [nrad, ntab, 2]")
        if self.table.shape[0] != len(self.l):
            raise DimensionError("Species.table rows != len(l)")
        if any(l < 0 or l > 2 for l in self.l):
            raise ConfigError("Species.l must be in 0..2")
        if not self.rc > 0:
            raise ConfigError("Species.rc must be > 0")

    @property
    def norb(self) -> int:
        return sum(ORB_PER_L[l] for l in self.l)

    @property
    def ntab(self) -> int:
        return self.table.shape[1]


@dataclass
class System:
    lattice: np.ndarray  # [3,3] rows = lattice vectors (bohr)
    grid: tuple[int, int, int]
    species_of_atom: np.ndarray  # [natom] int
    tau: np.ndarray  # [natom, 3] Cartesian bohr
    species: list[Species]
    _keep: list = field(default_factory=list, repr=False)

    def __post_init__(self):
        self.lattice = np.ascontiguousarray(self.lattice, dtype=np.float64).reshape(3, 3)
        self.species_of_atom = np.ascontiguousarray(self.species_of_atom, dtype=np.int32)
        self.tau = np.ascontiguousarray(self.tau, dtype=np.float64).reshape(-1, 3)
        self.grid = tuple(int(g) for g in self.grid)
        if len(self.tau) != len(self.species_of_atom):
            raise DimensionError("System: tau and species_of_atom lengths differ")
        if any(g < 1 for g in self.grid):
            raise DimensionError("System: grid dimensions must be >= 1")

    @property
    def natom(self) -> int:
        return len(self.tau)

    @property
    def npts(self) -> int:
        return self.grid[0] * self.grid[1] * self.grid[2]

    @property
    def dV(self) -> float:
        return abs(float(np.linalg.det(self.lattice))) / self.npts

    @property
    def nbasis(self) -> int:
        return int(sum(self.species[s].norb for s in self.species_of_atom))

    def norb_of_atom(self) -> np.ndarray:
        return np.array([self.species[s].norb for s in self.species_of_atom], dtype=np.int64)

    def to_c(self) -> _abi.kbg_system:
        """ctypes kbg_system pointing into this System's arrays."""
        sp_arr = (_abi.kbg_species * len(self.species))()
        keep = []
        for i, sp in enumerate(self.species):
            l = np.ascontiguousarray(sp.l, dtype=np.int32)
            keep += [l, sp.table]
            sp_arr[i].nrad = len(sp.l)
            sp_arr[i].l = l.ctypes.data_as(C.POINTER(C.c_int))
            sp_arr[i].rc = sp.rc
            sp_arr[i].ntab = sp.ntab
            sp_arr[i].table = sp.table.ctypes.data_as(C.POINTER(C.c_double))
        s = _abi.kbg_system()
        for i in range(9):
            s.lattice[i] = float(self.lattice.reshape(-1)[i])
        for i in range(3):
            s.grid[i] = self.grid[i]
        s.natom = self.natom
        s.species = self.species_of_atom.ctypes.data_as(C.POINTER(C.c_int))
        s.tau = self.tau.ctypes.data_as(C.POINTER(C.c_double))
        s.nspecies = len(self.species)
        s.spec = C.cast(sp_arr, C.POINTER(_abi.kbg_species))
        keep.append(sp_arr)
        self._keep = keep  # keep the pointed-to buffers alive
        self._c = s
        return s

    @staticmethod
    def from_c(s: _abi.kbg_system) -> "System":
        species = []
        for i in range(s.nspecies):
            sp = s.spec[i]
            l = [sp.l[k] for k in range(sp.nrad)]
            tab = np.ctypeslib.as_array(sp.table, shape=(sp.nrad * sp.ntab * 2,)).copy()
            species.append(Species(l=l, rc=sp.rc, table=tab.reshape(sp.nrad, sp.ntab, 2)))
        natom = s.natom
        return System(
            lattice=np.array(list(s.lattice)).reshape(3, 3),
            grid=tuple(s.grid),
            species_of_atom=np.ctypeslib.as_array(s.species, shape=(natom,)).copy(),
            tau=np.ctypeslib.as_array(s.tau, shape=(natom * 3,)).copy().reshape(natom, 3),
            species=species,
        )


def radial_table(l: int, alpha: float, rc: float, ntab: int = 1024) -> np.ndarray:
    """u(r) = R(r)/r^l for R = N r^l exp(-alpha r^2)(1-(r/rc)^2)^3, normalised."""
    out = np.zeros((ntab, 2))
    _abi.kbgsynth().kbg_synth_radial_table(l, alpha, rc, ntab, _abi.dptr(out))
    return out


def good_size(n: int) -> int:
    return int(_abi.kbgsynth().kbg_synth_good_size(n))


class Fe3O4:
    """Synthetic magnetite inputs from libkbgsynth."""

    CONFIGS = {
        # name: (kind, rep, ecut_ry)
        "primitive14_150Ry": (_abi.KBG_CELL_PRIMITIVE, 1, 150.0),
        "cubic56_200Ry": (_abi.KBG_CELL_CUBIC, 1, 200.0),
        "super448_200Ry": (_abi.KBG_CELL_CUBIC, 2, 200.0),
        "super1512_200Ry": (_abi.KBG_CELL_CUBIC, 3, 200.0),
    }

    def __init__(self, kind: int = _abi.KBG_CELL_CUBIC, rep: int = 1, ecut_ry: float = 200.0,
                 seed: int = 1402, ntab: int = 1024):
        self._lib = _abi.kbgsynth()
        h = C.c_void_p()
        raise_for_status(self._lib.kbg_synth_create(kind, rep, ecut_ry, seed, ntab, C.byref(h)),
                         "kbg_synth_create")
        self._h = h
        self.kind, self.rep, self.ecut_ry, self.seed = kind, rep, ecut_ry, seed
        self.system = System.from_c(self._lib.kbg_synth_system(h).contents)
        self.dV = float(self._lib.kbg_synth_dV(h))

    @classmethod
    def config(cls, name: str, **kw) -> "Fe3O4":
        if name.startswith("sweep56_"):
            ecut = float(name.split("_")[1].rstrip("Ry"))
            return cls(_abi.KBG_CELL_CUBIC, 1, ecut, **kw)
        kind, rep, ecut = cls.CONFIGS[name]
        return cls(kind, rep, ecut, **kw)

    def veff(self, nspin: int = 1, seed: int = 1402) -> np.ndarray:
        out = np.zeros((nspin, self.system.npts))
        raise_for_status(self._lib.kbg_synth_veff(self._h, nspin, seed, _abi.dptr(out)), "kbg_synth_veff")
        return out

    def dm(self, index: dict, nspin: int = 1, seed: int = 1402) -> np.ndarray:
        out = np.zeros((nspin, index["nnz"]))
        ix = _abi.index_from_numpy(index)
        raise_for_status(self._lib.kbg_synth_dm(self._h, C.byref(ix), nspin, seed, _abi.dptr(out)),
                         "kbg_synth_dm")
        return out

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._lib.kbg_synth_free(h)
            self._h = None
