"""Formats either side of the grid pass, in the reference's band-pipeline types.

The grid pass reads the density matrix and writes H as pair-sparse real-space blocks (the kbg_index
pair list). The reference's band pipeline (SPEC-only -- no code in
proj/) exchanges:

* ``RealSpaceOperator`` -- dense n x n block M_R per lattice offset R, invariant M_{-R} = M_R^dagger
  and R = 0 present. It houses H and S.
* ``KPointSet`` -- fractional k points with weights summing to 1 within 1e-12.
* ``bloch_transform`` -- M(k) = sum_R exp(+2 pi i k.R) M_R, validated Hermitian (Part 1).
* ``DensityMatrices`` -- real-space folding rho(R) = sum_k w_k exp(-2 pi i k.R) rho_k (Part 6,
  SPEC.md:275-283), which becomes the grid pass's DM input.

Every conversion runs on the GPU through libkbgrid (kb_formats.cu); this module only adapts types.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import ConfigError, ConsistencyError, DimensionError
from .grid import GridPass


@dataclass
class KPointSet:
    """points (nk, 3) fractional, weights > 0 with sum 1 within 1e-12."""

    points: np.ndarray
    weights: np.ndarray

    def __post_init__(self):
        self.points = np.ascontiguousarray(np.atleast_2d(self.points), dtype=np.float64)
        self.weights = np.ascontiguousarray(self.weights, dtype=np.float64).reshape(-1)
        if self.points.shape[1] != 3 or len(self.points) != len(self.weights) or len(self.points) == 0:
            raise DimensionError(f"KPointSet: points {self.points.shape} vs weights {self.weights.shape}")
        if not np.all(self.weights > 0):
            raise ConfigError("KPointSet: weights must be > 0")
        if abs(self.weights.sum() - 1.0) > 1e-12:
            raise ConfigError(f"KPointSet: weights sum to {self.weights.sum():.17g}, not 1 within 1e-12")

    @staticmethod
    def monkhorst_pack(n1: int, n2: int, n3: int) -> "KPointSet":
        """Gamma-centred uniform grid k_i = m_i / n_i (time-reversal symmetric), uniform weights."""
        g = np.stack(np.meshgrid(np.arange(n1) / n1, np.arange(n2) / n2, np.arange(n3) / n3, indexing="ij"), -1)
        pts = g.reshape(-1, 3)
        return KPointSet(pts, np.full(len(pts), 1.0 / len(pts)))


@dataclass
class RealSpaceOperator:
    """dim n, blocks [(R, M_R)] with M_{-R} = M_R^dagger and R = 0 present."""

    n: int
    blocks: list = field(default_factory=list)  # [(tuple R, ndarray (n, n))]

    def block(self, R) -> np.ndarray:
        for r, m in self.blocks:
            if tuple(r) == tuple(R):
                return m
        raise ConsistencyError(f"RealSpaceOperator: no block for R={tuple(R)}")

    def validate(self, tol: float = 1e-13) -> None:
        have = {tuple(r) for r, _ in self.blocks}
        if (0, 0, 0) not in have:
            raise ConsistencyError("RealSpaceOperator: R=0 block missing")
        amax = max((np.abs(m).max() for _, m in self.blocks), default=0.0)
        for r, m in self.blocks:
            mr = tuple(-x for x in r)
            if mr not in have:
                raise ConsistencyError(f"RealSpaceOperator: missing -R partner of R={tuple(r)}")
            d = np.abs(self.block(mr) - m.conj().T).max()
            if d > tol * max(amax, 1e-300):
                raise ConsistencyError(f"RealSpaceOperator: M_(-R) != M_R^dagger at R={tuple(r)} by {d:.3e}")


def to_realspace_operator(gp: GridPass, pairs: np.ndarray) -> RealSpaceOperator:
    """pair-sparse blocks (one spin, nnz values) -> RealSpaceOperator (GPU scatter)."""
    dense = gp.to_realspace(pairs)
    return RealSpaceOperator(gp.nbasis(), [(tuple(int(x) for x in r), dense[i]) for i, r in enumerate(gp.offsets())])


def from_realspace_operator(gp: GridPass, op: RealSpaceOperator) -> np.ndarray:
    """RealSpaceOperator -> pair-sparse blocks of this index (GPU gather). Every offset of the pair list
    must be present in op (DimensionError naming the first missing R); imaginary parts must vanish."""
    if op.n != gp.nbasis():
        raise DimensionError(f"from_realspace_operator: n = {op.n}, basis has {gp.nbasis()}")
    stack = []
    for r in gp.offsets():
        try:
            m = op.block(tuple(int(x) for x in r))
        except ConsistencyError:
            raise DimensionError(f"from_realspace_operator: no block for R={tuple(int(x) for x in r)}") from None
        if np.iscomplexobj(m):
            if np.abs(m.imag).max() > 0:
                raise ConsistencyError(f"from_realspace_operator: complex block at R={tuple(r)} (grid pass is real)")
            m = m.real
        stack.append(m)
    return gp.from_realspace(np.stack(stack))


def bloch_transform(gp: GridPass, pairs: np.ndarray, k) -> np.ndarray:
    """Part 1 for one k or an (nk, 3) array: M(k) = sum_R exp(+2 pi i k.R) M_R.
    Validates M_{-R} = M_R^T (ConsistencyError naming the pair and R)."""
    k = np.asarray(k, dtype=np.float64)
    out = gp.bloch(pairs, k)
    return out[0] if k.ndim == 1 else out


def density_matrices_k(gp: GridPass, C: np.ndarray, f, eps=None):
    """Part 6 at one k: rho_k = sum_i f_i c_i c_i^dagger and, with eps, the energy density
    matrix E_k = sum_i eps_i f_i c_i c_i^dagger. C: (n, m) states as columns. GPU (one ZGEMM each)."""
    f = np.asarray(f, dtype=np.float64)
    rho = gp.density_matrix_k(C, f)
    if eps is None:
        return rho
    return rho, gp.density_matrix_k(C, np.asarray(eps, dtype=np.float64) * f)


def fold_density_matrices(gp: GridPass, rho_k: np.ndarray, kset: KPointSet, imag_tol: float = 1e-10) -> np.ndarray:
    """Part 6 folding: DM_R = sum_k w_k exp(-2 pi i k.R) rho_k on the pair list.
    The grid pass takes a real DM; an imaginary part above imag_tol * max|DM| (a k set without
    time-reversal partners) raises ConsistencyError."""
    dm, max_imag = gp.fold(rho_k, kset.points, kset.weights)
    scale = max(np.abs(dm).max(), 1e-300)
    if max_imag > imag_tol * scale:
        raise ConsistencyError(f"fold_density_matrices: imaginary part {max_imag:.3e} (k set not time-reversal "
                               f"symmetric?)")
    return dm


__all__ = ["KPointSet", "RealSpaceOperator", "to_realspace_operator", "from_realspace_operator",
           "bloch_transform", "density_matrices_k", "fold_density_matrices"]
