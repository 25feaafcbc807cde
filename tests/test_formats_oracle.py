"""CPU: the numpy restatement of the format converters (oracle/formats.py) against the worked examples
of the reference's band-pipeline SPEC, and the host-side SPEC types
(KPointSet, RealSpaceOperator invariants)."""
import numpy as np
import pytest

from oracle import formats as F
from paper_1402_4247_b200.errors import ConfigError, ConsistencyError, DimensionError
from paper_1402_4247_b200.formats import KPointSet, RealSpaceOperator


def chain(t):
    """1x1 chain: one atom with one orbital, M_{+-1} = t, M_0 = 0."""
    pair_a = np.array([0, 0, 0])
    pair_b = np.array([0, 0, 0])
    pair_R = np.array([[-1, 0, 0], [0, 0, 0], [1, 0, 0]])
    pair_off = np.array([0, 1, 2, 3])
    return np.array([t, 0.0, t]), pair_a, pair_b, pair_R, pair_off, [1]


def random_symmetric(seed=7, natom=3, norb=(2, 3, 1), Rmax=1):
    """Random pair list with M_{b,a,-R} = M_{a,b,R}^T over all R in [-Rmax, Rmax]^3 (mt-style seeded)."""
    rng = np.random.default_rng(seed)
    keys = []
    for a in range(natom):
        for b in range(natom):
            for R in np.ndindex(*(2 * Rmax + 1,) * 3):
                R = tuple(np.array(R) - Rmax)
                if rng.random() < 0.4 or (a == b and R == (0, 0, 0)):
                    keys.append((a, b, R))
    keys = sorted(set(keys) | {(b, a, tuple(-x for x in R)) for a, b, R in keys})
    off = [0]
    for a, b, _ in keys:
        off.append(off[-1] + norb[a] * norb[b])
    vals = np.zeros(off[-1])
    idx = {k: i for i, k in enumerate(keys)}
    for i, (a, b, R) in enumerate(keys):
        j = idx[(b, a, tuple(-x for x in R))]
        if j < i:
            continue
        blk = rng.uniform(-1, 1, (norb[a], norb[b]))
        if i == j:
            blk = 0.5 * (blk + blk.T)
        vals[off[i]:off[i + 1]] = blk.ravel()
        vals[off[j]:off[j + 1]] = blk.T.ravel()
    pa = np.array([k[0] for k in keys])
    pb = np.array([k[1] for k in keys])
    pR = np.array([k[2] for k in keys])
    return vals, pa, pb, pR, np.array(off), list(norb)


def test_bloch_single_block_R0_is_constant():
    """single block R=0 -> M(k) = M_0 for every k."""
    m0 = np.array([[1.0, 2.0], [2.0, -3.0]])
    args = (m0.ravel(), np.array([0]), np.array([0]), np.array([[0, 0, 0]]), np.array([0, 4]), [2])
    for k in ([0, 0, 0], [0.25, 0.1, -0.3], [0.5, 0.5, 0.5]):
        assert np.array_equal(F.bloch(*args, k), m0.astype(np.complex128))


@pytest.mark.parametrize("k", [0.0, 0.125, 0.25, 1 / 3, 0.5, 0.9])
def test_bloch_chain_is_2t_cos(k):
    """1x1 chain, M_{+-1} = t, M_0 = 0 -> M(k) = 2t cos(2 pi k)."""
    t = 0.7
    m = F.bloch(*chain(t), [k, 0.3, -0.2])
    assert abs(m[0, 0] - 2 * t * np.cos(2 * np.pi * k)) < 1e-15


def test_bloch_gamma_is_sum_and_symmetric():
    """k = 0 -> sum_R M_R, real-symmetric when all blocks are real."""
    vals, pa, pb, pR, off, norb = random_symmetric()
    m = F.bloch(vals, pa, pb, pR, off, norb, [0, 0, 0])
    dense = F.to_realspace(vals, pa, pb, pR, off, norb)
    assert np.abs(m.imag).max() == 0.0
    assert np.allclose(m.real, dense.sum(0), rtol=0, atol=1e-15)
    assert np.abs(m.real - m.real.T).max() <= 1e-15 * np.abs(m).max()


def test_bloch_hermitian_at_general_k():
    vals, pa, pb, pR, off, norb = random_symmetric(seed=3)
    m = F.bloch(vals, pa, pb, pR, off, norb, [0.17, -0.31, 0.42])
    assert np.abs(m - m.conj().T).max() <= 1e-14 * np.abs(m).max()


def test_fold_inverts_bloch_on_a_full_grid():
    """Discrete Fourier inversion: with a Gamma-centred n^3 grid, n > 2 max|R|, folding the Bloch images
    returns every M_R exactly up to rounding, with zero imaginary part."""
    vals, pa, pb, pR, off, norb = random_symmetric(seed=11)
    ks = KPointSet.monkhorst_pack(3, 3, 3)
    rho_k = np.stack([F.bloch(vals, pa, pb, pR, off, norb, k) for k in ks.points])
    back, max_imag = F.fold(rho_k, ks.points, ks.weights, pa, pb, pR, off, norb)
    assert np.abs(back - vals).max() <= 1e-14
    assert max_imag <= 1e-14


def test_to_realspace_places_blocks():
    vals, pa, pb, pR, off, norb = random_symmetric(seed=5)
    dense = F.to_realspace(vals, pa, pb, pR, off, norb)
    Rs = [tuple(r) for r in F.offsets(pR)]
    oo = F.orbital_offsets(norb)
    for p in range(len(pa)):
        a, b = pa[p], pb[p]
        blk = dense[Rs.index(tuple(pR[p])), oo[a]:oo[a + 1], oo[b]:oo[b + 1]]
        assert np.array_equal(blk.ravel(), vals[off[p]:off[p + 1]])
    assert np.count_nonzero(dense) == np.count_nonzero(vals)


def test_kpointset_invariants():
    KPointSet([[0, 0, 0], [0.5, 0, 0]], [0.5, 0.5])
    with pytest.raises(ConfigError):
        KPointSet([[0, 0, 0], [0.5, 0, 0]], [0.5, 0.6])
    with pytest.raises(ConfigError):
        KPointSet([[0, 0, 0]], [-1.0])
    with pytest.raises(DimensionError):
        KPointSet([[0, 0, 0]], [0.5, 0.5])
    mp = KPointSet.monkhorst_pack(2, 3, 4)
    assert len(mp.points) == 24 and abs(mp.weights.sum() - 1) < 1e-15


def test_realspace_operator_invariants():
    m = np.array([[1.0, 2.0], [3.0, 4.0]])
    op = RealSpaceOperator(2, [((0, 0, 0), np.eye(2)), ((1, 0, 0), m), ((-1, 0, 0), m.T)])
    op.validate()
    with pytest.raises(ConsistencyError, match=r"R=\(1, 0, 0\)"):
        RealSpaceOperator(2, [((0, 0, 0), np.eye(2)), ((1, 0, 0), m)]).validate()
    with pytest.raises(ConsistencyError, match="R=0"):
        RealSpaceOperator(2, [((1, 0, 0), m), ((-1, 0, 0), m.T)]).validate()
    with pytest.raises(ConsistencyError):
        RealSpaceOperator(2, [((0, 0, 0), m)]).validate()
