"""GPU tridiagonal eigensolver (kb_tridiag.cu: Sturm multisection + inverse iteration) against the
reference's own kband::solve_tridiag (implicit QL, oracle/_ref) and the reference's test contract
(/root/reference/proj/tests/test_tridiag.cpp): decoupled diagonal exact, n = 1, the Chebyshev spectrum
to 1e-13, residual ||T v - lambda v|| <= 1e-11 scale, unitarity defect <= 1e-12, trace, ascending order;
plus eigenvalues within 1e-12 scale of the reference, repeated eigenvalues, and eigen_hh end to end."""
import numpy as np
import pytest

from oracle import kband_ref as R
from paper_1402_4247_b200 import eigen as E
from paper_1402_4247_b200.errors import DimensionError

pytestmark = [pytest.mark.gpu]


@pytest.fixture(scope="module", autouse=True)
def _built(built):
    yield


def check_contract(d, e, w, z, scale):
    n = len(d)
    t = np.diag(d) + np.diag(e, 1) + np.diag(e, -1)
    assert np.all(np.diff(w) >= 0)
    assert abs(w.sum() - d.sum()) <= 1e-11 * n * max(1.0, np.abs(np.concatenate([d, e])).max())
    if z is not None:
        res = np.linalg.norm(t @ z - z * w, axis=0).max()
        assert res <= 1e-11 * scale, res
        assert np.abs(z.T @ z - np.eye(n)).max() <= 1e-12


def test_decoupled_diagonal_and_n1():
    w, z = E.gpu_solve_tridiag(np.array([4.0, 2.0, 7.0]), np.array([0.0, 0.0]), True)
    assert np.array_equal(w, [2.0, 4.0, 7.0])
    check_contract(np.array([4.0, 2.0, 7.0]), np.zeros(2), w, z, 7.0)
    w1, z1 = E.gpu_solve_tridiag(np.array([-3.5]), np.zeros(0), True)
    assert np.array_equal(w1, [-3.5]) and z1[0, 0] == 1.0


def test_chebyshev_spectrum():
    w, _ = E.gpu_solve_tridiag(np.zeros(4), np.ones(3), False)
    expect = 2 * np.cos(np.arange(4, 0, -1) * np.pi / 5)
    assert np.abs(w - expect).max() <= 1e-13 * 2


@pytest.mark.parametrize("n", [2, 3, 9, 33, 300, 1040])
def test_random_problems_match_reference(n):
    rng = np.random.default_rng(77 + n)
    d, e = rng.uniform(-2, 2, n), rng.uniform(-2, 2, n - 1)
    w, z = E.gpu_solve_tridiag(d, e, True)
    check_contract(d, e, w, z, 4.0)
    if R.available():
        wr, _ = R.solve_tridiag(d, e, False)
        assert np.abs(w - wr).max() <= 1e-12 * 4.0


def test_repeated_eigenvalues():
    """Block-diagonal copies of one 3x3 block: every eigenvalue 4-fold; the vectors of each cluster are
    re-orthogonalized."""
    blk_d, blk_e = np.array([1.0, -0.5, 2.0]), np.array([0.7, -0.3])
    d = np.tile(blk_d, 4)
    e = np.concatenate([np.concatenate([blk_e, [0.0]]) for _ in range(4)])[:-1]
    w, z = E.gpu_solve_tridiag(d, e, True)
    check_contract(d, e, w, z, 3.0)
    ref = np.linalg.eigvalsh(np.diag(blk_d) + np.diag(blk_e, 1) + np.diag(blk_e, -1))
    assert np.abs(w - np.repeat(ref, 4)).max() <= 1e-13 * 3


def test_errors():
    with pytest.raises(DimensionError):
        E.gpu_solve_tridiag(np.zeros(3), np.zeros(1), True)


@pytest.mark.skipif(not R.available(), reason="reference kband library not built")
@pytest.mark.parametrize("n", [97, 568])
def test_eigen_hh_with_gpu_solver(n):
    rng = np.random.default_rng(5 + n)
    x = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    a = 0.5 * (x + x.conj().T)
    nrm = np.linalg.norm(a)
    w, c = E.eigen_hh(a, True, solve_tridiag=E.gpu_solve_tridiag)
    wr, _ = R.eigen_hh(a, False)
    assert np.abs(w - wr).max() <= 1e-11 * nrm
    assert np.linalg.norm(a @ c - c * w) <= 1e-9 * nrm
    assert np.abs(c.conj().T @ c - np.eye(n)).max() <= 1e-9


def test_eigen_hh_small_and_diagonal():
    """kbg_hh_eigen edge cases: 1x1, 2x2, and a diagonal matrix (every Householder stage skipped)."""
    w1, c1 = E.eigen_hh(np.array([[2.5 + 0j]]))
    assert np.array_equal(w1, [2.5]) and abs(abs(c1[0, 0]) - 1.0) <= 1e-15
    a2 = np.array([[1.0, 2.0 - 1.0j], [2.0 + 1.0j, -3.0]])
    w2, c2 = E.eigen_hh(a2)
    assert np.abs(w2 - np.linalg.eigvalsh(a2)).max() <= 1e-13
    assert np.abs(a2 @ c2 - c2 * w2).max() <= 1e-13
    dg = np.diag([3.0, -1.0, 2.0, 0.5, -1.0]).astype(np.complex128)
    wd, cd = E.eigen_hh(dg)
    assert np.allclose(wd, [-1.0, -1.0, 0.5, 2.0, 3.0], atol=1e-15)
    assert np.abs(dg @ cd - cd * wd).max() <= 1e-14
    assert np.abs(cd.conj().T @ cd - np.eye(5)).max() <= 1e-13
