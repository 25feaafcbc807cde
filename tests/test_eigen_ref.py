"""CPU: the reference's own kband eigensolver (oracle/_ref/libkband_ref.so, compiled from
/root/reference/proj/src) is the checker of the GPU Eigen_HH. Pin the shim: its
results against numpy's LAPACK and the reference's own test expectations (test_householder.cpp)."""
import numpy as np
import pytest

from oracle import kband_ref as R

pytestmark = pytest.mark.skipif(not R.available(), reason="reference kband library not built (needs /root/reference)")


def hermitian(n, seed):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    return 0.5 * (x + x.conj().T)


@pytest.mark.parametrize("n", [1, 2, 8, 33])
def test_reference_eigen_hh_matches_lapack(n):
    a = hermitian(n, n)
    w, v = R.eigen_hh(a)
    assert np.abs(w - np.linalg.eigvalsh(a)).max() <= 1e-12 * max(1.0, np.linalg.norm(a))
    assert np.abs(a @ v - v * w).max() <= 1e-10 * np.linalg.norm(a)


def test_reference_record_invariants():
    """test_householder.cpp:71-87: u zero through the stage, |u|^2 = 2h, |phase| = 1."""
    a = hermitian(12, 3)
    d, e, u, h, s, ph = R.tridiagonalize(a)
    for i in range(11):
        assert np.all(u[i, :i + 1] == 0)
        assert abs(np.vdot(u[i], u[i]).real - 2 * h[i]) <= 1e-12 * 2 * h[i]
        assert abs(abs(ph[i]) - 1) <= 1e-14


def test_reference_fault_hook_breaks_spectrum():
    """test_householder.cpp:106-115."""
    a = hermitian(10, 5)
    d, e, *_ = R.tridiagonalize(a, fault_sign=True)
    w, _ = R.solve_tridiag(d, e, False)
    assert np.abs(np.sort(w) - np.linalg.eigvalsh(a)).max() > 1e-6 * np.linalg.norm(a)
