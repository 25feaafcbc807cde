"""GPU parity: libkbgrid (CUDA, sm_100a) vs the CPU oracle on identical bytes.

Bar (BASELINE.json north_star): index lists bit-exact; rho and H within 1e-10
relative, normwise max|d|/max|ref| (the reference's normwise convention,
/root/reference/proj/tests/test_householder.cpp:67), plus per-element relative
1e-10 on entries with |ref| > 1e-4 max|ref|.
"""
import numpy as np
import pytest

from paper_1402_4247_b200 import _abi
from paper_1402_4247_b200.errors import ConfigError, ConsistencyError
from paper_1402_4247_b200.grid import GridPass
from paper_1402_4247_b200.system import Fe3O4

pytestmark = pytest.mark.gpu

INDEX_KEYS = ("blk_ptr", "cov_atom", "cov_R", "cov_mask", "pair_a", "pair_b", "pair_R", "pair_off", "pair_mirror")
TOL = 1e-10


def normwise(x, ref):
    return float(np.abs(x - ref).max() / np.abs(ref).max())


def elementwise(x, ref, floor=1e-4):
    m = np.abs(ref) > floor * np.abs(ref).max()
    return float((np.abs(x - ref)[m] / np.abs(ref)[m]).max())


class Case:
    def __init__(self, name, nspin):
        from oracle.oracle import Oracle

        self.f = Fe3O4.config(name)
        self.gp = GridPass(self.f.system, device=0)
        self.gix = self.gp.build_index()
        self.o = Oracle(self.f.system)
        self.oix = self.o.build_index()
        self.dm = self.f.dm(self.oix, nspin=nspin)
        self.veff = self.f.veff(nspin=nspin)


_cases = {}


def case(name, nspin=1):
    key = (name, nspin)
    if key not in _cases:
        _cases[key] = Case(name, nspin)
    return _cases[key]


@pytest.fixture(scope="module", autouse=True)
def _built(built):
    yield
    _cases.clear()


@pytest.mark.parametrize("name", ["primitive14_150Ry", "sweep56_100Ry", "cubic56_200Ry"])
def test_index_bit_exact(name):
    c = case(name)
    for k in INDEX_KEYS:
        assert np.array_equal(c.gix[k], c.oix[k]), k
    for k in ("nnz", "nbpair", "natompt", "sum_m", "sum_m2"):
        assert c.gix[k] == c.oix[k], k


def test_cubic_index_matches_survey_figures():
    ix = case("cubic56_200Ry").gix
    assert ix["natompt"] == 3_597_832
    assert len(ix["pair_a"]) == 4376 and ix["nnz"] == 470_264
    assert ix["sum_m2"] == 4_146_964_624 or abs(ix["sum_m2"] - 4.147e9) < 1e6


@pytest.mark.parametrize("name,nspin", [("primitive14_150Ry", 1), ("primitive14_150Ry", 2), ("cubic56_200Ry", 1)])
def test_density_parity(name, nspin):
    c = case(name, nspin)
    rho = c.gp.density(c.dm)
    ref = c.o.density(c.dm)
    assert normwise(rho, ref) <= TOL
    assert elementwise(rho, ref) <= TOL


@pytest.mark.parametrize("name,nspin", [("primitive14_150Ry", 1), ("primitive14_150Ry", 2), ("cubic56_200Ry", 1)])
def test_hamiltonian_parity(name, nspin):
    c = case(name, nspin)
    h = c.gp.hamiltonian(c.veff, c.f.dV)
    ref = c.o.hamiltonian(c.veff, c.f.dV)
    assert normwise(h, ref) <= TOL
    assert elementwise(h, ref) <= TOL


def test_block_orbitals_parity():
    c = case("primitive14_150Ry")
    nonempty = np.nonzero(np.diff(c.gix["blk_ptr"]))[0]
    for b in nonempty[:: max(1, len(nonempty) // 7)]:
        phi = c.gp.block_orbitals(int(b))
        ref = c.o.block_orbitals(int(b))
        assert phi.shape == ref.shape
        assert np.abs(phi - ref).max() <= 1e-13 * max(1.0, np.abs(ref).max())


def test_hamiltonian_symmetry_bitwise():
    c = case("primitive14_150Ry")
    h = c.gp.hamiltonian(c.veff, c.f.dV)[0]
    ix, norb = c.gix, c.f.system.norb_of_atom()
    off, mir = ix["pair_off"], ix["pair_mirror"]
    for p in range(len(mir)):
        na, nb = norb[ix["pair_a"][p]], norb[ix["pair_b"][p]]
        q = mir[p]
        assert np.array_equal(h[off[p]:off[p + 1]].reshape(na, nb), h[off[q]:off[q + 1]].reshape(nb, na).T)


def test_density_repeatable_bitwise():
    c = case("primitive14_150Ry")
    r1 = c.gp.density(c.dm)
    r2 = c.gp.density(c.dm)
    assert np.array_equal(r1, r2)


def test_fault_hook_is_caught():
    """kband fault_proc6_sign analogue (householder.hpp:27-28, test_householder.cpp:106-115)."""
    c = case("primitive14_150Ry")
    ref = c.o.hamiltonian(c.veff, c.f.dV)
    c.gp.set_option(_abi.KBG_OPT_FAULT_SIGN, 1)
    try:
        bad = c.gp.hamiltonian(c.veff, c.f.dV)
    finally:
        c.gp.set_option(_abi.KBG_OPT_FAULT_SIGN, 0)
    assert normwise(bad, ref) > 1e-6


def test_errors():
    c = case("primitive14_150Ry")
    with pytest.raises(ConfigError):
        c.gp.density(np.zeros((3, c.gix["nnz"])))
    bad = c.dm.copy()
    bad[0, 0] += 1.0  # breaks DM_ba(-R) = DM_ab(R)^T
    with pytest.raises(ConsistencyError):
        c.gp.density(bad)


@pytest.mark.parametrize("persist", [0, 1])
def test_kernel_modes_agree(persist):
    """Persistent warp-specialized kernels and one-CTA-per-block kernels give the same results."""
    c = case("cubic56_200Ry")
    c.gp.set_option(_abi.KBG_OPT_PERSIST, persist)
    try:
        rho = c.gp.density(c.dm)
        h = c.gp.hamiltonian(c.veff, c.f.dV)
    finally:
        c.gp.set_option(_abi.KBG_OPT_PERSIST, 1)
    assert normwise(rho, c.o.density(c.dm)) <= TOL
    assert normwise(h, c.o.hamiltonian(c.veff, c.f.dV)) <= TOL
