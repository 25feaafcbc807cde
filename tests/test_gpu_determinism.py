"""Deterministic H (KBG_OPT_DETERMINISTIC): bitwise-repeatable results, the reference's core design
value (/root/reference/proj/include/kband/common.hpp:58-64: results "bitwise independent of the team
size"; SPEC.md:307 topology invariance).

Every H contribution is split into two limbs on fixed power-of-two grids derived from max|V| and added
with exact FP64 atomics (kb_gridcore.cuh h_scatter), so the order in which blocks, tasks and kernels
arrive cannot change a bit. The tests check that on the product path and
through properties only an order-independent accumulation has: the one-CTA-per-block kernels and the
persistent kernels (with every intra-block schedule) give the SAME bits, and scaling V by 2^k scales H
by exactly 2^k.
"""
import numpy as np
import pytest

from paper_1402_4247_b200 import _abi
from paper_1402_4247_b200.errors import ConvergenceError
from paper_1402_4247_b200.grid import GridPass
from paper_1402_4247_b200.system import Fe3O4

pytestmark = pytest.mark.gpu


MODES = (1,)


def det_pass(system, mode=1, **kw):
    gp = GridPass(system, device=0, **kw)
    gp.set_option(_abi.KBG_OPT_DETERMINISTIC, mode)
    return gp


class Case:
    def __init__(self, name, nspin, mode=1):
        self.f = Fe3O4.config(name)
        self.gp = det_pass(self.f.system, mode)
        self.ix = self.gp.build_index()
        self.dm = self.f.dm(self.ix, nspin=nspin)
        self.veff = self.f.veff(nspin=nspin)


_cases = {}


def case(name, nspin=1, mode=1):
    if (name, nspin, mode) not in _cases:
        _cases[(name, nspin, mode)] = Case(name, nspin, mode)
    return _cases[(name, nspin, mode)]


@pytest.fixture(scope="module", autouse=True)
def _built(built):
    yield
    _cases.clear()


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("name,nspin", [("cubic56_200Ry", 1), ("primitive14_150Ry", 2), ("sweep56_100Ry", 1)])
def test_hamiltonian_repeatable_bitwise(name, nspin, mode):
    c = case(name, nspin, mode)
    h1 = c.gp.hamiltonian(c.veff, c.f.dV)
    for _ in range(3):
        assert np.array_equal(h1, c.gp.hamiltonian(c.veff, c.f.dV))
    _, h2 = c.gp.grid_pass(c.dm, c.veff, c.f.dV)
    assert np.array_equal(h1, h2)


@pytest.mark.parametrize("mode", MODES)
def test_device_api_repeatable_bitwise(mode):
    import torch

    c = case("cubic56_200Ry", 1, mode)
    dev = torch.device("cuda", 0)
    v = torch.from_numpy(c.veff).to(dev)
    h = torch.empty((1, c.ix["nnz"]), dtype=torch.float64, device=dev)
    c.gp.hamiltonian_dev(v, c.f.dV, h)
    torch.cuda.synchronize()
    first = h.cpu().numpy()
    for _ in range(5):
        c.gp.hamiltonian_dev(v, c.f.dV, h)
        torch.cuda.synchronize()
        assert np.array_equal(first, h.cpu().numpy())
    assert np.array_equal(first, c.gp.hamiltonian(c.veff, c.f.dV))
    # accumulate (canonical blocks) + mirror = the fused finalize/mirror
    c.gp.hamiltonian_accumulate_dev(v, c.f.dV, h)
    c.gp.hamiltonian_mirror_dev(h)
    torch.cuda.synchronize()
    assert np.array_equal(first, h.cpu().numpy())


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("persist,schedule", [(0, 3), (1, 0), (1, 1), (1, 3)])
def test_kernels_and_schedules_same_bits(persist, schedule, mode):
    """Different kernels and work orders, same H bits: the accumulation is order independent."""
    c = case("cubic56_200Ry", 1, mode)
    ref = c.gp.hamiltonian(c.veff, c.f.dV)
    gp = det_pass(c.f.system, mode)
    gp.set_option(_abi.KBG_OPT_SCHEDULE, schedule)
    gp.set_option(_abi.KBG_OPT_PERSIST, persist)
    gp.build_index()
    assert np.array_equal(gp.hamiltonian(c.veff, c.f.dV), ref)


@pytest.mark.parametrize("mode", MODES)
def test_deterministic_matches_fp64_atomics(mode):
    c = case("cubic56_200Ry", 1, mode)
    h_det = c.gp.hamiltonian(c.veff, c.f.dV)
    c.gp.set_option(_abi.KBG_OPT_DETERMINISTIC, 0)
    try:
        h_fp = c.gp.hamiltonian(c.veff, c.f.dV)
        h_fp2 = c.gp.hamiltonian(c.veff, c.f.dV)
    finally:
        c.gp.set_option(_abi.KBG_OPT_DETERMINISTIC, mode)
    assert np.abs(h_fp2 - h_fp).max() <= 1e-14 * np.abs(h_fp).max()
    assert np.abs(h_det - h_fp).max() <= 1e-14 * np.abs(h_fp).max()


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("k", [-7, 3, 40])
def test_power_of_two_scaling_is_exact(k, mode):
    """H(2^k V) = 2^k H(V) bit for bit: the grids move with max|V|, every rounding is the same."""
    c = case("primitive14_150Ry", 1, mode)
    h = c.gp.hamiltonian(c.veff, c.f.dV)
    hk = c.gp.hamiltonian(c.veff * 2.0 ** k, c.f.dV)
    assert np.array_equal(hk, h * 2.0 ** k)


@pytest.mark.parametrize("mode", MODES)
def test_zero_potential_gives_exact_zero(mode):
    c = case("primitive14_150Ry", 1, mode)
    assert not np.any(c.gp.hamiltonian(np.zeros_like(c.veff), c.f.dV))


@pytest.mark.parametrize("det", [1, 0])
@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
def test_nonfinite_potential_raises(bad, det):
    """kband raises ConvergenceError on non-finite values (householder.cpp:119-123): every V value is
    checked (deterministic path: the max|V| pass; FP64-atomic path: the H kernels' V loads)."""
    c = case("primitive14_150Ry")
    c.gp.set_option(_abi.KBG_OPT_DETERMINISTIC, det)
    try:
        for pos in (0, c.veff.shape[1] // 3, c.veff.shape[1] - 1):
            v = c.veff.copy()
            v[0, pos] = bad
            with pytest.raises(ConvergenceError):
                c.gp.hamiltonian(v, c.f.dV)
            with pytest.raises(ConvergenceError):
                c.gp.grid_pass(c.dm, v, c.f.dV)
        # the context stays usable
        h = c.gp.hamiltonian(c.veff, c.f.dV)
        assert np.isfinite(h).all()
    finally:
        c.gp.set_option(_abi.KBG_OPT_DETERMINISTIC, 1)


@pytest.mark.parametrize("name,nspin", [("cubic56_200Ry", 1), ("cubic56_200Ry", 2), ("sweep56_400Ry", 1)])
def test_deterministic_oracle_parity(name, nspin):
    """The deterministic accumulation keeps the parity bar of tests/test_gpu_parity.py against the oracle."""
    from oracle.oracle import Oracle

    from test_gpu_parity import assert_parity

    c = case(name, nspin, 1)
    o = Oracle(c.f.system)
    o.build_index()
    assert_parity(c.gp.hamiltonian(c.veff, c.f.dV), o.hamiltonian(c.veff, c.f.dV))
