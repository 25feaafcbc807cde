"""The CUDA library (libkbgrid, sm_100a) vs the committed golden fixtures of the independent numpy
restatement (tests/golden/make_golden.py): an orthorhombic dimer and a triclinic trimer whose grids are
not multiples of the 4^3 block (ragged edge blocks), with several periodic images of one atom covering
the same block. Fixture style of the reference's test support (seeded inputs, independent naive
restatement as the oracle: /root/reference/proj/tests/test_support.hpp:9-71).

Bar: index lists bit-exact; rho and H within 1e-12 normwise; per element 1e-10 where |ref| > 1e-4
max|ref| and 1e-8 where 1e-8 max|ref| < |ref| <= 1e-4 max|ref| (the two restatements' own rounding,
~n eps sum|terms|, is no longer negligible there); H symmetric bitwise and repeatable bitwise."""
import numpy as np
import pytest

from paper_1402_4247_b200 import _abi
from paper_1402_4247_b200.grid import GridPass

from test_golden import CASES, INDEX_KEYS, load_case  # noqa: E402 (tests/ is on sys.path under pytest)

pytestmark = pytest.mark.gpu


def elementwise(x, ref, floor, ceil=None):
    a = np.abs(ref) / np.abs(ref).max()
    m = (a > floor) & (a <= (ceil if ceil is not None else np.inf))
    return float((np.abs(x - ref)[m] / np.abs(ref)[m]).max()) if m.any() else 0.0


@pytest.mark.parametrize("name", CASES)
def test_gpu_matches_golden(built, name):
    s, z = load_case(name)
    gp = GridPass(s, device=0)
    gp.set_option(_abi.KBG_OPT_DETERMINISTIC, 1)  # bitwise comparisons between calls below
    ix = gp.build_index()
    for k in INDEX_KEYS:
        assert np.array_equal(ix[k].reshape(-1), z[k].reshape(-1)), k
    rho = gp.density(z["dm"][None])[0]
    h = gp.hamiltonian(z["veff"][None], float(z["dV"]))[0]
    assert np.abs(rho - z["rho"]).max() <= 1e-12 * np.abs(z["rho"]).max()
    assert np.abs(h - z["h"]).max() <= 1e-12 * np.abs(z["h"]).max()
    for x, ref in ((rho, z["rho"]), (h, z["h"])):
        assert elementwise(x, ref, 1e-4) <= 1e-10
        assert elementwise(x, ref, 1e-8, 1e-4) <= 1e-8
    # one call with both halves (two streams) gives the same bits as the separate calls
    rho2, h2 = gp.grid_pass(z["dm"][None], z["veff"][None], float(z["dV"]))
    assert np.array_equal(rho2[0], rho) and np.array_equal(h2[0], h)
    assert np.array_equal(gp.hamiltonian(z["veff"][None], float(z["dV"]))[0], h)


@pytest.mark.parametrize("name", CASES)
def test_gpu_golden_symmetry(built, name):
    s, z = load_case(name)
    gp = GridPass(s, device=0)
    ix = gp.build_index()
    h = gp.hamiltonian(z["veff"][None], float(z["dV"]))[0]
    norb = s.norb_of_atom()
    off, mir = ix["pair_off"], ix["pair_mirror"]
    for p in range(len(mir)):
        na, nb = norb[ix["pair_a"][p]], norb[ix["pair_b"][p]]
        q = mir[p]
        assert np.array_equal(h[off[p]:off[p + 1]].reshape(na, nb), h[off[q]:off[q + 1]].reshape(nb, na).T)
