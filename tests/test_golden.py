"""Oracle vs the committed golden fixtures of an independent numpy restatement
(tests/golden/make_golden.py). Index lists bit-exact; rho/H within 1e-12."""
import os

import numpy as np
import pytest

from paper_1402_4247_b200.system import Species, System

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
CASES = ["dimer_ortho", "trimer_triclinic"]
INDEX_KEYS = ("blk_ptr", "cov_atom", "cov_R", "cov_mask", "pair_a", "pair_b", "pair_R", "pair_off", "pair_mirror")


def load_case(name):
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    species = []
    i = 0
    while f"sp{i}_l" in z:
        species.append(Species(l=list(z[f"sp{i}_l"]), rc=float(z[f"sp{i}_rc"]), table=z[f"sp{i}_table"]))
        i += 1
    s = System(lattice=z["lattice"], grid=tuple(z["grid"]), species_of_atom=z["spc"], tau=z["tau"], species=species)
    return s, z


@pytest.mark.parametrize("name", CASES)
def test_oracle_matches_golden(built, name):
    from oracle.oracle import Oracle

    s, z = load_case(name)
    o = Oracle(s)
    ix = o.build_index()
    for k in INDEX_KEYS:
        assert np.array_equal(ix[k].reshape(-1), z[k].reshape(-1)), k
    rho = o.density(z["dm"][None])[0]
    h = o.hamiltonian(z["veff"][None], float(z["dV"]))[0]
    assert np.abs(rho - z["rho"]).max() <= 1e-12 * np.abs(z["rho"]).max()
    assert np.abs(h - z["h"]).max() <= 1e-12 * np.abs(z["h"]).max()
