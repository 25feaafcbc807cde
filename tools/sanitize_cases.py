"""Small GPU cases for compute-sanitizer (tools/gpurun/gpurun_sanitize.sh, "Race
detection / sanitizers"). Each case runs the product path on cuda:0 and checks a property of the
result, so a case that runs clean under the sanitizer also computed the right thing.

python tools/sanitize_cases.py smoke|eigen|veff|formats
  smoke    __graft_entry__.smoke(): 14-atom Fe3O4 grid pass (index, rho, H) vs the oracle
  eigen    eigen_hh of random Hermitian n = 96 (per-column back transform) and, with SAN_BIG=1,
           n = 1030 (blocked WY back transform); residual and orthonormality
  veff     V_eff from the grid-pass rho (Poisson + LSDA), nspin 1 and 2; finite, spin-symmetric
  formats  RealSpaceOperator round trip (bit-exact) and Bloch transform Hermiticity
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _hermitian(n, seed):
    r = np.random.default_rng(seed)
    a = r.standard_normal((n, n)) + 1j * r.standard_normal((n, n))
    return (a + a.conj().T) / 2


def case_smoke():
    import __graft_entry__ as g

    g.smoke()


def case_eigen():
    from paper_1402_4247_b200 import eigen as E

    sizes = [96] + ([1030] if os.environ.get("SAN_BIG") == "1" else [])
    for n in sizes:
        a = _hermitian(n, n)
        w, c = E.eigen_hh(a)
        nrm = np.linalg.norm(a)
        res = np.abs(a @ c - c * w).max() / nrm
        orth = np.abs(c.conj().T @ c - np.eye(n)).max()
        assert res <= 1e-9 and orth <= 1e-9, (n, res, orth)
        print(f"ok: eigen_hh n={n} residual {res:.2e} orthonormality {orth:.2e}")


def case_veff():
    from paper_1402_4247_b200.grid import GridPass
    from paper_1402_4247_b200.system import Fe3O4

    f = Fe3O4.config("primitive14_150Ry")
    gp = GridPass(f.system)
    ix = gp.build_index()
    rho = np.abs(gp.density(f.dm(ix)))
    v1, e1 = gp.veff(rho)
    v2, e2 = gp.veff(np.concatenate([rho / 2, rho / 2]))
    assert np.isfinite(v1).all() and np.isfinite(v2).all()
    assert np.array_equal(v2[0], v2[1]), "equal spin densities must give equal spin potentials"
    print(f"ok: veff nspin 1/2, E_H {e1[0]:.6e}, E_x {e1[1]:.6e}")


def case_formats():
    from paper_1402_4247_b200.formats import bloch_transform, from_realspace_operator, to_realspace_operator
    from paper_1402_4247_b200.grid import GridPass
    from paper_1402_4247_b200.system import Fe3O4

    f = Fe3O4.config("primitive14_150Ry")
    gp = GridPass(f.system)
    gp.build_index()
    h = gp.hamiltonian(f.veff(), f.dV)[0]
    op = to_realspace_operator(gp, h)
    assert np.array_equal(from_realspace_operator(gp, op), h)
    hk = bloch_transform(gp, h, np.array([[0.0, 0.0, 0.0], [0.25, 0.5, 0.125]]))
    herm = max(np.abs(m - m.conj().T).max() for m in hk) / np.abs(hk).max()
    assert herm <= 1e-13, herm
    print(f"ok: formats round trip bit-exact, H(k) Hermitian to {herm:.1e}")


if __name__ == "__main__":
    globals()["case_" + sys.argv[1]]()
