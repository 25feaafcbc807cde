"""CPU oracle: index figures, physics identities, determinism.

These pin the oracle before it is trusted as the checker: the index figures
match SURVEY.md 8(a)/8(d) (derived there by an independent numpy probe), and
the identities 8(c)1-6 and 9 hold.
"""
import numpy as np
import pytest

from paper_1402_4247_b200 import _abi
from paper_1402_4247_b200.system import Fe3O4, Species, System, radial_table


@pytest.fixture(scope="module")
def prim(built):
    from oracle.oracle import Oracle

    f = Fe3O4.config("primitive14_150Ry")
    o = Oracle(f.system)
    ix = o.build_index()
    return f, o, ix


def blocks_of(ix, norb, p):
    off = ix["pair_off"]
    a, b = ix["pair_a"][p], ix["pair_b"][p]
    return off[p], off[p + 1], norb[a], norb[b]


def trace_dm_x(ix, norb, dm, x):
    """sum_ab Tr(DM_ab(R) X_ba(-R))"""
    tot = 0.0
    mir = ix["pair_mirror"]
    for p in range(len(mir)):
        s0, s1, na, nb = blocks_of(ix, norb, p)
        q = mir[p]
        t0, t1, _, _ = blocks_of(ix, norb, q)
        tot += np.sum(dm[s0:s1].reshape(na, nb) * x[t0:t1].reshape(nb, na).T)
    return tot


def test_primitive_index_matches_survey(prim):
    f, o, ix = prim
    assert f.system.grid == (45, 45, 45) and f.system.natom == 14 and f.system.nbasis == 142
    assert ix["natompt"] == 877_088
    assert len(ix["pair_a"]) == 1094 and ix["nnz"] == 117_566
    assert ix["sum_m2"] == 1_008_327_984


def test_cubic_index_matches_survey(built):
    from oracle.oracle import Oracle

    f = Fe3O4.config("cubic56_200Ry")
    ix = Oracle(f.system).build_index()
    assert f.system.grid == (72, 72, 72) and f.system.nbasis == 568
    assert ix["natompt"] == 3_597_832
    assert len(ix["pair_a"]) == 4376 and ix["nnz"] == 470_264
    assert abs(ix["sum_m2"] - 4.147e9) / 4.147e9 < 1e-3
    assert abs(ix["sum_m"] - 38_949_896) < 1


def test_electron_count_identity(prim):
    """8(c)1: sum_r rho dV = sum_ab Tr(DM_ab S_ba)."""
    f, o, ix = prim
    dm = f.dm(ix)
    rho = o.density(dm)
    S = o.hamiltonian(np.ones((1, f.system.npts)), f.dV)
    ne = rho.sum() * f.dV
    tr = trace_dm_x(ix, f.system.norb_of_atom(), dm[0], S[0])
    assert abs(ne - tr) <= 1e-12 * max(1.0, abs(ne))


def test_energy_identity(prim):
    """8(c)2: sum_r rho V dV = sum_ab Tr(DM_ab H_ba)."""
    f, o, ix = prim
    dm, v = f.dm(ix), f.veff()
    rho = o.density(dm)
    H = o.hamiltonian(v, f.dV)
    e = (rho * v).sum() * f.dV
    tr = trace_dm_x(ix, f.system.norb_of_atom(), dm[0], H[0])
    assert abs(e - tr) <= 1e-12 * max(1.0, abs(e))


def test_constant_potential_gives_scaled_overlap(prim):
    """8(c)3: V = c -> H = c S; S symmetric positive definite, S_ii ~ 1."""
    f, o, ix = prim
    S = o.hamiltonian(np.ones((1, f.system.npts)), f.dV)[0]
    H = o.hamiltonian(np.full((1, f.system.npts), -2.5), f.dV)[0]
    assert np.abs(H + 2.5 * S).max() <= 2e-12 * np.abs(S).max()
    norb = f.system.norb_of_atom()
    # on-site blocks (a, a, 0): symmetric, SPD, diagonal ~ 1 (quadrature of normalised orbitals)
    for p in np.nonzero((ix["pair_a"] == ix["pair_b"]) & (np.abs(ix["pair_R"]).sum(1) == 0))[0]:
        s0, s1, na, _ = blocks_of(ix, norb, p)
        B = S[s0:s1].reshape(na, na)
        assert np.abs(B - B.T).max() <= 1e-14 * np.abs(B).max()
        assert np.linalg.eigvalsh(0.5 * (B + B.T)).min() > 0
        assert np.all(np.abs(np.diag(B) - 1.0) < 0.05)


def test_hamiltonian_symmetry(prim):
    """8(c)6: H_ba(-R) = H_ab(R)^T (the oracle sums every ordered pair directly)."""
    f, o, ix = prim
    H = o.hamiltonian(f.veff(), f.dV)[0]
    norb = f.system.norb_of_atom()
    mx = np.abs(H).max()
    for p, q in enumerate(ix["pair_mirror"]):
        s0, s1, na, nb = blocks_of(ix, norb, p)
        t0, t1, _, _ = blocks_of(ix, norb, q)
        assert np.abs(H[s0:s1].reshape(na, nb) - H[t0:t1].reshape(nb, na).T).max() <= 1e-14 * mx


def test_thread_count_does_not_change_bits(prim):
    """8(c)9 / kband test_linalg.cpp:40-46."""
    f, o, ix = prim
    dm, v = f.dm(ix), f.veff()
    assert np.array_equal(o.density(dm, threads=1), o.density(dm, threads=5))
    assert np.array_equal(o.hamiltonian(v, f.dV, threads=1), o.hamiltonian(v, f.dV, threads=3))


def single_s_system(grid=(20, 20, 20), L=12.0, pos=(3.0, 4.5, 6.0)):
    tab = radial_table(0, 0.7, 4.0, 512)[None]
    sp = Species(l=[0], rc=4.0, table=tab)
    return System(lattice=np.eye(3) * L, grid=grid, species_of_atom=[0], tau=[pos], species=[sp])


def test_single_s_orbital_density_is_phi_squared(built):
    """8(c)4: one s orbital, DM = 1 -> rho = phi^2 with the analytic radial function."""
    from oracle.oracle import Oracle

    s = single_s_system()
    o = Oracle(s)
    ix = o.build_index()
    dm = np.ones((1, ix["nnz"]))  # single pair (0,0,0), 1x1
    assert len(ix["pair_a"]) == 1
    rho = o.density(dm)[0].reshape(s.grid)
    N, L, rc, alpha = 20, 12.0, 4.0, 0.7
    i, j, k = np.meshgrid(*[np.arange(N)] * 3, indexing="ij")
    r = np.stack([i, j, k], -1) / N * L - np.array([3.0, 4.5, 6.0])
    r = (r + L / 2) % L - L / 2  # minimum image (rc < L/2)
    d = np.sqrt((r ** 2).sum(-1))
    tab = radial_table(0, alpha, rc, 4096)
    # normalisation constant from the table at r=0 (u(0) = N)
    nrm = tab[0, 0]
    u = np.where(d < rc, nrm * np.exp(-alpha * d * d) * (1 - (d / rc) ** 2) ** 3, 0.0)
    phi = 0.28209479177387814 * u
    assert np.abs(rho - phi ** 2).max() <= 1e-9 * (phi ** 2).max()


def test_shift_by_grid_vector_permutes_exactly(built):
    """8(c)5: shifting every atom by one grid vector permutes the masks/lists."""
    from oracle.oracle import Oracle

    N, L = 24, 12.0
    s1 = single_s_system(grid=(N, N, N), L=L, pos=(3.0, 4.5, 6.0))
    s2 = single_s_system(grid=(N, N, N), L=L, pos=(3.0, 4.5, 6.0 + 4 * L / N))  # 4 points = 1 block along z
    o1, o2 = Oracle(s1), Oracle(s2)
    ix1, ix2 = o1.build_index(), o2.build_index()
    dm = np.ones((1, 1))
    r1 = o1.density(dm)[0].reshape(N, N, N)
    r2 = o2.density(dm)[0].reshape(N, N, N)
    assert np.abs(np.roll(r1, 4, axis=2) - r2).max() <= 1e-12 * r1.max()
    assert ix1["natompt"] == ix2["natompt"]


def test_errors_follow_kband_taxonomy(built):
    from oracle.oracle import Oracle
    from paper_1402_4247_b200.errors import ConfigError

    s = single_s_system()
    o = Oracle(s)
    o.build_index()
    with pytest.raises(ConfigError):
        o.density(np.ones((3, 1)))
    bad = single_s_system()
    bad.species_of_atom[0] = 5
    with pytest.raises(ConfigError):
        Oracle(bad)
