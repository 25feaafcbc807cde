"""GPU parity of the format converters (kb_formats.cu) against oracle/formats.py on the
Fe3O4 pair lists: RealSpaceOperator conversion (bit-exact, a pure copy), Bloch transform and the
real-space folding of density matrices (normwise <= 1e-13; FP64 phases from sincospi vs numpy cos/sin),
plus size-independent properties: Hermiticity of M(k) and fold(bloch(M)) = M on a full k grid."""
import numpy as np
import pytest

from oracle import formats as F
from paper_1402_4247_b200.errors import ConsistencyError
from paper_1402_4247_b200.formats import (KPointSet, bloch_transform, density_matrices_k, fold_density_matrices,
                                          from_realspace_operator, to_realspace_operator)
from paper_1402_4247_b200.grid import GridPass
from paper_1402_4247_b200.system import Fe3O4

pytestmark = pytest.mark.gpu
TOL = 1e-13

_cache = {}


def setup(name):
    if name not in _cache:
        f = Fe3O4.config(name)
        gp = GridPass(f.system)
        ix = gp.build_index()
        dm = f.dm(ix)[0]
        h = gp.hamiltonian(f.veff(), f.dV)[0]
        args = (ix["pair_a"], ix["pair_b"], ix["pair_R"].reshape(-1, 3), ix["pair_off"], f.system.norb_of_atom())
        _cache[name] = (f, gp, ix, dm, h, args)
    return _cache[name]


@pytest.fixture(scope="module", autouse=True)
def _built(built):
    yield
    _cache.clear()


def normwise(x, ref):
    return float(np.abs(x - ref).max() / np.abs(ref).max())


@pytest.mark.parametrize("name", ["primitive14_150Ry", "cubic56_200Ry"])
def test_realspace_roundtrip_bit_exact(name):
    f, gp, ix, dm, h, args = setup(name)
    assert np.array_equal(gp.offsets(), F.offsets(args[2]))
    dense = gp.to_realspace(h)
    assert np.array_equal(dense, F.to_realspace(h, *args))
    assert np.array_equal(gp.from_realspace(dense), h)
    op = to_realspace_operator(gp, h)
    op.validate()
    assert np.array_equal(from_realspace_operator(gp, op), h)


@pytest.mark.parametrize("name", ["primitive14_150Ry", "cubic56_200Ry"])
def test_bloch_parity(name):
    f, gp, ix, dm, h, args = setup(name)
    ks = np.array([[0, 0, 0], [0.5, 0, 0], [0.13, -0.27, 0.41], [0.25, 0.25, 0.25]])
    out = bloch_transform(gp, h, ks)
    for k, m in zip(ks, out):
        ref = F.bloch(h, *args, k)
        assert normwise(m, ref) <= TOL
        assert np.abs(m - m.conj().T).max() <= 1e-14 * np.abs(m).max()  # validated Hermitian
    # Gamma: sum over R, real
    assert np.abs(out[0].imag).max() == 0.0


def test_bloch_rejects_non_hermitian_naming_the_pair():
    f, gp, ix, dm, h, args = setup("primitive14_150Ry")
    bad = h.copy()
    bad[ix["pair_off"][5] + 1] += 1.0
    with pytest.raises(ConsistencyError, match=r"pair \d+ .*R=\("):
        bloch_transform(gp, bad, [0.1, 0.2, 0.3])


@pytest.mark.parametrize("name", ["primitive14_150Ry", "cubic56_200Ry"])
def test_fold_inverts_bloch(name):
    """Full Gamma-centred grid with n_i > 2 max|R_i|: fold(bloch(DM)) = DM, imaginary part ~ 0."""
    f, gp, ix, dm, h, args = setup(name)
    R = gp.offsets()
    n = [int(2 * np.abs(R[:, i]).max() + 1) for i in range(3)]
    ks = KPointSet.monkhorst_pack(*n)
    rho_k = bloch_transform(gp, dm, ks.points)
    back = fold_density_matrices(gp, rho_k, ks)
    assert normwise(back, dm) <= 1e-13


def test_fold_parity_general_kset():
    f, gp, ix, dm, h, args = setup("primitive14_150Ry")
    rng = np.random.default_rng(1402)
    n = gp.nbasis()
    ks = KPointSet(np.array([[0.1, 0.2, 0.3], [-0.1, -0.2, -0.3], [0.4, 0.0, 0.25]]), np.array([0.25, 0.25, 0.5]))
    rho_k = rng.uniform(-1, 1, (3, n, n)) + 1j * rng.uniform(-1, 1, (3, n, n))
    got, mi = gp.fold(rho_k, ks.points, ks.weights)
    ref, ref_mi = F.fold(rho_k, ks.points, ks.weights, *args)
    assert normwise(got, ref) <= TOL
    assert abs(mi - ref_mi) <= 1e-12 * ref_mi
    with pytest.raises(ConsistencyError):
        fold_density_matrices(gp, rho_k, ks)  # random rho_k: imaginary part does not vanish


def test_device_variants_match_host():
    import torch

    f, gp, ix, dm, h, args = setup("primitive14_150Ry")
    dev = torch.device("cuda", 0)
    n = gp.nbasis()
    ks = np.array([[0.1, 0.2, 0.3], [0.0, 0.5, 0.0]])
    d_h = torch.from_numpy(h).to(dev)
    d_out = torch.empty((2, n, n, 2), dtype=torch.float64, device=dev)
    gp.bloch_dev(d_h, ks, d_out)
    d_back = torch.empty_like(d_h)
    gp.fold_dev(d_out, ks, np.array([0.5, 0.5]), d_back)
    d_dense = torch.empty((len(gp.offsets()), n, n), dtype=torch.float64, device=dev)
    gp.to_realspace_dev(d_h, d_dense)
    d_h2 = torch.empty_like(d_h)
    gp.from_realspace_dev(d_dense, d_h2)
    torch.cuda.synchronize()
    host = gp.bloch(h, ks)
    assert np.array_equal(d_out.cpu().numpy().view(np.complex128)[..., 0], host)
    assert np.array_equal(d_back.cpu().numpy(), gp.fold(host, ks, np.array([0.5, 0.5]))[0])
    assert np.array_equal(d_h2.cpu().numpy(), h)


def _states(n, m, seed):
    rng = np.random.default_rng(seed)
    z = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    q, _ = np.linalg.qr(z)  # orthonormal columns: C^H S C = I with S = I
    return q[:, :m]


def test_density_matrix_k_parity_and_spec_examples():
    """rho_k = sum_i f_i c_i c_i^dagger; step occupation -> c1c1^dagger + c2c2^dagger;
    f = 0 -> rho = 0; trace identity Tr(rho_k S_k) = sum_i f_i (S = I, orthonormal states)."""
    f_, gp, ix, dm, h, args = setup("primitive14_150Ry")
    n = gp.nbasis()
    C = _states(n, 40, 5)
    f = 1.0 / (1.0 + np.exp(np.linspace(-3, 3, 40)))
    eps = np.linspace(-1, 1, 40)
    rho, E = density_matrices_k(gp, C, f, eps)
    ref = (C * f) @ C.conj().T
    assert normwise(rho, ref) <= TOL
    assert normwise(E, (C * (eps * f)) @ C.conj().T) <= TOL
    assert np.abs(rho - rho.conj().T).max() <= 1e-14 * np.abs(rho).max()
    assert abs(np.trace(rho).real - f.sum()) <= 1e-10
    step = np.zeros(4)
    step[:2] = 1.0
    C4 = _states(n, 4, 9)
    r2 = gp.density_matrix_k(C4, step)
    exact = np.outer(C4[:, 0], C4[:, 0].conj()) + np.outer(C4[:, 1], C4[:, 1].conj())
    assert np.abs(r2 - exact).max() <= 1e-14
    assert np.abs(gp.density_matrix_k(C4, np.zeros(4))).max() == 0.0


def test_part6_chain_to_grid_density():
    """States at every k of a full grid -> rho_k (GPU) -> fold (GPU) -> grid density (GPU): the grid
    electron count sum_r rho(r) dV equals sum_ab Tr(DM_ab S_ba) (SURVEY.md 8(c) identity 1)."""
    f_, gp, ix, dm, h, args = setup("primitive14_150Ry")
    n = gp.nbasis()
    ks = KPointSet.monkhorst_pack(2, 2, 2)
    rho_k = []
    for i, k in enumerate(ks.points):
        C = _states(n, 30, 100 + i)
        rho_k.append(gp.density_matrix_k(C, np.full(30, 0.5)))
    # time-reversal partner of each k on this grid is itself (k = -k mod 1): symmetrise
    rho_k = np.stack([0.5 * (r + r.conj()) for r in rho_k])
    dm_pairs = fold_density_matrices(gp, rho_k, ks)
    # the folded DM must satisfy the grid pass's DM invariant to be accepted (symmetrise over R <-> -R)
    mir = ix["pair_mirror"]
    norb = f_.system.norb_of_atom()
    sym = dm_pairs.copy()
    for p in range(len(mir)):
        q = mir[p]
        na, nb = norb[ix["pair_a"][p]], norb[ix["pair_b"][p]]
        blk = dm_pairs[ix["pair_off"][p]:ix["pair_off"][p + 1]].reshape(na, nb)
        other = dm_pairs[ix["pair_off"][q]:ix["pair_off"][q + 1]].reshape(nb, na)
        sym[ix["pair_off"][p]:ix["pair_off"][p + 1]] = (0.5 * (blk + other.T)).ravel()
    rho = gp.density(sym)[0]
    S = gp.hamiltonian(np.ones(f_.system.npts), f_.dV)[0]
    tr = 0.0
    for p in range(len(mir)):
        q = mir[p]
        na, nb = norb[ix["pair_a"][p]], norb[ix["pair_b"][p]]
        tr += np.sum(sym[ix["pair_off"][p]:ix["pair_off"][p + 1]].reshape(na, nb)
                     * S[ix["pair_off"][q]:ix["pair_off"][q + 1]].reshape(nb, na).T)
    assert abs(rho.sum() * f_.dV - tr) <= 1e-10 * max(1.0, abs(tr))
