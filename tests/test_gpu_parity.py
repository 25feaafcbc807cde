"""GPU parity: libkbgrid (CUDA, sm_100a) vs the CPU oracle on identical bytes.

Bar (BASELINE.json north_star): index lists bit-exact; rho and H within 1e-10
relative, normwise max|d|/max|ref| (the reference's normwise convention,
/root/reference/proj/tests/test_householder.cpp:67), plus per-element relative
error on every entry with |ref| > 1e-8 max|ref| (hard part 8):
<= 1e-10 above 1e-4 max|ref|, <= ELEM_TOL_SMALL between 1e-8 and 1e-4 max|ref|
(there the oracle's own rounding, ~n eps sum|terms|, is no longer negligible
against |ref|).
"""
import numpy as np
import pytest

from paper_1402_4247_b200 import _abi
from paper_1402_4247_b200.errors import ConfigError, ConsistencyError, ConvergenceError
from paper_1402_4247_b200.grid import GridPass
from paper_1402_4247_b200.system import Fe3O4

pytestmark = pytest.mark.gpu

INDEX_KEYS = ("blk_ptr", "cov_atom", "cov_R", "cov_mask", "pair_a", "pair_b", "pair_R", "pair_off", "pair_mirror")
TOL = 1e-10


def normwise(x, ref):
    return float(np.abs(x - ref).max() / np.abs(ref).max())


ELEM_TOL_SMALL = 1e-8


def elementwise(x, ref, floor=1e-4, ceil=None):
    """max relative error over the entries with floor < |ref| / max|ref| (<= ceil)."""
    a = np.abs(ref) / np.abs(ref).max()
    m = a > floor
    if ceil is not None:
        m &= a <= ceil
    if not m.any():
        return 0.0
    return float((np.abs(x - ref)[m] / np.abs(ref)[m]).max())


def assert_parity(x, ref):
    assert normwise(x, ref) <= TOL
    assert elementwise(x, ref, 1e-4) <= TOL
    assert elementwise(x, ref, 1e-8, 1e-4) <= ELEM_TOL_SMALL


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


@pytest.mark.parametrize("name", ["primitive14_150Ry", "sweep56_100Ry", "cubic56_200Ry", "super448_200Ry",
                                  "super1512_200Ry"])
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


PARITY_CASES = [("primitive14_150Ry", 1), ("primitive14_150Ry", 2), ("cubic56_200Ry", 1), ("cubic56_200Ry", 2)]


@pytest.mark.parametrize("name,nspin", PARITY_CASES)
def test_density_parity(name, nspin):
    c = case(name, nspin)
    assert_parity(c.gp.density(c.dm), c.o.density(c.dm))


@pytest.mark.parametrize("name,nspin", PARITY_CASES)
def test_hamiltonian_parity(name, nspin):
    c = case(name, nspin)
    assert_parity(c.gp.hamiltonian(c.veff, c.f.dV), c.o.hamiltonian(c.veff, c.f.dV))


def test_supercell448_full_parity():
    """Config 3 (448 atoms, 144^3 points) against the oracle over the whole grid: rho and H."""
    c = case("super448_200Ry")
    assert_parity(c.gp.density(c.dm), c.o.density(c.dm))
    assert_parity(c.gp.hamiltonian(c.veff, c.f.dV), c.o.hamiltonian(c.veff, c.f.dV))


@pytest.mark.parametrize("nranks,ranks", [(40, (0, 19, 39))])
def test_supercell1512_sampled_parity(nranks, ranks):
    """Config 4 (1512 atoms, 216^3 points): a full oracle pass is minutes of host time, so the
    comparison is on samples -- a sharded context of `nranks` owns a contiguous, cost-balanced ~1/40
    of the blocks; its rho (owned points, others 0) and its partial H (the contributions of its blocks,
    mirrored) must match the oracle run over exactly the same block range. Three shards: both ends of
    the grid (periodic wrap-around images) and the middle."""
    from oracle.oracle import Oracle

    f = Fe3O4.config("super1512_200Ry")
    o = Oracle(f.system)
    oix = o.build_index()
    dm = f.dm(oix)
    veff = f.veff()
    for r in ranks:
        gp = GridPass(f.system, device=0, rank=r, nranks=nranks)
        gp.build_index()
        b0, b1 = gp.shard_range()
        assert 0 <= b0 < b1 <= oix["nblock"]
        assert_parity(gp.density(dm), o.density(dm, blocks=(b0, b1)))
        assert_parity(gp.hamiltonian(veff, f.dV), o.hamiltonian(veff, f.dV, blocks=(b0, b1)))
        gp.close()


@pytest.mark.parametrize("name", ["primitive14_150Ry", "cubic56_200Ry"])
def test_block_orbitals_bit_exact(name):
    """G2 (A2): the orbital values of a block are the oracle's bit for bit -- the device evaluation
    (kb_device.cuh eval_orbitals_pair) uses explicit round-to-nearest operations in the oracle's
    expression order (oracle compiled with -ffp-contract=off)."""
    c = case(name)
    nonempty = np.nonzero(np.diff(c.gix["blk_ptr"]))[0]
    for b in nonempty[:: max(1, len(nonempty) // 9)]:
        phi = c.gp.block_orbitals(int(b))
        ref = c.o.block_orbitals(int(b))
        assert phi.shape == ref.shape
        assert np.array_equal(phi, ref), f"block {b}: max |d| {np.abs(phi - ref).max():.3e}"


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


@pytest.mark.parametrize("schedule", [0, 1, 2])
def test_schedules_agree(schedule):
    """Static LPT lists and the per-block task queue (KBG_OPT_SCHEDULE) give the same results; rho stays
    bitwise deterministic under the queue (per-task partial sums reduced in task order)."""
    c = case("cubic56_200Ry")
    gp = GridPass(c.f.system)
    gp.set_option(_abi.KBG_OPT_SCHEDULE, schedule)
    gp.build_index()
    rho = gp.density(c.dm)
    h = gp.hamiltonian(c.veff, c.f.dV)
    assert np.array_equal(rho, gp.density(c.dm))
    assert normwise(rho, c.gp.density(c.dm)) <= 1e-14
    assert normwise(h, c.gp.hamiltonian(c.veff, c.f.dV)) <= 1e-13
    with pytest.raises(ConfigError):
        gp.set_option(_abi.KBG_OPT_SCHEDULE, 4)


def test_sharded_contexts_sum_to_full():
    """Two rank contexts on one GPU: disjoint rho shards and partial H sum to the full pass."""
    from paper_1402_4247_b200.shard import block_costs, partition

    c = case("primitive14_150Ry")
    rho_full = c.gp.density(c.dm)
    h_full = c.gp.hamiltonian(c.veff, c.f.dV)
    parts = []
    for r in range(2):
        gp = GridPass(c.f.system, device=0, rank=r, nranks=2)
        gp.build_index()
        parts.append((gp.shard_range(), gp.density(c.dm), gp.hamiltonian(c.veff, c.f.dV)))
    assert parts[0][0][0] == 0 and parts[0][0][1] == parts[1][0][0] and parts[1][0][1] == c.gix["nblock"]
    assert [p[0] for p in parts] == partition(block_costs(c.gix, c.f.system.norb_of_atom()), 2)
    rho = parts[0][1] + parts[1][1]
    h = parts[0][2] + parts[1][2]
    assert normwise(rho, rho_full) <= 1e-14
    assert normwise(h, h_full) <= 1e-13


def test_grid_pass_matches_separate_calls():
    """kbg_grid_pass (rho and H on two streams, overlapped copies) = kbg_density + kbg_hamiltonian."""
    c = case("cubic56_200Ry")
    rho, h = c.gp.grid_pass(c.dm, c.veff, c.f.dV)
    assert np.array_equal(rho, c.gp.density(c.dm))
    assert normwise(h, c.gp.hamiltonian(c.veff, c.f.dV)) <= 1e-14
    assert normwise(h, c.o.hamiltonian(c.veff, c.f.dV)) <= TOL
    bad = c.dm.copy()
    bad[0, 1] += 1.0  # pair 0 is (0, 0, R=0) here: break its transpose symmetry off the diagonal
    with pytest.raises(ConsistencyError):
        c.gp.grid_pass(bad, c.veff, c.f.dV)
    bad = c.dm.copy()
    bad[0, c.gix["pair_off"][len(c.gix["pair_off"]) // 2] + 3] = np.nan  # a non-canonical or canonical pair
    with pytest.raises(ConvergenceError):
        c.gp.grid_pass(bad, c.veff, c.f.dV)
    bad = c.dm.copy()
    p = int(np.nonzero(c.gix["pair_mirror"] != np.arange(len(c.gix["pair_mirror"])))[0][-1])  # last a != b or R != 0 pair
    bad[0, c.gix["pair_off"][p]] += 1e-6  # its mirror block no longer matches
    with pytest.raises(ConsistencyError):
        c.gp.grid_pass(bad, c.veff, c.f.dV)


def test_device_api_matches_host_api():
    import torch

    c = case("primitive14_150Ry", 2)
    dev = torch.device("cuda", 0)
    d_dm = torch.from_numpy(c.dm).to(dev)
    d_v = torch.from_numpy(c.veff).to(dev)
    rho = torch.empty((2, c.f.system.npts), dtype=torch.float64, device=dev)
    h = torch.empty((2, c.gix["nnz"]), dtype=torch.float64, device=dev)
    c.gp.density_dev(d_dm, rho)
    c.gp.hamiltonian_dev(d_v, c.f.dV, h)
    torch.cuda.synchronize()
    assert np.array_equal(rho.cpu().numpy(), c.gp.density(c.dm))
    assert normwise(h.cpu().numpy(), c.gp.hamiltonian(c.veff, c.f.dV)) <= 1e-14


@pytest.mark.parametrize("name", ["sweep56_100Ry", "sweep56_250Ry", "sweep56_400Ry"])
def test_cutoff_sweep_parity(name):
    """Config 5 (grid-cutoff sweep) end points: coarser and finer grids than configs[1]."""
    c = case(name)
    assert normwise(c.gp.density(c.dm), c.o.density(c.dm)) <= TOL
    assert normwise(c.gp.hamiltonian(c.veff, c.f.dV), c.o.hamiltonian(c.veff, c.f.dV)) <= TOL


def test_large_config_identities():
    """448-atom 2x2x2 supercell at full size (config 3): size-independent properties --
    electron-count identity sum rho dV = Tr(DM S) and H_ba(-R) = H_ab(R)^T."""
    f = Fe3O4.config("super448_200Ry")
    gp = GridPass(f.system)
    ix = gp.build_index()
    dm = f.dm(ix)
    rho = gp.density(dm)[0]
    S = gp.hamiltonian(np.ones((1, f.system.npts)), f.dV)[0]
    norb = f.system.norb_of_atom()
    off, mir = ix["pair_off"], ix["pair_mirror"]
    tr = 0.0
    for p in range(len(mir)):
        na, nb = norb[ix["pair_a"][p]], norb[ix["pair_b"][p]]
        q = mir[p]
        Sq = S[off[q]:off[q + 1]].reshape(nb, na)
        assert np.array_equal(S[off[p]:off[p + 1]].reshape(na, nb), Sq.T)
        tr += np.sum(dm[0, off[p]:off[p + 1]].reshape(na, nb) * Sq.T)
    ne = rho.sum() * f.dV
    assert abs(ne - tr) <= 1e-10 * max(1.0, abs(ne))


def test_largest_config_identities():
    """1512-atom 3x3x3 supercell at full size (config 5, 216^3 points): electron count
    sum rho dV = sum DM.S and energy sum rho V dV = sum DM.H over the pair-sparse blocks (both
    orientations stored), and H_ba(-R) = H_ab(R)^T on a sample of the ~118 k pairs."""
    f = Fe3O4.config("super1512_200Ry")
    gp = GridPass(f.system)
    ix = gp.build_index()
    dm = f.dm(ix)
    veff = f.veff()
    rho = gp.density(dm)[0]
    S = gp.hamiltonian(np.ones((1, f.system.npts)), f.dV)[0]
    H = gp.hamiltonian(veff, f.dV)[0]
    ne, e = rho.sum() * f.dV, float(np.dot(rho, veff[0])) * f.dV
    assert abs(ne - float(np.dot(dm[0], S))) <= 1e-10 * abs(ne)
    assert abs(e - float(np.dot(dm[0], H))) <= 1e-10 * np.abs(rho * veff[0]).sum() * f.dV
    norb = f.system.norb_of_atom()
    off, mir = ix["pair_off"], ix["pair_mirror"]
    for p in range(0, len(mir), 97):
        na, nb = norb[ix["pair_a"][p]], norb[ix["pair_b"][p]]
        q = mir[p]
        assert np.array_equal(H[off[p]:off[p + 1]].reshape(na, nb), H[off[q]:off[q + 1]].reshape(nb, na).T)


@pytest.mark.parametrize("name", ["sweep56_100Ry", "cubic56_200Ry", "super448_200Ry"])
def test_plan_uses_task_queues(name):
    """The persistent kernels with both task queues (schedule 3) fit shared memory on the sweep's
    coarsest grid and the supercell: the rho queue's per-task sums are sized by the rho task count
    (the H count is ~2.4x larger and had pushed these configs onto the ~30 % slower static lists)."""
    f = Fe3O4.config(name)
    gp = GridPass(f.system)
    gp.build_index()
    plan = gp.plan_info()
    assert plan["persist"] == 1 and plan["schedule"] == 3, plan
    assert max(plan["smem_h"], plan["smem_rho"]) <= 227 * 1024, plan


@pytest.mark.parametrize("name,nspin", [("cubic56_200Ry", 1), ("primitive14_150Ry", 2)])
def test_grid_pass_pinned_zero_copy(name, nspin):
    """Pinned (mapped) host V is read in place by the persistent H kernel (no H2D copy of V):
    the same H as from pageable buffers, rho unchanged bitwise."""
    import torch

    c = case(name, nspin)
    dm_p = torch.from_numpy(c.dm).pin_memory().numpy()
    v_p = torch.from_numpy(c.veff).pin_memory().numpy()
    rho_p, h_p = c.gp.grid_pass(dm_p, v_p, c.f.dV)
    rho, h = c.gp.grid_pass(c.dm, c.veff, c.f.dV)
    assert np.array_equal(rho_p, rho)
    assert normwise(h_p, h) <= 1e-14
    assert normwise(h_p, c.o.hamiltonian(c.veff, c.f.dV)) <= TOL
    assert normwise(c.gp.hamiltonian(v_p, c.f.dV), h) <= 1e-14


@pytest.mark.parametrize("name,thr", [("sweep56_100Ry", 255), ("cubic56_200Ry", 128)])
def test_sparse_dfma_switch_parity(name, thr):
    """A5's switch (KBG_OPT_SPARSE_DFMA): tasks below the point-density threshold run point-exact FP64
    FMAs instead of DMMA (255: every task). Same H within rounding, oracle parity kept."""
    c = case(name)
    h_dmma = c.gp.hamiltonian(c.veff, c.f.dV)
    c.gp.set_option(_abi.KBG_OPT_SPARSE_DFMA, thr)
    try:
        h = c.gp.hamiltonian(c.veff, c.f.dV)
    finally:
        c.gp.set_option(_abi.KBG_OPT_SPARSE_DFMA, 0)
    assert normwise(h, h_dmma) <= 1e-13
    assert_parity(h, c.o.hamiltonian(c.veff, c.f.dV))


@pytest.mark.parametrize("fused,nspin", [(0, 1), (1, 1), (1, 2), (2, 1), (2, 2)])
def test_grid_pass_dev_matches_separate_kernels(fused, nspin):
    """kbg_grid_pass_dev (separate kernels, or the fused rho + H persistent kernel with
    KBG_OPT_FUSED_PASS = 1, or 2 = auto by L2 footprint, the default): rho bitwise equal to kbg_density_dev, H equal to the mirrored H within the
    FP64-atomic order difference."""
    import torch

    c = case("cubic56_200Ry", nspin)
    dev = torch.device("cuda", 0)
    dm = torch.from_numpy(c.dm).to(dev)
    v = torch.from_numpy(c.veff).to(dev)
    rho0 = torch.zeros((nspin, c.f.system.npts), dtype=torch.float64, device=dev)
    h0 = torch.zeros((nspin, c.gix["nnz"]), dtype=torch.float64, device=dev)
    c.gp.density_dev(dm, rho0)
    c.gp.hamiltonian_dev(v, c.f.dV, h0)
    rho1, h1 = torch.zeros_like(rho0), torch.zeros_like(h0)
    c.gp.set_option(_abi.KBG_OPT_FUSED_PASS, fused)
    try:
        c.gp.grid_pass_dev(dm, v, c.f.dV, rho1, h1)
        torch.cuda.synchronize()
    finally:
        c.gp.set_option(_abi.KBG_OPT_FUSED_PASS, 2)
    assert torch.equal(rho0, rho1)
    assert float((h1 - h0).abs().max() / h0.abs().max()) <= 1e-14
    assert_parity(h1.cpu().numpy(), c.o.hamiltonian(c.veff, c.f.dV))


@pytest.mark.parametrize("bad", [-1, 3])
def test_fused_pass_option_range(bad):
    """KBG_OPT_FUSED_PASS takes 0, 1 or 2 (auto); anything else is a configuration error."""
    c = case("cubic56_200Ry", 1)
    with pytest.raises(ConfigError):
        c.gp.set_option(_abi.KBG_OPT_FUSED_PASS, bad)
    c.gp.set_option(_abi.KBG_OPT_FUSED_PASS, 2)
