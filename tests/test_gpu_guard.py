"""Out-of-bounds write guard for the device entry points ("Race detection /
sanitizers"). compute-sanitizer is closed on the GPU pool, so every output of kbg_density_dev,
kbg_hamiltonian_dev and kbg_veff_dev is written into the middle of a larger device buffer whose red
zones (GUARD doubles on each side) hold a sentinel bit pattern; after the call the red zones must be
untouched and the result must match the host API's (rho and V_eff within 1e-14, H within 1e-13
normwise: atomics)."""
import numpy as np
import pytest

from paper_1402_4247_b200.grid import GridPass
from paper_1402_4247_b200.system import Fe3O4

pytestmark = pytest.mark.gpu
GUARD = 4096
SENTINEL = 0x7FF4DEADBEEF1402  # bit pattern of a signalling NaN (no kernel produces it)


def guarded(torch, shape):
    n = int(np.prod(shape))
    buf = torch.full((n + 2 * GUARD,), SENTINEL, dtype=torch.int64, device="cuda").view(torch.float64)
    return buf, buf[GUARD:GUARD + n].view(*shape)


def red_zones_intact(torch, buf):
    bits = buf.view(torch.int64).cpu().numpy()
    return bool((bits[:GUARD] == SENTINEL).all() and (bits[-GUARD:] == SENTINEL).all())


@pytest.mark.parametrize("name,nspin", [("primitive14_150Ry", 1), ("primitive14_150Ry", 2), ("cubic56_200Ry", 1)])
def test_device_outputs_stay_in_bounds(built, name, nspin):
    import torch

    f = Fe3O4.config(name)
    gp = GridPass(f.system)
    ix = gp.build_index()
    dm = np.atleast_2d(f.dm(ix, nspin=nspin))
    veff = np.atleast_2d(f.veff(nspin=nspin))
    npts, nnz = veff.shape[1], dm.shape[1]

    dm_buf, dm_d = guarded(torch, dm.shape)
    dm_d.copy_(torch.from_numpy(dm))
    v_buf, v_d = guarded(torch, veff.shape)
    v_d.copy_(torch.from_numpy(veff))
    rho_buf, rho_d = guarded(torch, (nspin, npts))
    h_buf, h_d = guarded(torch, (nspin, nnz))
    ve_buf, ve_d = guarded(torch, (nspin, npts))

    gp.density_dev(dm_d, rho_d)
    gp.hamiltonian_dev(v_d, f.dV, h_d)
    torch.cuda.synchronize()
    rho_pos = rho_d.abs().contiguous()
    gp.veff_dev(rho_pos, ve_d)
    torch.cuda.synchronize()

    for what, buf in (("dm", dm_buf), ("veff in", v_buf), ("rho", rho_buf), ("H", h_buf), ("V_eff out", ve_buf)):
        assert red_zones_intact(torch, buf), f"{what}: a kernel wrote outside its buffer"
    rho_ref = gp.density(dm)
    h_ref = gp.hamiltonian(veff, f.dV)
    assert np.abs(rho_d.cpu().numpy() - rho_ref).max() <= 1e-14 * np.abs(rho_ref).max()
    assert np.abs(h_d.cpu().numpy() - h_ref).max() <= 1e-13 * np.abs(h_ref).max()
    v_ref, _ = gp.veff(rho_pos.cpu().numpy())
    assert np.abs(ve_d.cpu().numpy() - v_ref).max() <= 1e-14 * np.abs(v_ref).max()


@pytest.mark.parametrize("n", [1, 33, 1030])
def test_eigen_outputs_stay_in_bounds(built, n):
    """kbg_hh_eigen (host buffers) writes exactly n eigenvalues and n x n eigenvector entries: the
    per-column back transform (n < 1024) and the blocked WY one (n = 1030)."""
    from paper_1402_4247_b200 import _abi
    from paper_1402_4247_b200 import eigen as E

    r = np.random.default_rng(n)
    a = r.standard_normal((n, n)) + 1j * r.standard_normal((n, n))
    a = np.ascontiguousarray((a + a.conj().T) / 2)
    wbuf = np.full(n + 2 * GUARD, SENTINEL, dtype=np.int64).view(np.float64)
    cbuf = np.full(2 * (n * n + 2 * GUARD), SENTINEL, dtype=np.int64).view(np.complex128)
    w, c = wbuf[GUARD:GUARD + n], cbuf[GUARD:GUARD + n * n].reshape(n, n)
    st = _abi.kbgrid().kbg_hh_eigen(n, E._cptr(a), 1, _abi.dptr(w), E._cptr(c))
    assert st == 0, _abi.kbgrid().kbg_hh_last_error().decode()
    for what, buf in (("w", wbuf.view(np.int64)), ("c", cbuf.view(np.int64))):
        g = 2 * GUARD if what == "c" else GUARD
        assert (buf[:g] == SENTINEL).all() and (buf[-g:] == SENTINEL).all(), f"kbg_hh_eigen wrote outside {what}"
    assert np.abs(a @ c - c * w).max() <= 1e-9 * np.linalg.norm(a)
