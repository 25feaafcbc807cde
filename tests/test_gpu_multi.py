"""Multi-GPU H over peer memory (kb_comm.cu): runs tools/p2p_check.py under torchrun when the box has
>= 2 GPUs (skipped otherwise; the driver's GPU tier has one). Checks: identical bits on every rank,
<= 1e-14 of the NCCL all-reduce path, <= 1e-13 of the single-GPU H."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus():
    try:
        import torch

        return torch.cuda.device_count()
    except Exception:
        return 0


@pytest.mark.gpu
@pytest.mark.skipif(_ngpus() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("nspin,xsms", [(1, 0), (2, 8)])
def test_p2p_reduce_mirror_two_ranks(built, nspin, xsms):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(29531 + nspin), os.path.join(ROOT, "tools", "p2p_check.py")]
    env = dict(os.environ, P2P_NSPIN=str(nspin), P2P_XSMS=str(xsms))
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
    rec = json.loads(line)
    assert rec["ok"], rec


@pytest.mark.gpu
def test_p2p_missing_peer_fails_loudly(built):
    """Two sharded contexts in one process on one GPU (direct-pointer peers): only rank 0 runs the
    exchange, so its kernels give up after 10 s instead of hanging, and kbg_comm_check reports
    KBG_ERR_NCCL instead of handing back an invalid H."""
    import torch

    from paper_1402_4247_b200.errors import CollectiveError
    from paper_1402_4247_b200.grid import GridPass
    from paper_1402_4247_b200.system import Fe3O4

    f = Fe3O4.config("primitive14_150Ry")
    gps = [GridPass(f.system, device=0, rank=r, nranks=2) for r in range(2)]
    for gp in gps:
        gp.build_index()
    handles = [gp.comm_handle() for gp in gps]
    for gp in gps:
        gp.comm_open(handles)
    ix = gps[0].build_index()
    dev = torch.device("cuda", 0)
    v = torch.from_numpy(f.veff()).to(dev)
    h = torch.empty((1, ix["nnz"]), dtype=torch.float64, device=dev)
    gps[0].hamiltonian_allreduce_dev(v, f.dV, h)
    torch.cuda.synchronize()
    with pytest.raises(CollectiveError):
        gps[0].comm_check()


def _two_rank_contexts(name, det=1):
    from paper_1402_4247_b200 import _abi
    from paper_1402_4247_b200.grid import GridPass
    from paper_1402_4247_b200.system import Fe3O4

    f = Fe3O4.config(name)
    gps = [GridPass(f.system, device=0, rank=r, nranks=2) for r in range(2)]
    for gp in gps:
        gp.set_option(_abi.KBG_OPT_DETERMINISTIC, det)
        gp.set_option(_abi.KBG_OPT_EXCHANGE_SMS, 8)  # both ranks' exchange CTAs fit on one GPU
        gp.build_index()
    handles = [gp.comm_handle() for gp in gps]
    for gp in gps:
        gp.comm_open(handles)
    return f, gps


@pytest.mark.gpu
@pytest.mark.parametrize("nspin", [1, 2])
def test_two_ranks_on_one_gpu_exchange_matches_single_gpu(built, nspin):
    """The sharded H path (kb_comm.cu) on the driver's 1-GPU tier: two ranks' contexts on one GPU with
    direct-pointer peers, each exchange on 8 SMs of its own (KBG_OPT_EXCHANGE_SMS), so both are resident
    at once. With the deterministic accumulation the exchanged H equals the single-GPU H bit for bit on
    both ranks, and the ranks' rho points sum to the single-GPU rho exactly."""
    import numpy as np
    import torch

    from paper_1402_4247_b200 import _abi
    from paper_1402_4247_b200.grid import GridPass

    f, gps = _two_rank_contexts("cubic56_200Ry")
    ix = gps[0].build_index()
    dev = torch.device("cuda", 0)
    v = torch.from_numpy(f.veff(nspin=nspin)).to(dev)
    dm = torch.from_numpy(f.dm(ix, nspin=nspin)).to(dev)
    hs = [torch.empty((nspin, ix["nnz"]), dtype=torch.float64, device=dev) for _ in gps]
    rhos = [torch.zeros((nspin, f.system.npts), dtype=torch.float64, device=dev) for _ in gps]
    streams = [torch.cuda.Stream(device=dev) for _ in gps]
    for rep in range(2):
        for gp, st in zip(gps, streams):
            gp.hamiltonian_partial_dev(v, f.dV, st)
        for gp, h, st in zip(gps, hs, streams):
            gp.hamiltonian_exchange_dev(h, st)
        for gp, rho, st in zip(gps, rhos, streams):
            gp.density_dev(dm, rho, st)
        torch.cuda.synchronize()
        for gp in gps:
            gp.comm_check()
    single = GridPass(f.system, device=0)
    single.set_option(_abi.KBG_OPT_DETERMINISTIC, 1)
    single.build_index()
    h_ref = single.hamiltonian(f.veff(nspin=nspin), f.dV)
    rho_ref = single.density(f.dm(ix, nspin=nspin))
    for h in hs:
        assert np.array_equal(h.cpu().numpy(), h_ref)
    # each rank writes rho at its own points only (the rest stays as initialised: zeros)
    assert np.array_equal((rhos[0] + rhos[1]).cpu().numpy(), rho_ref)
