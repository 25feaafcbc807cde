"""Multi-rank host logic on CPU (gloo, world_size 2): cost-balanced contiguous
block shards, per-rank partial H summed by all_reduce, rho assembled from
shards == the single-rank result. Ranks run the oracle's block-range entry
points (rank emulation)."""
import os
import socket

import numpy as np
import pytest

from paper_1402_4247_b200.shard import block_costs, partition


def test_partition_properties():
    rng = np.random.default_rng(3)
    cost = rng.integers(0, 1000, size=997)
    for n in (1, 2, 3, 4, 8):
        parts = partition(cost, n)
        assert parts[0][0] == 0 and parts[-1][1] == len(cost)
        for (a0, a1), (b0, b1) in zip(parts, parts[1:]):
            assert a1 == b0
        w = cost + 1
        loads = [w[a:b].sum() for a, b in parts]
        assert max(loads) - min(loads) <= 2 * w.max()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist

    from oracle.oracle import Oracle
    from paper_1402_4247_b200 import _abi
    from paper_1402_4247_b200.system import Fe3O4

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    f = Fe3O4(_abi.KBG_CELL_PRIMITIVE, 1, 100.0)
    o = Oracle(f.system)
    ix = o.build_index()
    b0, b1 = partition(block_costs(ix, f.system.norb_of_atom()), world)[rank]
    dm, v = f.dm(ix, nspin=2), f.veff(nspin=2)
    rho = torch.from_numpy(o.density(dm, threads=2, blocks=(b0, b1)))
    h = torch.from_numpy(o.hamiltonian(v, f.dV, threads=2, blocks=(b0, b1)))
    dist.all_reduce(rho)  # shards are disjoint: the sum assembles rho
    dist.all_reduce(h)
    if rank == 0:
        rho_ref = o.density(dm, threads=2)
        h_ref = o.hamiltonian(v, f.dV, threads=2)
        q.put((float(np.abs(rho.numpy() - rho_ref).max() / np.abs(rho_ref).max()),
               float(np.abs(h.numpy() - h_ref).max() / np.abs(h_ref).max()), (b0, b1)))
    dist.destroy_process_group()


def test_two_rank_gloo_matches_single_rank(built):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    e_rho, e_h, rng = res
    assert rng[0] == 0 and rng[1] > 0
    assert e_rho <= 1e-14 and e_h <= 1e-13
