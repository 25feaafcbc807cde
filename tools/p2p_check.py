"""Multi-GPU check of the fused H reduction over peer memory (kb_comm.cu).

torchrun --nproc-per-node N tools/p2p_check.py [config]
Every rank: sharded context, kbg_hamiltonian_allreduce_dev -> full H. Checks (rank 0 prints one JSON line):
identical bits on every rank; equal to the NCCL path (accumulate + mirror + all_reduce) within 1e-14;
equal to the single-context full H within 1e-13; repeatable bitwise; times both collectives.
"""
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1402_4247_b200.grid import GridPass  # noqa: E402
from paper_1402_4247_b200.system import Fe3O4  # noqa: E402


def main(cfg="cubic56_200Ry"):
    world, rank, local = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    f = Fe3O4.config(cfg)
    gp = GridPass(f.system, device=local, rank=rank, nranks=world)
    ix = gp.build_index()
    handles = [None] * world
    dist.all_gather_object(handles, gp.comm_handle())
    gp.comm_open(handles)
    st = torch.cuda.current_stream()
    v = torch.from_numpy(f.veff()).to(dev)
    h_p2p = torch.empty((1, ix["nnz"]), dtype=torch.float64, device=dev)
    h_nccl = torch.empty_like(h_p2p)

    def p2p():
        gp.hamiltonian_allreduce_dev(v, f.dV, h_p2p, st)

    def nccl():
        gp.hamiltonian_dev(v, f.dV, h_nccl, st)
        dist.all_reduce(h_nccl)

    p2p()
    nccl()
    torch.cuda.synchronize()
    first = h_p2p.clone()
    p2p()
    torch.cuda.synchronize()
    repeat = bool(torch.equal(first, h_p2p))
    sums = [None] * world
    dist.all_gather_object(sums, hashlib.sha256(h_p2p.cpu().numpy().tobytes()).hexdigest())
    same_bits = len(set(sums)) == 1
    d_nccl = float((h_p2p - h_nccl).abs().max() / h_nccl.abs().max())

    def timeit(fn, reps=20):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            dist.barrier()
            e0.record(st)
            fn()
            e1.record(st)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = torch.tensor([float(np.median(ts))], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    t_p2p = timeit(p2p)
    t_nccl = timeit(nccl)
    t_acc = timeit(lambda: gp.hamiltonian_accumulate_dev(v, f.dV, h_nccl, st))
    if rank == 0:
        full = GridPass(f.system, device=local)
        full.build_index()
        ref = full.hamiltonian(f.veff(), f.dV)[0]
        d_full = float(np.abs(h_p2p.cpu().numpy()[0] - ref).max() / np.abs(ref).max())
        print(json.dumps({"config": cfg, "world": world, "same_bits_all_ranks": same_bits, "repeatable": repeat,
                          "rel_diff_vs_nccl": d_nccl, "rel_diff_vs_single_gpu": d_full,
                          "h_ms_p2p": round(t_p2p, 4), "h_ms_nccl_incl_mirror": round(t_nccl, 4),
                          "h_ms_accumulate_only": round(t_acc, 4),
                          "note": "H partials use atomics: not bitwise repeatable run to run (single GPU neither)",
                          "ok": bool(same_bits and d_nccl <= 1e-14 and d_full <= 1e-13)}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main(*sys.argv[1:])
