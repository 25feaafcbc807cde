"""Per-call wall time of kbg_grid_pass (host pointers) on N ranks under variations (diagnostic).
python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tools/e2e_probe.py [config]"""
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1402_4247_b200 import _abi  # noqa: E402
from paper_1402_4247_b200.grid import GridPass  # noqa: E402
from paper_1402_4247_b200.system import Fe3O4  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "cubic56_200Ry"
    world, rank, local = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    f = Fe3O4.config(cfg)
    gp = GridPass(f.system, device=local, rank=rank, nranks=world)
    ix = gp.build_index()
    if world > 1:
        handles = [None] * world
        dist.all_gather_object(handles, gp.comm_handle())
        gp.comm_open(handles)
    nnz, npts = ix["nnz"], f.system.npts
    dm_h, veff_h = f.dm(ix, nspin=1), f.veff(nspin=1)
    dp = C.POINTER(C.c_double)
    lib = gp._lib

    def bufs(pinned):
        mk = (lambda a: torch.from_numpy(a).pin_memory()) if pinned else (lambda a: torch.from_numpy(a.copy()))
        return mk(dm_h), mk(veff_h), mk(np.empty((1, npts))), mk(np.empty((1, nnz)))

    zc = [("", ""), ("1", ""), ("", "1"), ("1", "1")]  # KBG_NO_ZERO_COPY (V in place), ..._OUT (rho in place)
    for shard_io, pinned, zin, zout in [(1, True) + z for z in zc] + [(0, True, "", ""), (1, False, "", "")]:
        gp.set_option(_abi.KBG_OPT_SHARD_IO, shard_io)
        for k, v in (("KBG_NO_ZERO_COPY", zin), ("KBG_NO_ZERO_COPY_OUT", zout)):
            if v:
                os.environ[k] = v
            else:
                os.environ.pop(k, None)
        p_dm, p_v, p_rho, p_h = bufs(pinned)
        if True:
            for barrier in (False,):
                def call():
                    st = lib.kbg_grid_pass(gp.handle, 1, C.cast(p_dm.data_ptr(), dp), C.cast(p_v.data_ptr(), dp), f.dV,
                                           C.cast(p_rho.data_ptr(), dp), C.cast(p_h.data_ptr(), dp))
                    assert st == 0, lib.kbg_last_error(gp.handle)
                for _ in range(3):
                    call()
                ts = []
                for _ in range(20):
                    if barrier and world > 1:
                        dist.barrier()
                    torch.cuda.synchronize()
                    t0 = time.perf_counter()
                    call()
                    ts.append((time.perf_counter() - t0) * 1e3)
                med = float(np.median(ts))
                allm = [None] * world
                if world > 1:
                    dist.all_gather_object(allm, round(med, 4))
                else:
                    allm = [round(med, 4)]
                if rank == 0:
                    print(json.dumps({"config": cfg, "world": world, "shard_io": shard_io, "pinned": pinned,
                                      "no_zero_copy_in": bool(zin), "no_zero_copy_out": bool(zout), "median_ms_per_rank": allm,
                                      "min_ms_rank0": round(min(ts), 4)}), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
