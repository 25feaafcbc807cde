"""Two sharded contexts on one GPU driven from two host threads through kbg_grid_pass (diagnostic for
tests/test_gpu_multi.py): python tools/two_rank_probe.py  (env: KBG_NO_DM_GATHER, KBG_NO_ZERO_COPY, ...)"""
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1402_4247_b200 import _abi  # noqa: E402
from paper_1402_4247_b200.grid import GridPass  # noqa: E402
from paper_1402_4247_b200.system import Fe3O4  # noqa: E402


def main():
    f = Fe3O4.config(sys.argv[1] if len(sys.argv) > 1 else "cubic56_200Ry")
    xsms = int(os.environ.get("XSMS", "8"))
    gps = [GridPass(f.system, device=0, rank=r, nranks=2) for r in range(2)]
    for gp in gps:
        gp.set_option(_abi.KBG_OPT_EXCHANGE_SMS, xsms)
        gp.build_index()
    handles = [gp.comm_handle() for gp in gps]
    for gp in gps:
        gp.comm_open(handles)
    ix = gps[0].build_index()
    pin = (lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()) if os.environ.get("PIN", "1") == "1" \
        else (lambda a: np.ascontiguousarray(a).copy())
    dm, veff = pin(f.dm(ix)), pin(f.veff())
    outs = [(pin(np.zeros((1, f.system.npts))), pin(np.zeros((1, ix["nnz"])))) for _ in range(2)]
    errs = [None, None]
    t = [0.0, 0.0]

    def worker(r):
        t0 = time.time()
        try:
            gps[r].grid_pass(dm, veff, f.dV, out=outs[r])
        except Exception as e:  # noqa: BLE001
            errs[r] = repr(e)[:120]
        t[r] = time.time() - t0
    ts = [threading.Thread(target=worker, args=(r,)) for r in range(2)]
    for th in ts:
        th.start()
    for th in ts:
        th.join()
    env = {k: v for k, v in os.environ.items() if k.startswith("KBG_") or k in ("XSMS", "PIN")}
    print(env, "errors:", errs, "seconds:", [round(x, 3) for x in t], flush=True)


if __name__ == "__main__":
    main()
