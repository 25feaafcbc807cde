"""Timing experiments (results are WRONG under these flags): what does each part cost?
bit0 H: stores instead of atomics; bit1 H: no scatter; bit2 H: no w multiply;
bit3 rho: DM gathers from one L1-hot address."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1402_4247_b200 import _abi  # noqa: E402
from paper_1402_4247_b200.grid import GridPass  # noqa: E402
from paper_1402_4247_b200.system import Fe3O4  # noqa: E402

f = Fe3O4.config(sys.argv[1] if len(sys.argv) > 1 else "cubic56_200Ry")
gp = GridPass(f.system)
ix = gp.build_index()
dev = torch.device("cuda", 0)
d_dm = torch.from_numpy(f.dm(ix)).to(dev)
d_v = torch.from_numpy(f.veff()).to(dev)
rho = torch.empty((1, f.system.npts), dtype=torch.float64, device=dev)
h = torch.empty((1, ix["nnz"]), dtype=torch.float64, device=dev)
st = torch.cuda.current_stream()
flush = torch.empty(512 << 18, dtype=torch.float32, device=dev)


def t(fn, reps=10):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return round(float(np.median(ts)), 4)


for flag in (0, 1, 2, 4, 6, 8):
    gp.set_option(_abi.KBG_OPT_SCATTER_STORE, flag)
    print(json.dumps({"flag": flag, "density_ms": t(lambda: gp.density_dev(d_dm, rho, st)),
                      "h_ms": t(lambda: gp.hamiltonian_accumulate_dev(d_v, f.dV, h, st))}))
gp.set_option(_abi.KBG_OPT_SCATTER_STORE, 0)
