"""H accumulate time vs the placement of the H output buffer (diagnostic): python tools/hbuf_probe.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1402_4247_b200.grid import GridPass  # noqa: E402
from paper_1402_4247_b200.system import Fe3O4  # noqa: E402


def main():
    f = Fe3O4.config("cubic56_200Ry")
    dev = torch.device("cuda", 0)
    gp = GridPass(f.system)
    ix = gp.build_index()
    scatter = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    if scatter:  # timing experiment (needs a -DKBG_EXPERIMENTS=1 library): 1 plain stores, 2 no scatter
        from paper_1402_4247_b200 import _abi
        gp.set_option(_abi.KBG_OPT_SCATTER_STORE, scatter)
    st = torch.cuda.current_stream()
    d_v = torch.from_numpy(f.veff(nspin=1)).to(dev)
    flush = torch.empty((512 << 20) // 4, dtype=torch.float32, device=dev)
    bufs = []
    for k in range(12):
        bufs.append(torch.empty((1, ix["nnz"]), dtype=torch.float64, device=dev))
        torch.empty((1 + 3 * k) << 19, dtype=torch.uint8, device=dev)  # shift the next allocation
    big = torch.empty((64 << 20) // 8, dtype=torch.float64, device=dev)
    for off in range(0, 8 * (1 << 20) // 8 + 1, (1 << 20) // 8):  # offsets inside one big buffer, 1 MB steps
        bufs.append(big[off:off + ix["nnz"]].view(1, -1))
    import ctypes as C
    lib = C.CDLL(os.path.join(ROOT, "tools", "probe", "libredprobe.so"))
    lib.red_probe.restype = C.c_float
    lib.red_probe.argtypes = [C.c_void_p, C.c_int64, C.c_int]
    for i, h in enumerate(bufs):
        red_ms = lib.red_probe(h.data_ptr(), h.numel(), 8)
        ts = []
        for rep in range(13):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            gp.hamiltonian_accumulate_dev(d_v, f.dV, h, st)
            e1.record(st)
            e1.synchronize()
            if rep >= 3:
                ts.append(e0.elapsed_time(e1))
        print(json.dumps({"buf": i, "addr_mb": round((h.data_ptr() % (1 << 40)) / 2**20, 3),
                          "h_ms": round(float(np.median(ts)), 4), "red_probe_ms": round(red_ms, 4), "scatter_exp": scatter}), flush=True)


if __name__ == "__main__":
    main()
