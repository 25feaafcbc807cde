"""Where do the persistent kernels' warps spend their time? (KBG_OPT_DEBUG_COUNTERS)"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1402_4247_b200 import _abi  # noqa: E402
from paper_1402_4247_b200.grid import GridPass  # noqa: E402
from paper_1402_4247_b200.system import Fe3O4  # noqa: E402


def main(cfg="cubic56_200Ry"):
    f = Fe3O4.config(cfg)
    gp = GridPass(f.system)
    ix = gp.build_index()
    dev = torch.device("cuda", 0)
    d_dm = torch.from_numpy(f.dm(ix)).to(dev)
    d_v = torch.from_numpy(f.veff()).to(dev)
    rho = torch.empty((1, f.system.npts), dtype=torch.float64, device=dev)
    h = torch.empty((1, ix["nnz"]), dtype=torch.float64, device=dev)
    st = torch.cuda.current_stream()
    for name, fn in (("density", lambda: gp.density_dev(d_dm, rho, st)),
                     ("hamiltonian", lambda: gp.hamiltonian_accumulate_dev(d_v, f.dV, h, st))):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        gp.set_option(_abi.KBG_OPT_DEBUG_COUNTERS, 1)
        fn()
        torch.cuda.synchronize()
        out = (C.c_int64 * 12)()
        gp._lib.kbg_debug_counters(gp.handle, out, 12)
        p_wait, p_tot, c_wait, c_tail, c_tot, blocks, c_start, cp_lat, ncopy, _, red, cp_bytes = list(out)
        print(json.dumps({"kernel": name, "producer_wait_frac": round(p_wait / max(1, p_tot), 3),
                          "consumer_wait_frac": round(c_wait / max(1, c_tot), 3),
                          "consumer_tail_frac": round(c_tail / max(1, c_tot), 3),
                          "consumer_start_frac": round(c_start / max(1, c_tot), 3),
                          "copy_latency_cycles": round(cp_lat / max(1, ncopy)),
                          "copy_bytes_avg": round(cp_bytes / max(1, ncopy)),
                          "reduce_release_cycles": round(red / max(1, ncopy)),
                          "cycles_per_block_per_sm": round(p_tot / max(1, ncopy)),
                          "consumer_blocks": blocks, "consumer_cycles": c_tot}))


if __name__ == "__main__":
    main(*sys.argv[1:])
