"""Segment times of bench.py's step under variations (diagnostic): python tools/step_probe.py"""
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
    gp = GridPass(f.system, device=0, rank=0, nranks=1)
    gp.set_option(1, 8)
    ix = gp.build_index()
    ix = gp.build_index()
    st = torch.cuda.current_stream()
    d_dm = torch.from_numpy(f.dm(ix, nspin=1)).to(dev)
    d_v = torch.from_numpy(f.veff(nspin=1)).to(dev)
    rho = torch.empty((1, f.system.npts), dtype=torch.float64, device=dev)
    h = torch.empty((1, ix["nnz"]), dtype=torch.float64, device=dev)
    flush = torch.empty((512 << 20) // 4, dtype=torch.float32, device=dev)
    ops = {"rho": lambda: gp.density_dev(d_dm, rho, st),
           "h": lambda: gp.hamiltonian_accumulate_dev(d_v, f.dV, h, st),
           "mirror": lambda: gp.hamiltonian_mirror_dev(h, st)}
    for seq in (("rho", "h", "mirror"), ("h", "rho", "mirror"), ("h",), ("rho",)):
        for sync in (True, False):
            for nrep in (20, 100):
                evs = [[torch.cuda.Event(enable_timing=True) for _ in range(len(seq) + 1)] for _ in range(nrep + 3)]
                torch.cuda.synchronize()
                for rep in range(nrep + 3):
                    flush.zero_()
                    ev = evs[rep]
                    ev[0].record(st)
                    for i, k in enumerate(seq):
                        ops[k]()
                        ev[i + 1].record(st)
                    if sync:
                        ev[-1].synchronize()
                torch.cuda.synchronize()
                ts = [[ev[i].elapsed_time(ev[i + 1]) for i in range(len(seq))] for ev in evs[3:]]
                a = np.array(ts)
                print(json.dumps({"seq": list(seq), "sync_each_step": sync, "steps": nrep,
                                  "median_ms": [round(float(x), 4) for x in np.median(a, axis=0)],
                                  "first5_last5_ms": [[round(float(x), 4) for x in a[:5].mean(axis=0)],
                                                      [round(float(x), 4) for x in a[-5:].mean(axis=0)]]}), flush=True)


if __name__ == "__main__":
    main()
