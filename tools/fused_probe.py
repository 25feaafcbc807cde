"""Fused rho + H pass (kbg_grid_pass_dev) vs the separate kernels (density_dev, hamiltonian_accumulate_dev,
hamiltonian_mirror_dev): time per pass (CUDA events, L2 flushed) and agreement; "auto" = the default
KBG_OPT_FUSED_PASS = 2 (fused below the L2 footprint threshold, separate kernels above).
python tools/fused_probe.py [config ...]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1402_4247_b200.grid import GridPass  # noqa: E402
from paper_1402_4247_b200.system import Fe3O4  # noqa: E402


def main(configs):
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream()
    flush = torch.empty((512 << 20) // 4, dtype=torch.float32, device=dev)
    for cfg in configs:
        f = Fe3O4.config(cfg)
        gp = GridPass(f.system)
        ix = gp.build_index()
        dm = torch.from_numpy(f.dm(ix)).to(dev)
        v = torch.from_numpy(f.veff()).to(dev)
        rho = [torch.zeros((1, f.system.npts), dtype=torch.float64, device=dev) for _ in range(2)]
        h = [torch.zeros((1, ix["nnz"]), dtype=torch.float64, device=dev) for _ in range(2)]

        def separate():
            gp.density_dev(dm, rho[0], st)
            gp.hamiltonian_accumulate_dev(v, f.dV, h[0], st)
            gp.hamiltonian_mirror_dev(h[0], st)

        def fused():
            gp.grid_pass_dev(dm, v, f.dV, rho[1], h[1], st)

        from paper_1402_4247_b200 import _abi

        def mode(m, fn):
            def run():
                gp.set_option(_abi.KBG_OPT_FUSED_PASS, m)
                fn()
            return run

        res = {"config": cfg}
        for name, fn in (("separate", separate), ("fused", mode(1, fused)), ("auto", mode(2, fused)),
                         ("separate2", separate), ("fused2", mode(1, fused)), ("auto2", mode(2, fused))):
            for _ in range(3):
                fn()
            ts = []
            for _ in range(20):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                fn()
                e1.record(st)
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            res[name + "_ms"] = round(float(np.median(ts)), 4)
        torch.cuda.synchronize()
        res["rho_bitwise"] = bool(torch.equal(rho[0], rho[1]))
        res["h_rel"] = float((h[0] - h[1]).abs().max() / h[0].abs().max())
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["cubic56_200Ry", "super448_200Ry", "sweep56_100Ry", "sweep56_400Ry"])
