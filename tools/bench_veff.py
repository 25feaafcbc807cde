"""Measurement of V_eff from rho (kb_veff.cu) and of one full SCF grid iteration.

python tools/bench_veff.py [--configs cubic56_200Ry,super448_200Ry,super1512_200Ry]
Per config: kbg_veff_dev (device-resident; CUDA events, median of 10, L2 flushed): rho_total + D2Z +
Poisson + Z2D + V_eff/energies. Compulsory HBM bytes = 8 npts (rho) + 8 npts (V_loc) + 8 npts (V_eff)
plus the FFT round trip (read/write of the real grid and the half spectrum, ~4 x 8 npts); numpy
oracle on the host for comparison. For the 56-atom cell also one full SCF grid iteration on the
device: density -> V_eff -> H (accumulate + mirror).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import veff as V  # noqa: E402  (host reference leg, timed)
from paper_1402_4247_b200 import _abi  # noqa: E402
from paper_1402_4247_b200.grid import GridPass  # noqa: E402
from paper_1402_4247_b200.system import Fe3O4  # noqa: E402


def ev_time(fn, st, flush, reps=10):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="cubic56_200Ry,super448_200Ry,super1512_200Ry")
    ap.add_argument("--xc", type=int, default=0, help="KBG_OPT_XC: 0 exchange only, 1 LSDA (PW92)")
    a = ap.parse_args()
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream()
    flush = torch.empty(512 << 18, dtype=torch.float32, device=dev)
    for cfg in a.configs.split(","):
        f = Fe3O4.config(cfg)
        gp = GridPass(f.system)
        gp.set_option(_abi.KBG_OPT_XC, a.xc)
        n = f.system.npts
        rng = np.random.default_rng(1402)
        rho_h = rng.uniform(0.0, 0.2, (1, n))
        vloc_h = f.veff()[0]
        rho = torch.from_numpy(rho_h).to(dev)
        vloc = torch.from_numpy(vloc_h).to(dev)
        out = torch.empty_like(rho)
        en = torch.empty(2, dtype=torch.float64, device=dev)
        ms = ev_time(lambda: gp.veff_dev(rho, out, vloc, en, st), st, flush)
        nbytes = 8 * n * (3 + 4)
        t0 = time.perf_counter()
        V.veff(rho_h, f.system.lattice, tuple(f.system.grid), vloc_h, xc=a.xc)
        host_ms = (time.perf_counter() - t0) * 1e3
        rec = {"config": cfg, "xc": ["exchange", "lsda_pw92"][a.xc], "grid": list(f.system.grid), "npts": n, "veff_ms": round(ms, 4),
               "bytes_compulsory_plus_fft": nbytes, "achieved_gbs": round(nbytes / (ms * 1e-3) / 1e9, 1),
               "hbm_frac": round(nbytes / (ms * 1e-3) / 1e9 / peak, 3), "numpy_host_ms": round(host_ms, 1)}
        if cfg == "cubic56_200Ry":
            ix = gp.build_index()
            d_dm = torch.from_numpy(f.dm(ix)).to(dev)
            d_rho = torch.empty((1, n), dtype=torch.float64, device=dev)
            d_h = torch.empty((1, ix["nnz"]), dtype=torch.float64, device=dev)

            def scf():
                gp.density_dev(d_dm, d_rho, st)
                gp.veff_dev(d_rho, out, vloc, en, st)
                gp.hamiltonian_dev(out, f.dV, d_h, st)

            rec["scf_grid_iteration_ms"] = round(ev_time(scf, st, flush), 4)
        print(json.dumps(rec), flush=True)
        del gp


if __name__ == "__main__":
    main()
