"""Measurement of the format converters (kb_formats.cu) against the HBM roofline.

python tools/bench_formats.py [--configs cubic56_200Ry,super448_200Ry] [--nk 4] [--reps 10]
One JSON line per (config, op): device-resident inputs, CUDA events around the C-ABI _dev call
(phase kernel + converter kernel), L2 flushed between reps; algorithmic bytes = compulsory traffic:
  bloch         nnz*8 (pairs) + nk*n^2*16 (M(k) written)
  fold          nk*16*(entries of the distinct atom-pair blocks (a, b) of the pair list: all offsets R of
                one (a, b) read the same rho_k block) + nnz*8 (DM written)
  to_realspace  nR*n^2*8 (dense blocks written, zero fill included) + nnz*16
peak = MEASURED_PEAKS.json hbm_gbs (copy bandwidth).
"""
import argparse
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
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="cubic56_200Ry,super448_200Ry")
    ap.add_argument("--nk", type=int, default=4)
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream()
    flush = torch.empty(512 << 18, dtype=torch.float32, device=dev)
    rng = np.random.default_rng(1402)
    for cfg in a.configs.split(","):
        f = Fe3O4.config(cfg)
        gp = GridPass(f.system)
        ix = gp.build_index()
        n, nnz, nR = gp.nbasis(), int(ix["nnz"]), len(gp.offsets())
        kpts = rng.uniform(-0.5, 0.5, (a.nk, 3))
        w = np.full(a.nk, 1.0 / a.nk)
        d_pairs = torch.from_numpy(f.dm(ix)[0]).to(dev)
        norb = f.system.norb_of_atom()
        ab = np.unique(np.stack([ix["pair_a"], ix["pair_b"]], 1), axis=0)
        ab_elems = int((norb[ab[:, 0]] * norb[ab[:, 1]]).sum())
        d_mk = torch.empty((a.nk, n, n, 2), dtype=torch.float64, device=dev)
        d_back = torch.empty_like(d_pairs)
        ops = {"bloch": (lambda: gp.bloch_dev(d_pairs, kpts, d_mk, st), nnz * 8 + a.nk * n * n * 16),
               "fold": (lambda: gp.fold_dev(d_mk, kpts, w, d_back, st), a.nk * ab_elems * 16 + nnz * 8)}
        if nR * n * n * 8 < 8 << 30:
            d_dense = torch.empty((nR, n, n), dtype=torch.float64, device=dev)
            ops["to_realspace"] = (lambda: gp.to_realspace_dev(d_pairs, d_dense, st), nR * n * n * 8 + nnz * 16)
        for name, (fn, nbytes) in ops.items():
            for _ in range(3):
                fn()
            ts = []
            for _ in range(a.reps):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                fn()
                e1.record(st)
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            ms = float(np.median(ts))
            gbs = nbytes / (ms * 1e-3) / 1e9
            print(json.dumps({"config": cfg, "op": name, "n": n, "nnz": nnz, "nR": nR, "nk": a.nk,
                              "launches": gp.last_launches, "median_ms": round(ms, 4),
                              "algorithmic_bytes": nbytes, "achieved_gbs": round(gbs, 1), "peak_gbs": peak,
                              "frac": round(gbs / peak, 3)}), flush=True)
        del gp


if __name__ == "__main__":
    main()
