"""Per-kernel timing experiments (CUDA events, L2 flushed between reps).

python tools/kernel_times.py [--config cubic56_200Ry] [--reps 20]
Prints one JSON line per variant: density / hamiltonian accumulate with
atomic scatter vs plain-store scatter (timing experiment only), 4 vs 8 warps.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1402_4247_b200 import _abi  # noqa: E402
from paper_1402_4247_b200.grid import GridPass  # noqa: E402
from paper_1402_4247_b200.system import Fe3O4  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cubic56_200Ry")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--nspin", type=int, default=1)
    ap.add_argument("--schedules", default="3,0,1,2", help="KBG_OPT_SCHEDULE values (persistent kernels)")
    ap.add_argument("--fallback", type=int, default=1, help="also time the one-CTA-per-block kernels")
    ap.add_argument("--orders", default="2", help="KBG_OPT_BLOCK_ORDER values (persistent kernels)")
    ap.add_argument("--scatter", type=int, default=0, help="KBG_OPT_SCATTER_STORE timing experiment bits")
    ap.add_argument("--det", type=int, default=0, help="KBG_OPT_DETERMINISTIC (1: two-limb exact scatter)")
    ap.add_argument("--kernels", default="density,h_accumulate")
    ap.add_argument("--sparse", type=int, default=0, help="KBG_OPT_SPARSE_DFMA threshold (A5 switch)")
    ap.add_argument("--rebuild", type=int, default=0, help="extra build_index calls (bench.py builds twice)")
    a = ap.parse_args()
    f = Fe3O4.config(a.config)
    dev = torch.device("cuda", 0)
    flush = torch.empty(512 << 18, dtype=torch.float32, device=dev)
    st = torch.cuda.current_stream()

    def timeit(fn):
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
        return float(np.median(ts)), float(np.min(ts))

    ref = {}
    variants = [(int(x), 1, int(o)) for x in a.schedules.split(",") for o in a.orders.split(",")]
    variants += [(3, 0, 0)] if a.fallback else []
    for sched, persist, order in variants:
        gp = GridPass(f.system)
        gp.set_option(_abi.KBG_OPT_SCHEDULE, sched)
        gp.set_option(_abi.KBG_OPT_BLOCK_ORDER, order)
        ix = gp.build_index()
        for _ in range(a.rebuild):
            ix = gp.build_index()
        gp.set_option(_abi.KBG_OPT_PERSIST, persist)
        plan = gp.plan_info()
        gp.set_option(_abi.KBG_OPT_SCATTER_STORE, a.scatter)
        gp.set_option(_abi.KBG_OPT_DETERMINISTIC, a.det)
        gp.set_option(_abi.KBG_OPT_SPARSE_DFMA, a.sparse)
        d_dm = torch.from_numpy(f.dm(ix, nspin=a.nspin)).to(dev)
        d_v = torch.from_numpy(f.veff(nspin=a.nspin)).to(dev)
        rho = torch.empty((a.nspin, f.system.npts), dtype=torch.float64, device=dev)
        h = torch.empty((a.nspin, ix["nnz"]), dtype=torch.float64, device=dev)
        f_rho = a.nspin * (2 * ix["sum_m2"] + 2 * ix["sum_m"])
        f_h = a.nspin * 2 * ix["sum_m2"]
        for name, fn, fl, out in (
            ("density", lambda: gp.density_dev(d_dm, rho, st), f_rho, rho),
            ("h_accumulate", lambda: gp.hamiltonian_accumulate_dev(d_v, f.dV, h, st), f_h, h),
        ):
            if name not in a.kernels.split(","):
                continue
            med, mn = timeit(fn)
            out.zero_()
            fn()
            torch.cuda.synchronize()
            r1 = out.clone()
            out.zero_()
            fn()
            torch.cuda.synchronize()
            rec = {"config": a.config, "lib": os.environ.get("KBG_LIBKBGRID", "default"), "scatter_exp": a.scatter, "det": a.det, "sparse": a.sparse, "kernel": name, "schedule": sched, "persist": persist,
                   "block_order": order, "plan": plan,
                   "median_ms": round(med, 4), "min_ms": round(mn, 4),
                   "alg_tflops": round(fl / (med * 1e-3) / 1e12, 3),
                   "bitwise_repeat": bool(torch.equal(r1, out))}
            if name in ref:
                rec["rel_diff_vs_first"] = float((out - ref[name]).norm() / ref[name].norm())
            else:
                ref[name] = r1
            print(json.dumps(rec), flush=True)
        if "pass" in a.kernels.split(","):
            # density then H back to back on one stream, as in bench.py's step (and H then density):
            # per-kernel medians inside the pass
            for order in (("density", "h_accumulate"), ("h_accumulate", "density")):
                fns = {"density": lambda: gp.density_dev(d_dm, rho, st),
                       "h_accumulate": lambda: gp.hamiltonian_accumulate_dev(d_v, f.dV, h, st)}
                ts = {k: [] for k in order}
                for rep in range(a.reps + 3):
                    flush.zero_()
                    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
                    ev[0].record(st)
                    fns[order[0]]()
                    ev[1].record(st)
                    fns[order[1]]()
                    ev[2].record(st)
                    ev[2].synchronize()
                    if rep >= 3:
                        ts[order[0]].append(ev[0].elapsed_time(ev[1]))
                        ts[order[1]].append(ev[1].elapsed_time(ev[2]))
                print(json.dumps({"config": a.config, "lib": os.environ.get("KBG_LIBKBGRID", "default"),
                                  "pass_order": list(order), "det": a.det,
                                  **{k + "_median_ms": round(float(np.median(v)), 4) for k, v in ts.items()},
                                  **{k + "_mean_ms": round(float(np.mean(v)), 4) for k, v in ts.items()}}), flush=True)
        del gp


if __name__ == "__main__":
    main()
