"""HBM calibration probe = the paper's Table 2 experiment.

"normalized -- divided every element of a vector by its norm -- n vectors which consist of n elements",
timed per backend:
  host_1t / host_nt   oracle/ C++ host backend, 1 thread and all host threads (wall clock, best of 3)
  gpu_kernel          kbg_normalize_rows_dev on device-resident data (CUDA events, median of 10, L2 flushed)
  gpu_e2e             pinned host buffer -> H2D + kbg_normalize_rows_dev + D2H on one stream (wall clock)
  gpu_hostapi         kbg_normalize_rows on a pageable numpy array (allocation + copies inside; wall clock)
The kernel's compulsory traffic is 2 n^2 8 bytes (read once from HBM, second read from L2, write once);
achieved / MEASURED_PEAKS.json hbm_gbs calibrates the HBM roofline. Reports the crossover n where the
GPU beats the best host backend end to end (the paper saw CUDA win "when n exceeds 1000").
python tools/microbench_normalize.py [--sizes 100,300,1000,3000,10000,20000]
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

from oracle.oracle import normalize_rows as host_normalize  # noqa: E402  (host backend, timed)
from paper_1402_4247_b200.grid import normalize_rows, normalize_rows_dev  # noqa: E402


def best_wall(fn, reps=3):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return min(ts) * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="100,300,1000,3000,10000,20000")
    a = ap.parse_args()
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    nt = os.cpu_count() or 1
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream()
    flush = torch.empty(512 << 18, dtype=torch.float32, device=dev)
    rng = np.random.default_rng(1402)
    rows = []
    for n in [int(s) for s in a.sizes.split(",")]:
        x = rng.standard_normal((n, n))
        ref = host_normalize(x, 1)
        rec = {"n": n, "host_threads": nt}
        rec["host_1t_ms"] = round(best_wall(lambda: host_normalize(x, 1)), 4)
        rec["host_nt_ms"] = round(best_wall(lambda: host_normalize(x, nt)), 4)
        got = normalize_rows(x)
        rec["gpu_hostapi_ms"] = round(best_wall(lambda: normalize_rows(x)), 4)
        d = torch.from_numpy(x).to(dev)
        h_in = torch.from_numpy(x).pin_memory()
        h_out = torch.empty_like(h_in).pin_memory()

        def e2e():
            d.copy_(h_in, non_blocking=True)
            normalize_rows_dev(d, st)
            h_out.copy_(d, non_blocking=True)
            torch.cuda.synchronize()

        e2e()
        rec["gpu_e2e_ms"] = round(best_wall(e2e), 4)
        assert np.array_equal(h_out.numpy(), got)
        ts = []
        for r in range(13):
            d.copy_(torch.from_numpy(x).to(dev))
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            normalize_rows_dev(d, st)
            e1.record(st)
            e1.synchronize()
            if r >= 3:
                ts.append(e0.elapsed_time(e1))
        ms = float(np.median(ts))
        rec["gpu_kernel_ms"] = round(ms, 5)
        gbs = 2 * n * n * 8 / (ms * 1e-3) / 1e9
        rec["gpu_kernel_gbs"] = round(gbs, 1)
        rec["hbm_frac"] = round(gbs / peak, 3)
        rec["max_abs_diff_vs_host"] = float(np.abs(got - ref).max())
        rec["max_norm_err"] = float(np.abs(np.linalg.norm(got, axis=1) - 1).max())
        rows.append(rec)
        print(json.dumps(rec), flush=True)
    best_host = {r["n"]: min(r["host_1t_ms"], r["host_nt_ms"]) for r in rows}
    cross = next((r["n"] for r in rows if r["gpu_e2e_ms"] < best_host[r["n"]]), None)
    cross_k = next((r["n"] for r in rows if r["gpu_kernel_ms"] < best_host[r["n"]]), None)
    print(json.dumps({"summary": "table2", "peak_gbs": peak, "crossover_n_e2e": cross,
                      "crossover_n_kernel": cross_k,
                      "largest_n_hbm_frac": rows[-1]["hbm_frac"] if rows else None}), flush=True)


if __name__ == "__main__":
    main()
