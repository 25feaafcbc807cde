"""Measurement of the GPU Eigen_HH pieces (kb_eigen.cu) vs the reference's own kband on the
host cores (oracle/_ref/libkband_ref.so).

python tools/bench_eigen.py [--sizes 568,1040,2048]
Per n (random Hermitian, seed n): GPU tridiagonalize (device-resident, CUDA events, median of 5), GPU
back_transform of n eigenvectors, GPU normalize_columns, GPU eigen_hh end to end through the host API
(host LAPACK stemr tridiagonal step included, wall clock); reference kband tridiagonalize / back_transform
/ eigen_hh serial and threaded (wall clock, best of 2 -- the serial tridiagonalization is skipped above
n = 1100 to bound the run). Work: tridiagonalization streams ~16 n^3 bytes through L2 (hemv read + her2
read/write of the trailing block per stage) with 2 grid barriers per stage; back transform 8 n^2 m flops.
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

from oracle import kband_ref as R  # noqa: E402  (reference leg, timed)
from paper_1402_4247_b200 import _abi  # noqa: E402
from paper_1402_4247_b200 import eigen as E  # noqa: E402


def wall(fn, reps=2):
    best = 1e30
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="568,1040,2048")
    a = ap.parse_args()
    lib = _abi.kbgrid()
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream()
    nt = os.cpu_count() or 1
    for n in [int(x) for x in a.sizes.split(",")]:
        rng = np.random.default_rng(n)
        x = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
        A = 0.5 * (x + x.conj().T)
        rec = {"n": n}
        hA = torch.from_numpy(A.view(np.float64).reshape(n, 2 * n).copy())
        work = torch.empty((n, 2 * n), dtype=torch.float64, device=dev)
        d = torch.empty(n, dtype=torch.float64, device=dev)
        e = torch.empty(n, dtype=torch.float64, device=dev)
        u = torch.empty((n - 1, 2 * n), dtype=torch.float64, device=dev)
        h = torch.empty(n, dtype=torch.float64, device=dev)
        s = torch.empty(n, dtype=torch.float64, device=dev)
        ph = torch.empty(2 * n, dtype=torch.float64, device=dev)

        def tri():
            lib.kbg_hh_tridiagonalize_dev(n, work.data_ptr(), 0, d.data_ptr(), e.data_ptr(), u.data_ptr(),
                                          h.data_ptr(), s.data_ptr(), ph.data_ptr(), st.cuda_stream)

        ts = []
        for r in range(6):
            work.copy_(hA.to(dev))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            tri()
            e1.record(st)
            e1.synchronize()
            if r:
                ts.append(e0.elapsed_time(e1))
        t_tri = float(np.median(ts))
        rec["gpu_tridiagonalize_ms"] = round(t_tri, 3)
        rec["gpu_tridiagonalize_us_per_stage"] = round(1e3 * t_tri / (n - 1), 3)
        rec["gpu_tridiagonalize_l2_gbs"] = round(16.0 * n ** 3 / (t_tri * 1e-3) / 1e9, 1)
        # back transform of n eigenvectors from the reference tridiagonal solve
        dd, ee = d.cpu().numpy(), e.cpu().numpy()[: n - 1]
        _, z = R.solve_tridiag(dd, ee, True)
        Y = torch.from_numpy(np.ascontiguousarray(z)).to(dev)
        W = torch.empty((n, 2 * n), dtype=torch.float64, device=dev)

        def bt():
            lib.kbg_hh_back_transform_dev(n, n, u.data_ptr(), h.data_ptr(), ph.data_ptr(), Y.data_ptr(),
                                          W.data_ptr(), st.cuda_stream)

        bt()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            bt()
            e1.record(st)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        t_bt = float(np.median(ts))
        rec["gpu_back_transform_ms"] = round(t_bt, 3)
        rec["gpu_back_transform_tflops"] = round(8.0 * n ** 3 / (t_bt * 1e-3) / 1e12, 3)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        lib.kbg_hh_normalize_columns_dev(n, n, W.data_ptr(), st.cuda_stream)
        e1.record(st)
        e1.synchronize()
        rec["gpu_normalize_ms"] = round(e0.elapsed_time(e1), 3)
        rec["gpu_eigen_hh_e2e_host_lapack_ms"] = round(
            wall(lambda: E.eigen_hh(A, True, solve_tridiag=E.lapack_solve_tridiag)), 2)
        rec["gpu_eigen_hh_e2e_ms"] = round(wall(lambda: E.eigen_hh(A, True)), 2)  # kbg_hh_eigen, device-resident
        # the tridiagonal step: GPU (kbg_tridiag_solve, device-resident, events) vs host LAPACK stemr
        t = E.tridiagonalize(A)
        Dd = torch.from_numpy(t.d).to(dev)
        De = torch.from_numpy(t.e if n > 1 else np.zeros(1)).to(dev)
        Dw = torch.empty(n, dtype=torch.float64, device=dev)
        Dz = torch.empty((n, n), dtype=torch.float64, device=dev)
        ts = []
        for _ in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            assert lib.kbg_tridiag_solve_dev(n, Dd.data_ptr(), De.data_ptr(), 1, Dw.data_ptr(), Dz.data_ptr(),
                                             st.cuda_stream) == 0
            e1.record(st)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        rec["gpu_tridiag_solve_ms"] = round(float(np.median(ts[1:])), 3)
        rec["host_lapack_stemr_ms"] = round(wall(lambda: E.lapack_solve_tridiag(t.d, t.e, True)), 2)

        # reference kband on the host
        if n <= 1100:
            rec["ref_tridiagonalize_serial_ms"] = round(wall(lambda: R.tridiagonalize(A), 1), 1)
            rec["ref_eigen_hh_serial_ms"] = round(wall(lambda: R.eigen_hh(A, True, 1), 1), 1)
        rec["ref_eigen_hh_threads"] = nt
        rec["ref_eigen_hh_threaded_ms"] = round(wall(lambda: R.eigen_hh(A, True, nt), 1), 1)
        rd, re_, ru, rh, rs, rph = R.tridiagonalize(A)
        rec["ref_back_transform_threaded_ms"] = round(wall(lambda: R.back_transform(ru, rh, rs, rph, z, nt), 1), 1)
        rec["max_eig_residual_rel"] = None
        w, v = E.eigen_hh(A, True, solve_tridiag=E.lapack_solve_tridiag)
        rec["max_eig_residual_rel"] = float(np.abs(A @ v - v * w).max() / np.linalg.norm(A))
        w, v = E.eigen_hh(A, True)
        rec["max_eig_residual_rel_gpu_solver"] = float(np.abs(A @ v - v * w).max() / np.linalg.norm(A))
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
