"""Tuning sweep: kbg_hh_tridiagonalize_dev time vs cooperative grid size (KBG_TRI_GRID).
python tools/tridiag_grid_sweep.py [sizes] [grids]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1402_4247_b200 import _abi  # noqa: E402


def main(sizes="568,1040,2048", grids="16,24,32,48,64,96,128,148,296"):
    lib = _abi.kbgrid()
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream()
    for n in (int(x) for x in sizes.split(",")):
        rng = np.random.default_rng(n)
        x = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
        a = 0.5 * (x + x.conj().T)
        hA = torch.from_numpy(np.ascontiguousarray(a).view(np.float64).reshape(n, 2 * n).copy())
        work = torch.empty_like(hA, device=dev)
        d = torch.empty(n, dtype=torch.float64, device=dev)
        e = torch.empty(n, dtype=torch.float64, device=dev)
        u = torch.empty((n - 1, 2 * n), dtype=torch.float64, device=dev)
        h = torch.empty(n, dtype=torch.float64, device=dev)
        s = torch.empty(n, dtype=torch.float64, device=dev)
        ph = torch.empty(2 * n, dtype=torch.float64, device=dev)
        rec = {"n": n}
        for g in grids.split(","):
            os.environ["KBG_TRI_GRID"] = g
            ts = []
            for r in range(4):
                work.copy_(hA.to(dev))
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                assert lib.kbg_hh_tridiagonalize_dev(n, work.data_ptr(), 0, d.data_ptr(), e.data_ptr(), u.data_ptr(),
                                                     h.data_ptr(), s.data_ptr(), ph.data_ptr(), st.cuda_stream) == 0
                e1.record(st)
                e1.synchronize()
                if r:
                    ts.append(e0.elapsed_time(e1))
            rec[g] = round(float(np.median(ts)), 3)
        os.environ.pop("KBG_TRI_GRID", None)
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main(*sys.argv[1:])
