"""One kbg_tridiag_solve_dev per size on random tridiagonal problems (for an ncu launch list of the
eigenvalue / eigenvector / re-orthogonalization kernels): python tools/tridiag_times.py [sizes]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1402_4247_b200 import _abi  # noqa: E402


def main(sizes="1040,2048"):
    lib = _abi.kbgrid()
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream()
    for n in (int(x) for x in sizes.split(",")):
        rng = np.random.default_rng(n)
        d = torch.from_numpy(rng.uniform(-2, 2, n)).to(dev)
        e = torch.from_numpy(rng.uniform(-2, 2, n - 1)).to(dev)
        w = torch.empty(n, dtype=torch.float64, device=dev)
        z = torch.empty((n, n), dtype=torch.float64, device=dev)
        assert lib.kbg_tridiag_solve_dev(n, d.data_ptr(), e.data_ptr(), 1, w.data_ptr(), z.data_ptr(),
                                         st.cuda_stream) == 0
        torch.cuda.synchronize()
        print(n, float((z.T @ z - torch.eye(n, device=dev, dtype=torch.float64)).abs().max()), flush=True)


if __name__ == "__main__":
    main(*sys.argv[1:])
