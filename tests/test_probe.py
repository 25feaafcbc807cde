"""HBM probe = the paper's Table 2 normalization (SPEC.md:463-471 examples):
n = 1 gives a correct unit vector, every output row has unit norm within 1e-14, zero rows stay zero;
the GPU kernel matches the host backend (oracle) to rounding."""
import numpy as np
import pytest

from oracle.oracle import normalize_rows as host_normalize


@pytest.mark.parametrize("n", [1, 2, 7, 64])
def test_host_backend_unit_norms(n):
    x = np.random.default_rng(n).standard_normal((n, n))
    for threads in (1, 3):
        y = host_normalize(x, threads)
        assert np.abs(np.linalg.norm(y, axis=1) - 1).max() <= 1e-14
        assert np.allclose(y * np.linalg.norm(x, axis=1)[:, None], x, rtol=1e-14, atol=0)


def test_host_backend_zero_row_and_n1():
    y = host_normalize(np.array([[0.0, 0.0], [3.0, 4.0]]))
    assert np.array_equal(y, [[0.0, 0.0], [0.6, 0.8]])
    assert np.array_equal(host_normalize(np.array([[-2.5]])), [[-1.0]])


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(1, 1), (3, 5), (64, 64), (257, 1001), (1000, 1000)])
def test_gpu_normalize_matches_host(built, shape):
    from paper_1402_4247_b200.grid import normalize_rows

    x = np.random.default_rng(7).standard_normal(shape)
    x[0] = 0.0 if shape[0] > 1 else x[0]
    y = normalize_rows(x)
    ref = host_normalize(x)
    assert np.abs(y - ref).max() <= 1e-15
    nz = np.linalg.norm(x, axis=1) > 0
    assert np.abs(np.linalg.norm(y[nz], axis=1) - 1).max() <= 1e-14
    assert np.array_equal(y[~nz], x[~nz])


@pytest.mark.gpu
def test_gpu_normalize_device_in_place(built):
    import torch

    from paper_1402_4247_b200.grid import normalize_rows_dev

    x = np.random.default_rng(3).standard_normal((300, 2048))
    d = torch.from_numpy(x).cuda()
    normalize_rows_dev(d)
    torch.cuda.synchronize()
    assert np.abs(d.cpu().numpy() - host_normalize(x)).max() <= 1e-15
