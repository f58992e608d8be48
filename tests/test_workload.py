"""Synthetic workload generators: the torch/device path used for C3 agrees
with the host numpy path it stands in for."""
import numpy as np

from paper_2209_02815_b200 import workload as W


def test_gaussian_torch_matches_numpy_bits_of_splitmix():
    for cnt in (1, 2, 7, 1000, 4097):
        a = W.gaussian(W.seed_for(2, 1), cnt)
        b = W.gaussian_torch(W.seed_for(2, 1), cnt, "cpu", chunk=256).numpy()
        assert b.shape == a.shape
        assert np.max(np.abs(a - b)) <= 8 * np.finfo(float).eps * max(1.0, np.max(np.abs(a)))


def test_device_jacobian_matches_host_generator():
    J = W.synthetic_jacobian(16, 2000, 2)
    Jd = W.synthetic_jacobian_device(16, 2000, 2, "cpu", chunk_cols=300).numpy()
    assert np.max(np.abs(J - Jd)) <= 1e-13 * np.max(np.abs(J))
    s = np.linalg.svd(Jd, compute_uv=False)
    assert np.allclose(s, 10.0 ** (-4.0 * np.arange(16) / 16), rtol=1e-12)
