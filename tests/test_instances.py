"""Device problem generator (instances.gen_randsvd_device) and the on-disk
instance format — exercised on CPU tensors here (the same torch code runs on
the GPU box for C3/C4)."""

import numpy as np
import pytest
import torch

from paper_2311_04362_b200 import instances as inst


@pytest.fixture(scope="module")
def prob():
    return inst.gen_randsvd_device(3000, 40, 1e4, 1e-3, seed=5, device="cpu")


def test_construction(prob):
    a = prob.a.numpy()
    m, n = a.shape
    sv = np.linalg.svd(a, compute_uv=False)
    sigma = 1e4 ** (-np.arange(n) / (n - 1))
    np.testing.assert_allclose(sv, sigma, rtol=1e-12, atol=1e-15)
    x, r = prob.truth.x, prob.truth.r.numpy()
    assert abs(np.linalg.norm(x) - 1) < 1e-14
    assert abs(np.linalg.norm(r) - 1e-3) < 1e-15
    # r orthogonal to range(A): A'r at the u level
    assert np.linalg.norm(a.T @ r) < 1e-14 * np.linalg.norm(r) * 10
    np.testing.assert_allclose(prob.b.numpy(), a @ x + r, rtol=0, atol=1e-15)
    # x is the LS solution
    xl = np.linalg.lstsq(a, prob.b.numpy(), rcond=None)[0]
    assert np.linalg.norm(xl - x) < 1e4 * 1e-13


def test_deterministic_and_seeded(prob):
    again = inst.gen_randsvd_device(3000, 40, 1e4, 1e-3, seed=5, device="cpu")
    assert torch.equal(again.a, prob.a) and torch.equal(again.b, prob.b)
    other = inst.gen_randsvd_device(3000, 40, 1e4, 1e-3, seed=6, device="cpu")
    assert not torch.equal(other.a, prob.a)


def test_gaussian_blocks_independent_of_chunking():
    g1 = torch.empty(3 * inst.GEN_BLOCK + 5, 3, dtype=torch.float64)
    inst._gaussian_rows(g1, 0, 7, 0)
    g2 = torch.empty_like(g1)
    inst._gaussian_rows(g2[: inst.GEN_BLOCK], 0, 7, 0)
    inst._gaussian_rows(g2[inst.GEN_BLOCK:], inst.GEN_BLOCK, 7, 0)
    assert torch.equal(g1, g2)
    with pytest.raises(ValueError):
        inst._gaussian_rows(g2[1:], 1, 7, 0)


def test_cholesky_qr2_orthonormal():
    g = torch.randn(5000, 60, dtype=torch.float64, generator=torch.Generator().manual_seed(1))
    g0 = g.clone()
    r = inst.cholesky_qr2_inplace(g)
    eye = g.T @ g
    assert torch.linalg.matrix_norm(eye - torch.eye(60, dtype=torch.float64)) < 1e-14
    assert torch.all(torch.diagonal(r) > 0)
    assert torch.linalg.matrix_norm(g @ r - g0) / torch.linalg.matrix_norm(g0) < 1e-14


def test_validation():
    for args in [(10, 10, 1e2, 0.1), (10, 1, 1e2, 0.1), (10, 3, 0.5, 0.1), (10, 3, 10, -1)]:
        with pytest.raises(ValueError):
            inst.gen_randsvd_device(*args, seed=0, device="cpu")


def test_save_load_roundtrip(prob, tmp_path):
    d = inst.save_instance(str(tmp_path / "c"), prob, seed=5, generator="gen_randsvd_device")
    whole = inst.load_instance(d)
    np.testing.assert_array_equal(whole.a, prob.a.numpy())
    np.testing.assert_array_equal(whole.b, prob.b.numpy())
    np.testing.assert_array_equal(whole.truth.r, prob.truth.r.numpy())
    assert whole.truth.kappa == 1e4 and whole.truth.beta == 1e-3
    part = inst.load_instance(d, rows=(1000, 2000))
    np.testing.assert_array_equal(part.a, prob.a.numpy()[1000:2000])
    np.testing.assert_array_equal(part.truth.r, prob.truth.r.numpy()[1000:2000])
    with open(d + "/manifest.json", "w") as f:
        f.write('{"format": "other"}')
    with pytest.raises(ValueError):
        inst.load_instance(d)
