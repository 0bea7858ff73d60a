"""The reference's unit properties of the dense kernels on the path
(/root/reference/pkg/tests/test_linalg.py), held by the device drop-ins of
`paper_2311_04362_b200.linalg` with the reference's inputs and tolerances:

  householder_qr_econ  :23-60    identity, the [3; 4] column, reconstruction
                                 and orthogonality bars, diag(R) >= 0, bitwise
                                 reproducible, wide input rejected
  tri_solve_upper(_transpose) :63-108  identity, hand cases, residual bars,
                                 the normal-equations composition, zero diagonal
  rand_power_norm_est  :135-156  identity, null direction, tight in >= 99 of
                                 100 draws and never above sigma_max, deterministic
  cond_est             :159-173  identity, diagonal, the SVD ratio, zero diagonal

Where the reference asserts exact equality of a value the device forms by a
different (Lanczos / power) recurrence, the tolerance is written in the test.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

U = 2.0 ** -53


@pytest.fixture(scope="module")
def pkg():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2311_04362_b200 as p

    return p


def _upper(rng, n, shift):
    return np.triu(rng.standard_normal((n, n))) + shift * np.eye(n)


def test_qr_identity_and_hand_column(pkg):
    f = pkg.householder_qr_econ(np.eye(5))
    assert np.array_equal(f.q, np.eye(5)) and np.array_equal(f.r, np.eye(5))
    f = pkg.householder_qr_econ(np.array([[3.0], [4.0]]))
    np.testing.assert_allclose(f.r, [[5.0]], rtol=1e-15)
    np.testing.assert_allclose(f.q, [[0.6], [0.8]], rtol=1e-15)


@pytest.mark.parametrize("m,n,seed", [(20, 5, 0), (10, 3, 1), (50, 20, 2), (200, 40, 3)])
def test_qr_reconstruction_and_orthogonality(pkg, m, n, seed):
    a = np.random.default_rng(seed).standard_normal((m, n))
    f = pkg.householder_qr_econ(a)
    assert np.linalg.norm(f.q @ f.r - a) <= 100 * m * n * U * np.linalg.norm(a)
    assert np.linalg.norm(f.q.T @ f.q - np.eye(n)) <= 100 * n * U
    if (m, n) == (20, 5):  # test_linalg.py:34-38
        assert np.linalg.norm(f.q @ f.r - a) / np.linalg.norm(a) <= 1e-14
        assert np.linalg.norm(f.q.T @ f.q - np.eye(5)) <= 1e-14


def test_qr_sign_shape_and_reproducibility(pkg):
    a = np.random.default_rng(7).standard_normal((12, 6))
    f = pkg.householder_qr_econ(-a)
    assert np.all(np.diag(f.r) >= 0) and np.array_equal(f.r, np.triu(f.r))
    a = np.random.default_rng(9).standard_normal((15, 4))
    f1, f2 = pkg.householder_qr_econ(a), pkg.householder_qr_econ(a)
    assert np.array_equal(f1.q, f2.q) and np.array_equal(f1.r, f2.r)
    with pytest.raises(ValueError):
        pkg.householder_qr_econ(np.ones((3, 5)))


def test_qr_orthogonal_factors_preserve_singular_values(pkg):
    """test_linalg.py:124-132 through the device Q."""
    rng = np.random.default_rng(11)
    a = rng.standard_normal((12, 5))
    ql = pkg.householder_qr_econ(rng.standard_normal((12, 12))).q
    qr_ = pkg.householder_qr_econ(rng.standard_normal((5, 5))).q
    sv = np.linalg.svd(a, compute_uv=False)
    for t in (ql @ a, a @ qr_, ql @ a @ qr_):
        np.testing.assert_allclose(np.linalg.svd(t, compute_uv=False), sv, rtol=1e-10)
    q = pkg.householder_qr_econ(np.random.default_rng(2).standard_normal((9, 4))).q
    np.testing.assert_allclose(np.linalg.svd(q, compute_uv=False), np.ones(4), atol=1e-13)


def test_trisolve_hand_cases(pkg):
    c = np.array([3.0, -1.0, 2.0])
    assert np.array_equal(pkg.tri_solve_upper(np.eye(3), c), c)
    assert np.array_equal(pkg.tri_solve_upper_transpose(np.eye(3), c), c)
    np.testing.assert_allclose(pkg.tri_solve_upper(np.diag([2.0, 4.0]), np.array([2.0, 4.0])), [1.0, 1.0])
    r = np.array([[1.0, 1.0], [0.0, 1.0]])
    np.testing.assert_allclose(pkg.tri_solve_upper_transpose(r, np.array([1.0, 2.0])), [1.0, 1.0], rtol=1e-15)
    r = np.array([[1.0, 2.0], [0.0, 0.0]])
    for solve in (pkg.tri_solve_upper, pkg.tri_solve_upper_transpose):
        with pytest.raises(pkg.SingularMatrixError):
            solve(r, np.ones(2))


def test_trisolve_residuals(pkg):
    rng = np.random.default_rng(4)
    r = _upper(rng, 10, 5.0)
    c = rng.standard_normal(10)
    y = pkg.tri_solve_upper(r, c)
    assert np.linalg.norm(r @ y - c) / np.linalg.norm(c) <= 1e-13
    rng = np.random.default_rng(5)
    r = _upper(rng, 8, 4.0)
    c = rng.standard_normal(8)
    y = pkg.tri_solve_upper(r, pkg.tri_solve_upper_transpose(r, c))
    y_dense = np.linalg.solve(r.T @ r, c)
    assert np.linalg.norm(y - y_dense) / np.linalg.norm(y_dense) <= 1e-12
    rng = np.random.default_rng(6)
    for n in (5, 20, 50):
        r = _upper(rng, n, 2.0 + n)
        kappa = pkg.cond_est(r)
        assert kappa <= 1e8
        c = rng.standard_normal(n)
        y = pkg.tri_solve_upper(r, c)
        assert np.linalg.norm(r @ y - c) <= 100 * n * U * kappa * np.linalg.norm(c)


def test_normest_properties(pkg):
    # the reference's power iteration returns exactly 1.0 on the identity; the
    # device's normalisation may differ in the last place
    assert abs(pkg.rand_power_norm_est(np.eye(6), rng_seed=0) - 1.0) <= 4 * U
    est = pkg.rand_power_norm_est(np.diag([5.0, 0.0]), steps=1, rng_seed=1)
    assert 0.0 <= est <= 5.0
    rng = np.random.default_rng(12)
    hits = 0
    for seed in range(100):
        r = _upper(rng, 50, 1.0)
        sigma_max = np.linalg.svd(r, compute_uv=False)[0]
        est = pkg.rand_power_norm_est(r, steps=6, rng_seed=seed)
        assert est <= sigma_max * (1 + 1e-12)
        hits += est >= 0.5 * sigma_max
    assert hits >= 99
    r = _upper(np.random.default_rng(13), 20, 1.0)
    assert pkg.rand_power_norm_est(r, rng_seed=5) == pkg.rand_power_norm_est(r, rng_seed=5)


def test_condest_properties(pkg):
    # exact SVD in the reference (== 1.0, rel 1e-12, rel 1e-10); the device's
    # Lanczos extremes agree to the tolerances the reference itself uses for
    # the non-trivial cases
    assert abs(pkg.cond_est(np.eye(4)) - 1.0) <= 1e-14
    assert pkg.cond_est(np.diag([1.0, 1e-8])) == pytest.approx(1e8, rel=1e-12)
    r = _upper(np.random.default_rng(14), 9, 3.0)
    sv = np.linalg.svd(r, compute_uv=False)
    assert pkg.cond_est(r) == pytest.approx(sv[0] / sv[-1], rel=1e-10)
    with pytest.raises(pkg.SingularMatrixError):
        pkg.cond_est(np.diag([1.0, 0.0]))
