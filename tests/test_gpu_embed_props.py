"""The reference's unit properties of the sparse sign embedding
(/root/reference/pkg/tests/test_embed.py:23-107), held by the device
`sparse_sign_new` / `SparseSignEmbedding` with the reference's inputs and
tolerances: structure (zeta distinct rows per column, +-1 signs, unit column
norms, zeta = d takes every row, zeta > d rejected, determinism per seed,
Monte-Carlo isotropy of S'S), and the apply_* edge cases (zero input, a basis
column returns S's column exactly, the materialised product, apply_vec,
apply_sparse, a dimension mismatch, right-multiplication associativity).
The bitwise agreement with the reference's own patterns and products is in
tests/test_gpu_parity.py; these are the reference's small hand cases.
"""

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2311_04362_b200 as p

    return p


def _dense(s):
    return np.asarray(s.matrix.todense())


def test_structure(pkg):
    s = pkg.sparse_sign_new(d=4, m=3, zeta=4, rng_seed=0)
    assert np.all(np.abs(_dense(s)) == 0.5)
    for j in range(3):
        assert sorted(s.rows[j]) == [0, 1, 2, 3]
    s = pkg.sparse_sign_new(d=30, m=50, zeta=5, rng_seed=1)
    np.testing.assert_allclose(np.linalg.norm(_dense(s), axis=0), 1.0, atol=2 * 2.0 ** -53)
    s = pkg.sparse_sign_new(d=25, m=40, zeta=6, rng_seed=2)
    assert s.rows.shape == s.signs.shape == (40, 6)
    assert all(len(set(s.rows[j])) == 6 for j in range(40))
    assert np.all(np.abs(s.signs) == 1.0)
    assert s.scale == pytest.approx(1 / math.sqrt(6))
    with pytest.raises(ValueError):
        pkg.sparse_sign_new(d=3, m=5, zeta=4, rng_seed=0)
    s1, s2 = pkg.sparse_sign_new(20, 30, 4, rng_seed=7), pkg.sparse_sign_new(20, 30, 4, rng_seed=7)
    assert np.array_equal(s1.rows, s2.rows) and np.array_equal(s1.signs, s2.signs)


def test_monte_carlo_isotropy(pkg):
    """test_embed.py:53-61: the entrywise mean of S'S over 500 seeds is the
    identity to 0.1."""
    d, m, zeta = 40, 200, 8
    acc = np.zeros((m, m))
    for seed in range(500):
        dense = _dense(pkg.sparse_sign_new(d, m, zeta, seed))
        acc += dense.T @ dense
    acc /= 500
    assert np.max(np.abs(acc - np.eye(m))) <= 0.1


def test_apply_edge_cases(pkg):
    s = pkg.sparse_sign_new(10, 20, 3, 0)
    assert np.all(s.apply_dense(np.zeros((20, 4))) == 0)
    with pytest.raises(ValueError):
        s.apply_dense(np.ones((21, 2)))
    s = pkg.sparse_sign_new(30, 50, 3, 1)
    e3 = np.zeros((50, 1))
    e3[3, 0] = 1.0
    assert np.array_equal(s.apply_dense(e3)[:, 0], _dense(s)[:, 3])
    s = pkg.sparse_sign_new(30, 50, 3, 2)
    a = np.random.default_rng(3).standard_normal((50, 5))
    np.testing.assert_allclose(s.apply_dense(a), _dense(s) @ a, atol=1e-15)
    s = pkg.sparse_sign_new(15, 25, 4, 4)
    assert np.all(s.apply_vec(np.zeros(25)) == 0)
    e7 = np.zeros(25)
    e7[7] = 1.0
    assert np.array_equal(s.apply_vec(e7), _dense(s)[:, 7])


def test_apply_sparse_and_associativity(pkg):
    import scipy.sparse as sp

    s = pkg.sparse_sign_new(20, 40, 3, 5)
    a = sp.random(40, 6, density=0.2, random_state=np.random.default_rng(6), format="csr")
    np.testing.assert_allclose(s.apply_sparse(a), s.apply_dense(np.asarray(a.todense())), atol=1e-15)
    s = pkg.sparse_sign_new(25, 60, 4, 8)
    rng = np.random.default_rng(9)
    a = rng.standard_normal((60, 5))
    c = rng.standard_normal((5, 3))
    lhs, rhs = s.apply_dense(a @ c), s.apply_dense(a) @ c
    assert np.linalg.norm(lhs - rhs) <= 1e-14 * max(1.0, np.linalg.norm(rhs))
