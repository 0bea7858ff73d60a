"""CPU checks for SURVEY §8 rows f-3 (CLI) and f-4 (sparse A) against the
reference's own outputs (tests/golden/sparse_cli.npz, made by
tests/golden/make_golden_sparse_cli.py from the unmodified reference)."""

import hashlib
import json
import math
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "sparse_cli.npz")


@pytest.fixture(scope="module")
def g():
    return np.load(GOLD)


def _sha(*arrs):
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("m,n,seed", [(50, 5, 0), (2000, 40, 0), (300, 3, 7)])
def test_gen_sparse_matches_reference(g, m, n, seed):
    from paper_2311_04362_b200.problems import gen_sparse

    p = gen_sparse(m, n, seed)
    k = f"gs_{m}_{n}_{seed}"
    assert np.array_equal(p.a.indptr, g[k + "_indptr"])
    assert np.array_equal(p.a.indices, g[k + "_indices"])
    assert np.array_equal(p.a.data, g[k + "_data"])
    assert np.array_equal(p.b, g[k + "_b"])
    assert p.truth is None


def test_gen_sparse_digests(g):
    from paper_2311_04362_b200.problems import gen_sparse

    for key, want in json.loads(str(g["gs_digests"])).items():
        m, n, seed = map(int, key.split("_"))
        p = gen_sparse(m, n, seed)
        assert _sha(p.a.indptr.astype(np.int64), p.a.indices.astype(np.int32), p.a.data, p.b) == want, key


def test_gen_sparse_rejects_bad_shape():
    from paper_2311_04362_b200.problems import gen_sparse

    with pytest.raises(ValueError):
        gen_sparse(2, 3, 0)
    with pytest.raises(ValueError):
        gen_sparse(10, 2, 0)


@pytest.mark.parametrize("m,n,seed,d,zeta", [(5000, 50, 2, 1000, 8), (2000, 40, 0, 1200, 8), (300, 3, 7, 20, 4),
                                             (40000, 200, 5, 6000, 8)])
def test_oracle_sparse_sketch_bitwise(g, m, n, seed, d, zeta):
    from oracle import itsketch_oracle as orc
    from paper_2311_04362_b200.problems import gen_sparse

    p = gen_sparse(m, n, seed)
    pat = orc.sparse_sign_pattern(d, m, zeta, seed)
    sa = orc.sketch_apply_sparse(pat, p.a)
    k = f"sk_{m}_{n}_{seed}_{d}_{zeta}"
    if k in g:
        assert np.array_equal(sa, g[k])
    assert _sha(sa) == str(g[k + "_sha"])
    assert _sha(orc.sketch_apply(pat, p.b)) == str(g[k + "_sb_sha"])


def test_oracle_sparse_sketch_equals_densified():
    """Skipping A's zeros does not change any sum (x + 0 = x): the sparse and
    dense restatements agree bitwise, as the reference's test_embed checks."""
    import scipy.sparse as sp

    from oracle import itsketch_oracle as orc

    rng = np.random.default_rng(3)
    a = sp.random(400, 30, density=0.1, random_state=4, format="csr")
    pat = orc.sparse_sign_pattern(60, 400, 5, 1)
    assert np.array_equal(orc.sketch_apply_sparse(pat, a), orc.sketch_apply(pat, a.toarray()))
    del rng


@pytest.mark.parametrize("name", ["sp_basic", "sp_mom", "sp_damped", "sp_n3"])
def test_oracle_sparse_solve_matches_reference(g, name):
    from oracle import itsketch_oracle as orc
    from paper_2311_04362_b200.problems import gen_sparse

    m, n, seed = (int(v) for v in g[f"{name}_problem"])
    p = gen_sparse(m, n, seed)
    cfgd = json.loads(str(g[f"{name}_config"]))
    x, tr = orc.iterative_sketching(p.a, p.b, orc.Config(**cfgd))
    ref = g[f"{name}_iterates"]
    assert tr.stop_reason == str(g[f"{name}_stop"])
    assert len(tr.iterates) == len(ref)
    # the same scipy / LAPACK calls in the same order
    np.testing.assert_allclose(np.array(tr.iterates), ref, rtol=0, atol=1e-12 * np.abs(ref).max())
    np.testing.assert_allclose([tr.normest, tr.condest], g[f"{name}_est"], rtol=1e-12)


def test_choose_dim_matches_reference(g):
    from paper_2311_04362_b200.cli import choose_dim

    for m, n, acc, v, d in json.loads(str(g["dims"])):
        assert choose_dim(m, n, acc, v) == d, (m, n, acc, v)
    with pytest.raises(ValueError):
        choose_dim(10, 20, 1e-6)
    with pytest.raises(ValueError):
        choose_dim(100, 10, 0.0)
    with pytest.raises(ValueError):
        choose_dim(100, 10, 1e-6, "nope")


def test_bound_curve_matches_reference(g):
    from paper_2311_04362_b200.cli import RateHypothesisError, bound_curve

    for v, eps, kappa, na, nr, iters, first, fe, re in json.loads(str(g["bounds"])):
        bf, br = bound_curve(v, eps, kappa, na, nr, iters, first)
        np.testing.assert_allclose(bf, fe, rtol=1e-14)
        np.testing.assert_allclose(br, re, rtol=1e-14)
    with pytest.raises(RateHypothesisError):
        bound_curve("basic", 0.5, 1.0, 1.0, 1.0, 3)
    with pytest.raises(RateHypothesisError):
        bound_curve("momentum", 0.2, 1.0, 1.0, 1.0, 3, first_iter=0)
    with pytest.raises(ValueError):
        bound_curve("nope", 0.2, 1.0, 1.0, 1.0, 3)


def test_cli_dims_file_is_the_reference_file(g, tmp_path):
    from paper_2311_04362_b200.cli import main

    out = tmp_path / "dims.csv"
    assert main(["dims", "--m", "200000", "--n", "200", "--out", str(out)]) == 0
    assert out.read_text() == str(g["cli_dims"])


def test_cli_usage_errors_exit_64(tmp_path, capsys):
    from paper_2311_04362_b200.cli import EXIT_USAGE, main

    for argv in (["bad", "--m", "3"], ["kernel"], ["solve", "--m", "10"], ["dims", "--m", "x", "--n", "2",
                                                                         "--out", "o"], []):
        with pytest.raises(SystemExit) as e:
            main(argv)
        assert e.value.code == EXIT_USAGE, argv
    capsys.readouterr()


def test_cli_table_format(tmp_path):
    from paper_2311_04362_b200.cli import save_numeric_csv, write_table

    p = tmp_path / "t.csv"
    write_table(str(p), "a,b", [["z", 1.5], ["a", float("nan")], [3, 1e-300]])
    assert p.read_text().splitlines() == ["# schema=v1", "a,b", "3,1e-300", "a,nan", "z,1.5"]
    q = tmp_path / "x.csv"
    save_numeric_csv(str(q), ["x"], np.array([[0.1], [math.pi]]))
    assert q.read_bytes() == b"x\r\n0.1\r\n3.141592653589793\r\n"


def test_cli_without_gpu_fails_loudly(tmp_path):
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    from paper_2311_04362_b200.cli import main

    with pytest.raises(RuntimeError):
        main(["solve", "--m", "100", "--n", "5", "--cond", "10", "--resnorm", "1e-3", "--out", str(tmp_path / "x")])
