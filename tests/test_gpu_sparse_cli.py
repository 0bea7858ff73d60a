"""GPU parity of SURVEY §8 rows f-4 (sparse CSR A) and f-3 (the CLI with a
device flag) against the reference's outputs (tests/golden/sparse_cli.npz)
and the CPU oracle."""

import hashlib
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "sparse_cli.npz")


@pytest.fixture(scope="module")
def pkg():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2311_04362_b200 as p

    return p


@pytest.fixture(scope="module")
def g():
    return np.load(GOLD)


@pytest.fixture(scope="module")
def orc():
    from oracle import itsketch_oracle as o

    return o


def _sha(*arrs):
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def _odd_csr(m, n, seed):
    """A CSR with empty rows, a long row (> 32 entries), unsorted columns and
    a repeated column inside a row (non-canonical, as scipy allows)."""
    import scipy.sparse as sp

    rng = np.random.default_rng(seed)
    ptr, cols, vals = [0], [], []
    for j in range(m):
        k = 0 if j % 7 == 3 else (min(n, 40) if j % 97 == 5 else int(rng.integers(1, 6)))
        c = list(rng.choice(n, size=k, replace=False))
        if j % 13 == 1 and k >= 2:
            c.append(c[0])  # duplicate column
        rng.shuffle(c)
        cols += c
        vals += list(rng.standard_normal(len(c)))
        ptr.append(len(cols))
    return sp.csr_matrix((np.array(vals), np.array(cols, dtype=np.int32), np.array(ptr)), shape=(m, n))


# --------------------------------------------------------------------------
# sketch: bitwise apply_sparse
# --------------------------------------------------------------------------
@pytest.mark.parametrize("m,n,seed,d,zeta", [(5000, 50, 2, 1000, 8), (2000, 40, 0, 1200, 8), (300, 3, 7, 20, 4),
                                             (40000, 200, 5, 6000, 8)])
def test_csr_sketch_bitwise_reference(pkg, g, m, n, seed, d, zeta):
    p = pkg.gen_sparse(m, n, seed)
    s = pkg.sparse_sign_new(d, m, zeta, seed)
    sa = s.apply_sparse(p.a)
    k = f"sk_{m}_{n}_{seed}_{d}_{zeta}"
    if k in g:
        assert np.array_equal(sa, g[k])
    assert _sha(sa) == str(g[k + "_sha"])
    # with b as column n: the fused form the solver uses
    sab = s.apply_sparse(p.a, p.b)
    assert np.array_equal(sab[:, :n], sa)
    assert _sha(np.ascontiguousarray(sab[:, n])) == str(g[k + "_sb_sha"])


@pytest.mark.parametrize("m,n,d,zeta", [(3000, 60, 500, 8), (1000, 2500, 300, 4), (500, 9000, 100, 3)])
def test_csr_sketch_odd_structure(pkg, orc, m, n, d, zeta):
    """Empty rows, long rows, duplicate and unsorted columns; n large enough
    that the accumulator row leaves shared memory (n = 9000 uses W itself)."""
    a = _odd_csr(m, n, m + n)
    s = pkg.sparse_sign_new(d, m, zeta, 11)
    pat = orc.sparse_sign_pattern(d, m, zeta, 11)
    assert np.array_equal(s.apply_sparse(a), orc.sketch_apply_sparse(pat, a))


def test_csr_plan_rejects_bad_structure(pkg):
    import ctypes

    from paper_2311_04362_b200 import _lib
    from paper_2311_04362_b200 import device as dv

    dev = dv.current_device()
    lib = dv.lib(dev)
    ptr = torch.tensor([0, 2, 1, 3], dtype=torch.int64, device=dev)  # not monotone
    col = torch.tensor([0, 1, 2], dtype=torch.int32, device=dev)
    val = torch.ones(3, dtype=torch.float64, device=dev)
    h = ctypes.c_void_p()
    assert lib.itsk_csr_plan_create(dv.ptr(ptr), dv.ptr(col), dv.ptr(val), 3, 3, 3, dv.stream_ptr(),
                                    ctypes.byref(h)) == _lib.ITSK_EINVAL
    ptr = torch.tensor([0, 1, 2, 3], dtype=torch.int64, device=dev)
    col = torch.tensor([0, 5, 2], dtype=torch.int32, device=dev)  # column out of range
    assert lib.itsk_csr_plan_create(dv.ptr(ptr), dv.ptr(col), dv.ptr(val), 3, 3, 3, dv.stream_ptr(),
                                    ctypes.byref(h)) == _lib.ITSK_EINVAL


# --------------------------------------------------------------------------
# the pass: r bitwise scipy's b - A x, c = A'r to rounding
# --------------------------------------------------------------------------
@pytest.mark.parametrize("kind,m,n", [("gen", 20000, 100), ("gen", 200000, 10), ("odd", 3000, 60),
                                      ("odd", 1000, 2500), ("gen", 3, 3)])
def test_csr_pass_matches_scipy(pkg, kind, m, n):
    a = pkg.gen_sparse(m, n, 1).a if kind == "gen" else _odd_csr(m, n, 5)
    rng = np.random.default_rng(m)
    b, x, rp, rt = (rng.standard_normal(k) for k in (m, n, m, m))
    dev = torch.device("cuda", torch.cuda.current_device())
    A = pkg.CsrMatrix.from_scipy(a, dev)
    T = lambda v: torch.from_numpy(v).to(dev)  # noqa: E731
    r_out = torch.empty(m, dtype=torch.float64, device=dev)
    cs = A.pass_(T(b), T(x), r_out=r_out, r_prev=T(rp), r_true=T(rt)).cpu().numpy()
    r = b - a @ x
    assert np.array_equal(r_out.cpu().numpy(), r)  # csr_matvec's sequential row sums, bitwise
    c = a.T @ r
    scale = np.abs(a).T @ np.abs(r)
    assert np.all(np.abs(cs[:n] - c) <= 1e-13 * scale + 1e-300)
    assert cs[n] == pytest.approx(r @ r, rel=1e-12)
    assert cs[n + 1] == pytest.approx((r - rp) @ (r - rp), rel=1e-12)
    assert cs[n + 2] == pytest.approx((rt - r) @ (rt - r), rel=1e-12)
    assert cs[n + 3] == pytest.approx(b @ b, rel=1e-12)
    cs2 = A.pass_(T(b), T(x), r_prev=T(rp), r_true=T(rt)).cpu().numpy()
    # deterministic, with or without r_out (c and the four norms: the slots past them are scratch)
    assert np.array_equal(cs[:n + 4], cs2[:n + 4])


# --------------------------------------------------------------------------
# the solve
# --------------------------------------------------------------------------
@pytest.mark.parametrize("name", ["sp_basic", "sp_mom", "sp_damped", "sp_n3"])
def test_sparse_solve_parity_with_reference(pkg, g, name):
    m, n, seed = (int(v) for v in g[f"{name}_problem"])
    p = pkg.gen_sparse(m, n, seed)
    cfgd = json.loads(str(g[f"{name}_config"]))
    res = pkg.iterative_sketching(p.a, p.b, pkg.SolverConfig(**cfgd))
    tr = res.trace
    ref = g[f"{name}_iterates"]
    assert tr.stop_reason == str(g[f"{name}_stop"])
    assert len(tr.iterates) == len(ref)
    # S·A is bitwise, so R and x0 agree to LAPACK-vs-DMMA rounding; the loop's
    # A'r differs by summation order only
    x_ref = ref[-1]
    assert np.linalg.norm(res.solution - x_ref) <= 1e-10 * np.linalg.norm(x_ref)
    assert np.linalg.norm(tr.iterates[0] - ref[0]) <= 1e-10 * np.linalg.norm(ref[0])
    np.testing.assert_allclose([tr.normest, tr.condest], g[f"{name}_est"], rtol=1e-9)
    rn = np.array([np.linalg.norm(r) for r in tr.residual_vectors])
    np.testing.assert_allclose(rn, g[f"{name}_rnorms"], rtol=1e-10)
    # the final residual is the residual of the returned solution
    assert np.array_equal(tr.residual_vectors[-1], p.b - p.a @ res.solution)


def test_sparse_solve_device_csr_and_determinism(pkg):
    p = pkg.gen_sparse(30000, 64, 9)
    dev = torch.device("cuda", torch.cuda.current_device())
    A = pkg.CsrMatrix.from_scipy(p.a, dev)
    cfg = pkg.SolverConfig(d=1920, variant="momentum", max_iters=20, rng_seed=9)
    r1 = pkg.iterative_sketching(A, p.b, cfg)
    r2 = pkg.iterative_sketching(p.a, p.b, cfg)
    r3 = pkg.iterative_sketching(p.a, p.b, cfg, use_graph=False)
    assert np.array_equal(r1.solution, r2.solution) and np.array_equal(r2.solution, r3.solution)
    with pytest.raises(ValueError):
        pkg.iterative_sketching(p.a, p.b, pkg.SolverConfig(d=1920, track_be=True))


def test_sparse_graph_cache_two_matrices_same_shape(pkg):
    """Two different sparse A of the same shape (different nnz) solved back to
    back from scipy inputs (a fresh CsrMatrix per call): the cached loop
    graph of the first must not be replayed with the second's plan
    (plan addresses were reusable while a graph held them).  Each
    result equals the step-wise (no graph) solve of the same matrix."""
    cfg = pkg.SolverConfig(d=1920, variant="momentum", max_iters=20, rng_seed=9)
    p1 = pkg.gen_sparse(30000, 64, 9)
    p2 = pkg.gen_sparse(30000, 64, 10)
    assert p1.a.nnz != p2.a.nnz or not np.array_equal(p1.a.indices, p2.a.indices)
    want = [pkg.iterative_sketching(p.a, p.b, cfg, use_graph=False).solution for p in (p1, p2)]
    for _ in range(3):
        for p, w in zip((p1, p2), want):
            got = pkg.iterative_sketching(p.a, p.b, cfg)
            assert np.array_equal(got.solution, w)


# --------------------------------------------------------------------------
# CLI with the device flag
# --------------------------------------------------------------------------
def _csv(text):
    lines = [ln for ln in text.replace("\r\n", "\n").split("\n") if ln]
    return lines[0], lines[1], [ln.split(",") for ln in lines[2:]]


def test_cli_solve_matches_reference(pkg, g, tmp_path):
    from paper_2311_04362_b200.cli import main

    out = tmp_path / "x.csv"
    rc = main(["solve", "--m", "500", "--n", "10", "--cond", "1e6", "--resnorm", "1e-6", "--d", "200",
               "--out", str(out), "--device", "cuda:0"])
    assert rc == int(g["cli_solve_rc"])
    ref_x = [float(v) for v in str(g["cli_solve_x"]).split()[1:]]
    got = out.read_bytes().decode().split("\r\n")
    assert got[0] == "x" and got[-1] == ""
    x = np.array([float(v) for v in got[1:-1]])
    assert np.linalg.norm(x - ref_x) <= 1e-9 * np.linalg.norm(ref_x)
    s0, h, rows = _csv((tmp_path / "x.csv.summary.csv").read_text())
    rs0, rh, rrows = _csv(str(g["cli_solve_summary"]))
    assert (s0, h) == (rs0, rh) and len(rows) == 1
    assert rows[0][1] == rrows[0][1]                      # stop reason
    assert abs(int(rows[0][0]) - int(rrows[0][0])) <= 3   # iterations
    # fe: one-sided 2x, floored at kappa*u (both sit on the rounding plateau,
    # where reordering sums alone moves the reference's FE 0.1-1.5x)
    assert float(rows[0][2]) <= 2 * float(rrows[0][2]) + 1e6 * 2.0 ** -53
    assert rows[0][4] == "nan"


def test_cli_sparsebench_matches_reference(pkg, g, tmp_path):
    from paper_2311_04362_b200.cli import main

    out = tmp_path / "sp.csv"
    assert main(["sparsebench", "--rows", "2000", "--n", "40", "--repeats", "1", "--max-iters", "30",
                 "--out", str(out)]) == 0
    s0, h, rows = _csv(out.read_text())
    rs0, rh, rrows = _csv(str(g["cli_sparsebench"]))
    assert (s0, h) == (rs0, rh) and len(rows) == len(rrows) == 1
    assert rows[0][:3] == rrows[0][:3] and rows[0][4] == rrows[0][4]
    assert float(rows[0][5]) == pytest.approx(float(rrows[0][5]), rel=1e-10)


@pytest.mark.parametrize("cmd", ["compare", "convergence"])
def test_cli_trace_tables_match_reference(pkg, g, tmp_path, cmd):
    from paper_2311_04362_b200.cli import main

    out = tmp_path / f"{cmd}.csv"
    if cmd == "compare":
        argv = ["compare", "--m", "600", "--n", "12", "--cond", "1e8", "--resnorm", "1e-6", "--d", "240",
                "--max-iters", "40", "--out", str(out)]
    else:
        argv = ["convergence", "--m", "600", "--n", "12", "--cond", "1e4", "1e8", "--resnorm", "1e-6",
                "--d", "240", "--max-iters", "40", "--seed", "0", "1", "--out", str(out)]
    assert main(argv) == 0
    s0, h, rows = _csv(out.read_text())
    rs0, rh, rrows = _csv(str(g[f"cli_{cmd}"]))
    assert (s0, h) == (rs0, rh)

    def final(rs):
        last = {}
        for r in rs:
            key = (r[0], r[1], r[2])
            if int(r[3]) >= int(last.get(key, [0, 0, 0, -2])[3]):
                last[key] = r
        return last

    got, ref = final(rows), final(rrows)
    assert set(got) == set(ref)
    for key, r in ref.items():
        q = got[key]
        if key[0] == "householder_qr":
            # cuSOLVER's QR solve vs LAPACK's: both backward stable, FE at the
            # kappa*u rounding level
            assert float(q[4]) <= 2 * float(r[4]) + 10 * float(key[1]) * 2.0 ** -53, key
            continue
        assert abs(int(q[3]) - int(r[3])) <= max(3, int(0.15 * int(r[3]))), key
        # final forward / residual errors: one-sided 2x, floored at the
        # rounding plateau 10*kappa*u (the north-star's bound; reordering sums
        # alone moves the reference's own plateau FE 0.1-1.5x)
        plateau = 10 * float(key[1]) * 2.0 ** -53
        assert float(q[4]) <= 2 * float(r[4]) + plateau, key
        assert float(q[5]) <= 2 * float(r[5]) + plateau, key
    if cmd == "convergence":
        # the basic-variant bound columns (host formulas) equal the reference's
        bnd = {(r[1], r[2], r[3]): (r[8], r[9]) for r in rrows if r[0] == "is_basic"}
        for r in rows:
            if r[0] == "is_basic" and (r[1], r[2], r[3]) in bnd and bnd[(r[1], r[2], r[3])][0] != "nan":
                assert float(r[8]) == pytest.approx(float(bnd[(r[1], r[2], r[3])][0]), rel=1e-13)
