"""GPU parity: the B200 path (through the C-ABI / Python drop-in) against the
CPU oracle and the reference's golden fixtures.

Bars (per north_star): integer/byte work and the S·A sums bit-exact; the
refinement loop's FE/RE within 2x of the reference's (one-sided), and
||x - x_ref||/||x_ref|| <= 10*kappa*u + FE_ref; normest/condest to rounding.
"""

import ctypes
import hashlib
import json
import math

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


@pytest.fixture(scope="module")
def orc():
    from oracle import itsketch_oracle as o

    return o


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# --------------------------------------------------------------------------
# pattern + sketch (bit-exact)
# --------------------------------------------------------------------------
def test_pattern_matches_reference_bitwise(pkg, golden):
    g = golden("patterns.npz")
    for d, m, zeta, seed, k in g["pattern_cases"]:
        key = f"p_{d}_{m}_{zeta}_{seed}"
        s = pkg.sparse_sign_new(int(d), int(m), int(zeta), int(seed))
        np.testing.assert_array_equal(s.rows, g[key + "_rows"], err_msg=key)
        np.testing.assert_array_equal(s.signs, g[key + "_signs"], err_msg=key)
        a = np.random.default_rng(int(seed) + 100).standard_normal((int(m), int(k)))
        sa = s.apply_dense(a)
        assert np.array_equal(sa, g[key + "_sa"]), key
        # apply_vec == a column of apply_dense, bitwise (embed.py:69-74)
        assert np.array_equal(s.apply_vec(a[:, 0]), g[key + "_sa"][:, 0]), key


@pytest.mark.parametrize("div", ["2", "1000000"])
def test_pattern_short_first_draw_bitwise(pkg, golden, monkeypatch, div):
    """The first parallel draw given too few words (test hook): the one-CTA
    redraw kernel finishes it in stream order, then runs the redraw rounds;
    the pattern is still the reference's, bit for bit."""
    monkeypatch.setenv("ITSK_PATTERN_WORDS_DIV", div)
    g = golden("patterns.npz")
    for d, m, zeta, seed, k in g["pattern_cases"]:
        if int(m) * int(zeta) > 2_000_000:
            continue
        key = f"p_{d}_{m}_{zeta}_{seed}"
        s = pkg.sparse_sign_new(int(d), int(m), int(zeta), int(seed))
        np.testing.assert_array_equal(s.rows, g[key + "_rows"], err_msg=key)
        np.testing.assert_array_equal(s.signs, g[key + "_signs"], err_msg=key)


@pytest.mark.parametrize("d,m,zeta,seed", [(50, 20000, 8, 4), (400, 200000, 16, 5), (120, 60000, 12, 6)])
def test_pattern_many_redraws_bitwise(pkg, orc, d, m, zeta, seed):
    """Small d, large zeta: a large share of the columns repeats a row, so the
    first redraw rounds run as host-driven parallel draws before the one-CTA
    kernel takes the tail; the pattern is still numpy's, bit for bit."""
    s = pkg.sparse_sign_new(d, m, zeta, seed)
    p = orc.sparse_sign_pattern(d, m, zeta, seed)
    np.testing.assert_array_equal(s.rows, p.rows)
    np.testing.assert_array_equal(s.signs, p.signs)


def test_pattern_csr_grouping(pkg):
    s = pkg.sparse_sign_new(50, 400, 6, 9)
    ptr = s.ptr_dev.cpu().numpy().view(np.uint32).astype(np.int64)
    src = s.src_dev.cpu().numpy().view(np.uint32)
    assert ptr[0] == 0 and ptr[-1] == 400 * 6 and np.all(np.diff(ptr) >= 0)
    rows, signs = s.rows, s.signs
    for i in range(50):
        seg = src[ptr[i]:ptr[i + 1]]
        j = (seg & 0x7FFFFFFF).astype(np.int64)
        assert np.all(np.diff(j) > 0)  # ascending sources
        for jj, neg in zip(j, seg >> 31):
            t = int(np.nonzero(rows[jj] == i)[0][0])
            assert (signs[jj, t] < 0) == bool(neg)


def test_full_size_pattern_and_sketch_digests(pkg, golden, orc):
    g = golden("patterns.npz")
    for rec in json.loads(str(g["digests_json"])):
        s = pkg.sparse_sign_new(rec["d"], rec["m"], rec["zeta"], rec["seed"])
        if rec.get("kind") == "sa":
            a = np.random.default_rng(rec["a_seed"]).standard_normal((rec["m"], rec["k"]))
            assert _sha(s.apply_dense(a)) == rec["sa"]
        else:
            assert _sha(s.rows.astype(np.int64)) == rec["rows"], rec
            assert _sha(s.signs.astype(np.float64)) == rec["signs"], rec


SKETCH_VARIANTS = [
    {}, {"ITSK_SKETCH_UNR": "8"}, {"ITSK_SKETCH_UNR": "2"}, {"ITSK_SKETCH_GCPL": "2", "ITSK_SKETCH_UNR": "8"},
    {"ITSK_SKETCH_GCPL": "8", "ITSK_SKETCH_UNR": "4"},
    {"ITSK_SKETCH_GCPL": "4"}, {"ITSK_SKETCH_GCPL": "1"}, {"ITSK_SKETCH_RING": "1"},
    {"ITSK_SKETCH_RING": "0"},
]


@pytest.mark.parametrize("variant", SKETCH_VARIANTS)
def test_sketch_kernel_variants_bitwise(pkg, orc, monkeypatch, variant):
    """Every sketch kernel variant (register gather with 1..8 columns per lane
    and 2/4/8-source groups) equals scipy's order bitwise, for even and odd n,
    a padded leading dimension, and the fused b column."""
    for k, v in variant.items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng(11)
    for d, m, n, zeta in [(300, 5000, 40, 8), (64, 3000, 257, 4), (500, 2000, 3, 16), (40, 6000, 100, 8)]:
        pat = orc.sparse_sign_pattern(d, m, zeta, 2)
        s = pkg.sparse_sign_new(d, m, zeta, 2)
        a = rng.standard_normal((m, n))
        b = rng.standard_normal(m)
        ref = orc.sketch_apply(pat, np.column_stack([a, b]))
        dev = torch.device("cuda")
        lda = n + (n % 2) + 2                       # even, padded
        buf = torch.zeros((m, lda), dtype=torch.float64, device=dev)
        buf[:, :n] = torch.from_numpy(a).to(dev)
        got = s.apply_dense(buf[:, :n], torch.from_numpy(b).to(dev)).cpu().numpy()
        assert np.array_equal(got, ref), (variant, d, m, n, zeta)
        assert np.array_equal(s.apply_dense(a), ref[:, :n]), (variant, d, m, n, zeta)


@pytest.mark.parametrize("m,n,d,lda,withb", [(700000, 300, 6000, 300, True), (600000, 511, 2000, 512, True),
                                              (450000, 1000, 12000, 1000, True), (250001, 129, 700, 131, True),
                                              (300000, 256, 3000, 256, False), (90000, 40, 27000, 40, True),
                                              (120000, 70, 41000, 70, True)])
def test_sketch_window_sweep_bitwise(pkg, monkeypatch, m, n, d, lda, withb):
    """The window sweep (automatic from 2 GB of [A|b]: one persistent
    launch, the grid sweeping 20000-row source windows of one 128-column
    panel at a time with a bounded drift, each warp's (row, source) pairs
    materialised once in processing order and streamed) against the register gather
    (ITSK_SKETCH_SWEEP=0, itself bitwise scipy's order in the tests above):
    bitwise equal, including the fused b column, for both lane widths; odd
    leading dimension (the unvectorised loads), no b, a ragged last window,
    d beyond the grid's warps (up to 12 rows per warp, 27000 here; 41000: the
    64-column shape with up to 24 rows per warp)."""
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(m)
    buf = torch.randn(m, lda, dtype=torch.float64, device=dev, generator=g)
    a = buf[:, :n]
    b = torch.randn(m, dtype=torch.float64, device=dev, generator=g) if withb else None
    s = pkg.sparse_sign_new(d, m, 8, 5)
    monkeypatch.setenv("ITSK_SKETCH_SWEEP", "0")
    ref = s.apply_dense(a, b)
    monkeypatch.setenv("ITSK_SKETCH_DIRECT", "0")  # the materialised-order path (the direct mode has its own test)
    # window rows: default, small (many windows per chunk: a chunk spanning
    # more than `drift` windows must not wait for itself; warps without rows
    # must not run a counter ring ahead), 128- and 64-column panels
    for sweep, swcl, drift in (("1", "0", "2"), ("1", "2", "2"), ("7000", "0", "3"), ("7000", "2", "1"),
                               ("97", "0", "1")):
        if sweep == "97" and m > 300000:
            continue  # thousands of windows: on the smaller shapes only
        monkeypatch.setenv("ITSK_SKETCH_SWEEP", sweep)  # on below its automatic 2 GB threshold
        monkeypatch.setenv("ITSK_SKETCH_SWCL", swcl)
        monkeypatch.setenv("ITSK_SKETCH_DRIFT", drift)
        got = s.apply_dense(a, b)
        assert torch.equal(got, ref), (sweep, swcl, drift)


@pytest.mark.parametrize("m,n,d,zeta,lda,withb", [(400000, 100, 400, 8, 100, True), (300000, 100, 1200, 16, 102, True),
                                                   (250000, 37, 2000, 4, 37, True), (200000, 300, 500, 8, 300, False),
                                                   (150000, 511, 2368, 8, 512, True), (100000, 64, 90, 8, 64, True),
                                                   (50000, 200, 3, 2, 200, True)])
def test_sketch_direct_sweep_bitwise(pkg, monkeypatch, m, n, d, zeta, lda, withb):
    """The sweep's direct mode (no more sketch rows than the grid has warps: a
    warp owns one row and streams its entries straight from the pattern;
    chosen for wide rows of an A from 16 GB) against the register gather:
    bitwise equal for both lane widths, odd leading dimensions, no b, rows on
    only some of the warps, d equal to the number of warps, and windows of a
    few hundred rows."""
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(m + d)
    buf = torch.randn(m, lda, dtype=torch.float64, device=dev, generator=g)
    a = buf[:, :n]
    b = torch.randn(m, dtype=torch.float64, device=dev, generator=g) if withb else None
    s = pkg.sparse_sign_new(d, m, zeta, 7)
    monkeypatch.setenv("ITSK_SKETCH_SWEEP", "0")
    monkeypatch.setenv("ITSK_SKETCH_RING", "0")
    ref = s.apply_dense(a, b)
    monkeypatch.delenv("ITSK_SKETCH_RING")
    monkeypatch.setenv("ITSK_SKETCH_DIRECT", "1")
    for sweep, swcl, drift in (("1", "0", "2"), ("1", "2", "2"), ("3000", "0", "3"), ("3000", "2", "1"),
                               ("211", "0", "1"), ("211", "2", "2")):
        monkeypatch.setenv("ITSK_SKETCH_SWEEP", sweep)
        monkeypatch.setenv("ITSK_SKETCH_SWCL", swcl)
        monkeypatch.setenv("ITSK_SKETCH_DRIFT", drift)
        got = s.apply_dense(a, b)
        assert torch.equal(got, ref), (sweep, swcl, drift)


def test_pattern_argument_errors(pkg):
    with pytest.raises(ValueError):
        pkg.sparse_sign_new(3, 5, 4, 0)
    with pytest.raises(ValueError):
        pkg.sparse_sign_new(0, 5, 1, 0)
    s = pkg.sparse_sign_new(10, 20, 3, 0)
    with pytest.raises(ValueError):
        s.apply_dense(np.ones((21, 2)))
    assert np.all(s.apply_dense(np.zeros((20, 4))) == 0)


def test_sketch_c_abi_argument_errors(pkg):
    """itsk_sketch / itsk_sketch_rows refuse bad arguments with ITSK_EINVAL
    (-> ValueError) before touching memory: leading dimensions below n or
    from 2^31, a source-row window outside [0, m], null pointers, m from 2^31."""
    from paper_2311_04362_b200 import _lib
    from paper_2311_04362_b200 import device as dv

    dev = dv.current_device()
    lib = dv.lib(dev)
    s = pkg.sparse_sign_new(50, 200, 4, 0)
    a = torch.zeros((200, 8), dtype=torch.float64, device=dev)
    w = torch.zeros((50, 8), dtype=torch.float64, device=dev)
    st = dv.stream_ptr()
    P, S = dv.ptr(s.ptr_dev), dv.ptr(s.src_dev)

    def sketch(m=200, n=8, lda=8, ldw=8, A=dv.ptr(a), W=dv.ptr(w), ptr=P):
        return lib.itsk_sketch(A, m, n, lda, None, ptr, S, 50, 4, W, ldw, st)

    assert sketch() == _lib.ITSK_OK
    for kw in ({"lda": 7}, {"lda": 1 << 31}, {"ldw": 7}, {"A": None}, {"W": None}, {"ptr": None}, {"m": 1 << 31},
               {"m": 0}):
        with pytest.raises(ValueError):
            _lib.check(sketch(**kw))
    for r0, r1 in ((-1, 10), (10, 5), (0, 201)):
        with pytest.raises(ValueError):
            _lib.check(lib.itsk_sketch_rows(dv.ptr(a), 200, 8, 8, None, P, S, 50, 4, dv.ptr(w), 8, r0, r1, 0, st))
    torch.cuda.synchronize()


# --------------------------------------------------------------------------
# QR, triangular solves, estimates
# --------------------------------------------------------------------------
@pytest.mark.parametrize("m,n,seed", [(20, 5, 1), (200, 40, 2), (1000, 50, 3), (4000, 201, 4),
                                      (300, 33, 5), (64, 64, 6), (5000, 500, 7),
                                      # two-level blocking (n >= 384: outer blocks of 128 with a far
                                      # update): block-aligned, ragged last block, the C4 panel width
                                      (3000, 384, 8), (4100, 641, 9), (14000, 1000, 10), (16500, 1100, 11),
                                      # the C4 sketch's own shape (d = 24000, n = 2000)
                                      (24000, 2000, 12)])
def test_qr_matches_lapack(pkg, orc, m, n, seed):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((m, n))
    rhs = rng.standard_normal(m)
    f = pkg.householder_qr_econ(a, rhs)
    q_ref, r_ref = orc.householder_qr_econ(a)
    assert np.all(np.diag(f.r) >= 0)
    assert np.array_equal(f.r, np.triu(f.r))
    scale = np.linalg.norm(r_ref)
    assert np.linalg.norm(f.r - r_ref) <= 100 * n * U * scale
    z_ref = q_ref.T @ rhs
    assert np.linalg.norm(f.z - z_ref) <= 100 * n * U * np.linalg.norm(rhs)


@pytest.mark.parametrize("m,n,seed", [(14000, 1000, 10), (4100, 641, 9)])
def test_qr_sm_partition_bitwise(pkg, monkeypatch, m, n, seed):
    """The two-level QR's SM partition (green contexts: the panel chain on
    16 SMs, the GEMM-shaped updates on the rest) changes no operation order:
    R and z bitwise equal to the shared-SM run (ITSK_QR_GREEN=0), and the
    same on a repeat."""
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((m, n))
    rhs = rng.standard_normal(m)
    f1 = pkg.householder_qr_econ(a, rhs)
    f2 = pkg.householder_qr_econ(a, rhs)
    monkeypatch.setenv("ITSK_QR_GREEN", "0")
    f0 = pkg.householder_qr_econ(a, rhs)
    assert np.array_equal(f1.r, f2.r) and np.array_equal(f1.z, f2.z)
    assert np.array_equal(f1.r, f0.r) and np.array_equal(f1.z, f0.z)


@pytest.mark.parametrize("m,n,seed", [(40000, 64, 2), (30000, 130, 4)])
def test_qr_large_d_fallback_matches_lapack(pkg, orc, m, n, seed):
    """Beyond the panel kernel's shared memory (more than ~25600 rows at
    16-wide panels) itsk_qr_aug runs the single-kernel QR (qr.cu: one
    cluster, or the whole grid with barriers); held to the same bar as the
    panel / update path."""
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((m, n))
    rhs = rng.standard_normal(m)
    f = pkg.householder_qr_econ(a, rhs)
    q_ref, r_ref = orc.householder_qr_econ(a)
    assert np.all(np.diag(f.r) >= 0)
    assert np.linalg.norm(f.r - r_ref) <= 100 * n * U * np.linalg.norm(r_ref)
    assert np.linalg.norm(f.z - q_ref.T @ rhs) <= 100 * n * U * np.linalg.norm(rhs)


@pytest.mark.parametrize("m,n,seed", [(100000, 200, 3), (120001, 700, 5), (260000, 64, 7), (104000, 1000, 8)])
def test_qr_row_blocked_matches_lapack(pkg, orc, m, n, seed):
    """Beyond one factorisation's range (~50000 rows): TSQR over row blocks of
    <= 24000 rows, each with its share of the rhs column, then the stacked
    [R_i | z_i] — the same R (diag >= 0) and z = Q'b as LAPACK's single QR to
    the usual bar; no single set of reflectors, so .q says it is unavailable."""
    from paper_2311_04362_b200.linalg import qr_row_blocks

    rng = np.random.default_rng(seed)
    a = rng.standard_normal((m, n))
    rhs = rng.standard_normal(m)
    assert qr_row_blocks(m, n, torch.device("cuda", 0)) >= 2
    f = pkg.householder_qr_econ(a, rhs)
    q_ref, r_ref = orc.householder_qr_econ(a)
    assert np.all(np.diag(f.r) >= 0) and np.array_equal(f.r, np.triu(f.r))
    assert np.linalg.norm(f.r - r_ref) <= 100 * n * U * np.linalg.norm(r_ref)
    assert np.linalg.norm(f.z - q_ref.T @ rhs) <= 100 * n * U * np.linalg.norm(rhs)
    with pytest.raises(AttributeError, match="row-blocked"):
        f.q
    f2 = pkg.householder_qr_econ(a, rhs)
    assert np.array_equal(f.r, f2.r) and np.array_equal(f.z, f2.z)


def test_qr_hand_cases(pkg):
    f = pkg.householder_qr_econ(np.array([[3.0], [4.0]]))
    np.testing.assert_allclose(f.r, [[5.0]], rtol=1e-15)
    f = pkg.householder_qr_econ(np.eye(5))
    np.testing.assert_array_equal(f.r, np.eye(5))
    f = pkg.householder_qr_econ(-np.random.default_rng(7).standard_normal((12, 6)))
    assert np.all(np.diag(f.r) >= 0)
    with pytest.raises(ValueError):
        pkg.householder_qr_econ(np.ones((3, 5)))


def test_qr_singular_raises(pkg):
    a = np.random.default_rng(1).standard_normal((50, 6))
    a[:, 3] = 0.0
    with pytest.raises(pkg.SingularMatrixError):
        pkg.householder_qr_econ(a, np.ones(50))


def test_qr_deterministic(pkg):
    a = np.random.default_rng(9).standard_normal((3000, 120))
    f1, f2 = pkg.householder_qr_econ(a), pkg.householder_qr_econ(a)
    assert np.array_equal(f1.r, f2.r)


@pytest.mark.parametrize("m,n,seed,kappa", [(20, 5, 1, 1e2), (7, 7, 2, 1e1), (4000, 201, 4, 1e8), (14000, 1000, 10, 1e10),
                                             (40000, 64, 2, 1e4), (3000, 130, 6, 1e12)])
def test_qr_explicit_q(pkg, m, n, seed, kappa):
    """QrFactors.q (linalg.py:42-46: dorgqr's Q with the columns signed like
    R's rows), formed from the device QR's Householder vectors: orthonormal,
    Q R = A, Q'b = z, and equal to LAPACK's Q up to rounding times kappa —
    over the single-kernel, panel, two-level and large-d fallback paths."""
    rng = np.random.default_rng(seed)
    u0, _ = np.linalg.qr(rng.standard_normal((m, n)))
    v0, _ = np.linalg.qr(rng.standard_normal((n, n)))
    a = (u0 * np.logspace(0, -np.log10(kappa), n)) @ v0.T
    b = rng.standard_normal(m)
    f = pkg.householder_qr_econ(a, rhs=b)
    q, r = f.q, f.r
    u = np.finfo(float).eps
    assert q.shape == (m, n) and f.q is q
    assert np.linalg.norm(q.T @ q - np.eye(n)) <= 100 * n * u
    assert np.linalg.norm(q @ r - a) <= 100 * n * u * np.linalg.norm(a)
    assert np.linalg.norm(q.T @ b - f.z) <= 100 * n * u * np.linalg.norm(b)
    ql, rl = np.linalg.qr(a)
    sg = np.sign(np.diag(rl))
    ql = ql * sg
    if kappa <= 1e4:
        assert np.linalg.norm(q - ql) <= 100 * n * u * kappa
    # device input -> device Q
    ft = pkg.householder_qr_econ(torch.from_numpy(a).cuda())
    assert isinstance(ft.q, torch.Tensor) and np.array_equal(ft.q.cpu().numpy(), q)


def test_trsv_and_estimates_vs_reference(pkg, golden):
    g = golden("linalg.npz")
    import scipy.linalg as sl

    for i in range(5):
        r = g[f"tri{i}_r"]
        n = r.shape[0]
        c = np.random.default_rng(i).standard_normal(n)
        y = pkg.tri_solve_upper(r, c)
        np.testing.assert_allclose(y, sl.solve_triangular(r, c), rtol=1e-12, atol=1e-14)
        yt = pkg.tri_solve_upper_transpose(r, c)
        np.testing.assert_allclose(yt, sl.solve_triangular(r, c, trans="T"), rtol=1e-12, atol=1e-14)
        assert pkg.rand_power_norm_est(r, rng_seed=i) == pytest.approx(float(g[f"tri{i}_normest"]), rel=1e-12)
        assert pkg.cond_est(r) == pytest.approx(float(g[f"tri{i}_condest"]), rel=1e-9)
    with pytest.raises(pkg.SingularMatrixError):
        pkg.tri_solve_upper(np.array([[1.0, 2.0], [0.0, 0.0]]), np.ones(2))
    with pytest.raises(pkg.SingularMatrixError):
        pkg.tri_solve_upper_transpose(np.array([[1.0, 2.0], [0.0, 0.0]]), np.ones(2))


@pytest.mark.parametrize("n", [50, 200, 500, 1000])
def test_trsv_large_residual(pkg, n):
    rng = np.random.default_rng(n)
    r = np.triu(rng.standard_normal((n, n))) + (2.0 + n) * np.eye(n)
    c = rng.standard_normal(n)
    y = pkg.tri_solve_upper(r, c)
    kappa = np.linalg.cond(r)
    assert np.linalg.norm(r @ y - c) <= 100 * n * U * kappa * np.linalg.norm(c)
    yt = pkg.tri_solve_upper_transpose(r, c)
    assert np.linalg.norm(r.T @ yt - c) <= 100 * n * U * kappa * np.linalg.norm(c)


@pytest.mark.parametrize("n,kappa", [(50, 1e10), (200, 1e10), (200, 1e15), (257, 1e6), (33, 1e3), (500, 1e8)])
def test_trsv_rp_packed_layout(pkg, orc, n, kappa):
    """itsk_trsv_rp (R staged from itsk_pack_upper's layout, the diagonal-block
    inverses where kappa_1 <= 1e4: the loop tail's arithmetic; x0 and LSQR use
    it) on sketched R factors: residual bound of a backward-stable solve, and
    agreement with the substitution path (itsk_trsv) to kappa * u."""
    from paper_2311_04362_b200 import _lib
    from paper_2311_04362_b200 import device as dv

    a, _, _ = orc.gen_randsvd(max(4 * n, 400), n, kappa, 1e-6, n)
    _, r = orc.householder_qr_econ(orc.sketch_apply(orc.sparse_sign_pattern(2 * n, a.shape[0], 8, n), a))
    dev = dv.current_device()
    lib = dv.lib(dev)
    rt = torch.from_numpy(np.ascontiguousarray(r)).to(dev)
    nb = ctypes.c_int64()
    _lib.check(lib.itsk_pack_upper_doubles(n, ctypes.byref(nb)))
    rp = torch.empty(nb.value, dtype=torch.float64, device=dev)
    s = dv.stream_ptr()
    _lib.check(lib.itsk_pack_upper(dv.ptr(rt), n, dv.ptr(rp), s))
    c = np.random.default_rng(n).standard_normal(n)
    ct = torch.from_numpy(c).to(dev)
    kap = np.linalg.cond(r)
    for trans in (0, 1):
        y = torch.empty(n, dtype=torch.float64, device=dev)
        y0 = torch.empty(n, dtype=torch.float64, device=dev)
        _lib.check(lib.itsk_trsv_rp(dv.ptr(rt), dv.ptr(rp), n, dv.ptr(ct), dv.ptr(y), trans, s))
        _lib.check(lib.itsk_trsv(dv.ptr(rt), n, dv.ptr(ct), dv.ptr(y0), trans, s))
        y, y0 = y.cpu().numpy(), y0.cpu().numpy()
        m_ = r.T if trans else r
        assert np.linalg.norm(m_ @ y - c) <= 100 * n * U * np.linalg.norm(r) * np.linalg.norm(y), trans
        assert np.linalg.norm(y - y0) <= 100 * n * U * kap * np.linalg.norm(y0), trans


@pytest.mark.parametrize("n", [1500, 2000])
def test_estimates_global_r(pkg, orc, n):
    """n beyond the shared-memory packed R (C4: n = 2000): TRSV, normest and
    condest read R from global memory."""
    rng = np.random.default_rng(n)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    r = np.triu(q * np.logspace(0, -6, n)) + np.diag(np.logspace(0, -6, n))
    assert pkg.rand_power_norm_est(r, rng_seed=3) == pytest.approx(orc.rand_power_norm_est(r, rng_seed=3), rel=1e-12)
    assert pkg.cond_est(r) == pytest.approx(orc.cond_est(r), rel=1e-9)
    c = rng.standard_normal(n)
    y = pkg.tri_solve_upper(r, c)
    kappa = np.linalg.cond(r)
    assert np.linalg.norm(r @ y - c) <= 100 * n * U * kappa * np.linalg.norm(c)


def test_condest_on_sketch_factor(pkg, orc):
    a, b, t = orc.gen_randsvd(20000, 200, 1e10, 1e-12, 0)
    pat = orc.sparse_sign_pattern(4000, 20000, 8, 0)
    _, r = orc.householder_qr_econ(orc.sketch_apply(pat, a))
    assert pkg.cond_est(r) == pytest.approx(orc.cond_est(r), rel=1e-9)
    assert pkg.rand_power_norm_est(r, rng_seed=0) == pytest.approx(orc.rand_power_norm_est(r, rng_seed=0), rel=1e-12)


# --------------------------------------------------------------------------
# fused pass
# --------------------------------------------------------------------------
@pytest.mark.parametrize("m,n", [(1000, 1), (999, 7), (5000, 50), (20000, 200), (3001, 257), (4096, 500),
                                 (2000, 1000), (3000, 2000), (7, 4), (150, 64),
                                 # beyond the staged kernels' 2048 columns: the CTA-per-row kernel
                                 (1500, 2049), (1201, 3000), (700, 4097), (300, 6000), (5, 8192)])
def test_fused_pass_matches_numpy(pkg, m, n):
    import ctypes

    from paper_2311_04362_b200 import _lib
    from paper_2311_04362_b200 import device as dv

    rng = np.random.default_rng(m + n)
    a = rng.standard_normal((m, n))
    b = rng.standard_normal(m)
    x = rng.standard_normal(n)
    r_prev = rng.standard_normal(m)
    r_true = rng.standard_normal(m)
    dev = dv.current_device()
    T = lambda v: torch.from_numpy(v).to(dev)
    at, bt, xt, rpt, rtt = T(a), T(b), T(x), T(r_prev), T(r_true)
    r_out = torch.empty(m, dtype=torch.float64, device=dev)
    cs = torch.empty(n + 8, dtype=torch.float64, device=dev)
    lib = dv.lib(dev)
    nb = ctypes.c_int64()
    _lib.check(lib.itsk_pass_workspace(m, n, ctypes.byref(nb)))
    ws = dv.workspace(nb.value, dev)
    _lib.check(lib.itsk_fused_pass(dv.ptr(at), m, n, n, dv.ptr(bt), dv.ptr(xt), dv.ptr(rpt), dv.ptr(r_out),
                                   dv.ptr(rtt), dv.ptr(cs), dv.ptr(ws), ws.numel(), dv.stream_ptr()))
    torch.cuda.synchronize()
    r = b - a @ x
    c = a.T @ r
    got = cs.cpu().numpy()
    tol = 1e-13 * np.sqrt(n)
    np.testing.assert_allclose(r_out.cpu().numpy(), r, rtol=0, atol=tol * np.abs(a).sum(1).max() * 10)
    assert np.linalg.norm(got[:n] - c) <= 1e-13 * np.linalg.norm(np.abs(a).T @ np.abs(r)) * 10
    assert got[n] == pytest.approx(r @ r, rel=1e-12)
    assert got[n + 1] == pytest.approx((r - r_prev) @ (r - r_prev), rel=1e-12)
    assert got[n + 2] == pytest.approx((r_true - r) @ (r_true - r), rel=1e-12)
    assert got[n + 3] == pytest.approx(b @ b, rel=1e-12)


@pytest.mark.parametrize("m,n,lda", [(5003, 513, 514), (4099, 1025, 1026), (6001, 2047, 2048), (777, 1500, 1500),
                                     (9, 2000, 2000), (3001, 1800, 2300), (1000, 2048, 2048), (2500, 1409, 1410),
                                     (2500, 1408, 1500), (1203, 1999, 2600)])
def test_fused_pass_wide_padded_rows(pkg, m, n, lda):
    """Wide rows (512 < n <= 2048: the row-group kernel up to n = 1408, the
    row-slot kernel above) with NaN in every pad column (an odd n stored at an
    even leading dimension; a leading dimension well beyond n, which the
    row-slot kernel's per-row copies do not stage): the pads must never enter
    r, c or the norms; batches of 4 rows with a ragged last batch (m not a
    multiple of 4 per CTA)."""
    import ctypes

    from paper_2311_04362_b200 import _lib
    from paper_2311_04362_b200 import device as dv

    rng = np.random.default_rng(m * n)
    a = rng.standard_normal((m, n))
    b = rng.standard_normal(m)
    x = rng.standard_normal(n)
    r_prev = rng.standard_normal(m)
    dev = dv.current_device()
    store = torch.full((m, lda), float("nan"), dtype=torch.float64, device=dev)
    store[:, :n] = torch.from_numpy(a).to(dev)
    bt, xt, rpt = (torch.from_numpy(v).to(dev) for v in (b, x, r_prev))
    r_out = torch.empty(m, dtype=torch.float64, device=dev)
    cs = torch.empty(n + 8, dtype=torch.float64, device=dev)
    lib = dv.lib(dev)
    nb = ctypes.c_int64()
    _lib.check(lib.itsk_pass_workspace(m, n, ctypes.byref(nb)))
    ws = dv.workspace(nb.value, dev)
    _lib.check(lib.itsk_fused_pass(dv.ptr(store), m, n, lda, dv.ptr(bt), dv.ptr(xt), dv.ptr(rpt), dv.ptr(r_out),
                                   None, dv.ptr(cs), dv.ptr(ws), ws.numel(), dv.stream_ptr()))
    torch.cuda.synchronize()
    r = b - a @ x
    c = a.T @ r
    got = cs.cpu().numpy()
    assert np.isfinite(got[: n + 4]).all() and np.isfinite(r_out.cpu().numpy()).all()
    np.testing.assert_allclose(r_out.cpu().numpy(), r, rtol=0, atol=1e-13 * np.sqrt(n) * np.abs(a).sum(1).max() * 10)
    assert np.linalg.norm(got[:n] - c) <= 1e-13 * np.linalg.norm(np.abs(a).T @ np.abs(r)) * 10
    assert got[n] == pytest.approx(r @ r, rel=1e-12)
    assert got[n + 1] == pytest.approx((r - r_prev) @ (r - r_prev), rel=1e-12)
    assert got[n + 2] == 0.0
    assert got[n + 3] == pytest.approx(b @ b, rel=1e-12)


@pytest.mark.parametrize("m,n", [(200000, 200), (40000, 2000), (5000, 50)])
def test_fused_pass_ws_ready_is_bitwise_stable(pkg, m, n):
    """itsk_pass_workspace_init once, then repeated itsk_fused_pass_ex with
    ITSK_PASS_WS_READY (no per-call reset): every call returns the bytes of
    the resetting entry point — the counters do reset themselves."""
    import ctypes

    from paper_2311_04362_b200 import _lib
    from paper_2311_04362_b200 import device as dv

    dev = dv.current_device()
    g = torch.Generator(device=dev).manual_seed(m + n)
    a = torch.randn(m, n, dtype=torch.float64, device=dev, generator=g)
    b = torch.randn(m, dtype=torch.float64, device=dev, generator=g)
    x = torch.randn(n, dtype=torch.float64, device=dev, generator=g)
    lib = dv.lib(dev)
    nb = ctypes.c_int64()
    _lib.check(lib.itsk_pass_workspace(m, n, ctypes.byref(nb)))
    ws = dv.workspace(nb.value, dev)
    ws.fill_(255)  # garbage counters: the init must clear them
    s = dv.stream_ptr()
    ref = torch.empty(n + 8, dtype=torch.float64, device=dev)
    _lib.check(lib.itsk_fused_pass(dv.ptr(a), m, n, n, dv.ptr(b), dv.ptr(x), None, None, None, dv.ptr(ref),
                                   dv.ptr(ws), ws.numel(), s))
    ws.fill_(255)
    _lib.check(lib.itsk_pass_workspace_init(dv.ptr(ws), m, n, s))
    for _ in range(4):
        cs = torch.full((n + 8,), float("nan"), dtype=torch.float64, device=dev)
        _lib.check(lib.itsk_fused_pass_ex(dv.ptr(a), m, n, n, dv.ptr(b), 1.0, dv.ptr(x), None, None, None,
                                          dv.ptr(cs), dv.ptr(ws), ws.numel(), _lib.PASS_WS_READY, s))
        assert torch.equal(cs[: n + 4], ref[: n + 4])
    assert lib.itsk_fused_pass_ex(dv.ptr(a), m, n, n, dv.ptr(b), 1.0, dv.ptr(x), None, None, None, dv.ptr(cs),
                                  dv.ptr(ws), ws.numel(), 6, s) == _lib.ITSK_EINVAL


# --------------------------------------------------------------------------
# the drop-in solve
# --------------------------------------------------------------------------
SOLVE_NAMES = ["c1_basic", "c1_damped", "c1_momentum", "c1_seed1", "c3like", "bitwise", "consistent", "extra3",
               "zero_init", "be_direct", "be_fast", "diverge", "maxit0", "eps_override", "c4proxy_mom"]


def _problem(orc, g, name):
    m, n, kappa, beta, seed = g[f"{name}_problem"]
    a, b, truth = orc.gen_randsvd(int(m), int(n), kappa, beta, int(seed))
    cfg = json.loads(str(g[f"{name}_config"]))
    return a, b, truth, cfg


# Golden cases held to a different bar than the strict 2x (the measured
# per-case ratios are in profiles/r2_strict_bar.txt, scripts/strict_bar.py):
STRICT_EXCEPTIONS = {
    # zero init is the paper's deliberately unstable "bad_init" baseline
    # (solvers.py:364-365): its forward-error plateau is set by early rounding
    # errors; reordering only the reference's own matvec sums moves its FE
    # 12-40x (1.9e-7 -> 2.3e-6..7.5e-6), so the 2x bar does not apply.  The
    # same order of magnitude as that spread is required (measured: 22x).
    "zero_init": ("order_of_magnitude",),
    # beta = 0: both runs end at the rounding floor (FE 6.5e-15 vs 2.4e-15,
    # kappa = 1e3, kappa*u = 1.1e-13); a 2x bar on rounding noise below the
    # floor is not meaningful, the bar is max(2x reference, 10 kappa u).
    "consistent": ("rounding_floor",),
}


@pytest.mark.parametrize("name", SOLVE_NAMES)
def test_solve_parity_with_reference(pkg, orc, golden, name):
    g = golden("solves.npz")
    a, b, truth, cfgd = _problem(orc, g, name)
    t = pkg.Truth(x=truth.x, r=truth.r, kappa=truth.kappa, beta=truth.beta)
    res = pkg.iterative_sketching(a, b, pkg.SolverConfig(**cfgd), t)
    tr = res.trace
    ref_stop = str(g[f"{name}_stop"])
    ref_iters = len(g[f"{name}_iterates"]) - 1
    assert len(tr.iterates) == res.iterations + 1
    assert len(tr.residual_changes) == res.iterations
    assert len(tr.fe) == len(tr.re) == res.iterations + 1
    assert tr.normest == pytest.approx(float(g[f"{name}_normest"]), rel=1e-10)
    # R differs from LAPACK's by rounding; sigma_min(R) moves by ~kappa*u relative
    kap = float(g[f"{name}_condest"])
    assert tr.condest == pytest.approx(kap, rel=max(1e-9, 10 * kap * U))
    fe_ref, re_ref = g[f"{name}_fe"], g[f"{name}_re"]
    # iterate 0 is the sketch-and-solve start: agree to rounding of the QR
    if name != "diverge":
        assert tr.fe[0] <= 2 * fe_ref[0] + 1e-14 and fe_ref[0] <= 2 * tr.fe[0] + 1e-14
    if ref_stop == "diverged":
        assert tr.stop_reason == "diverged"
        return
    if ref_stop == "max_iters" and cfgd.get("max_iters", 50) <= 30:
        assert tr.stop_reason == "max_iters" and res.iterations == ref_iters
    else:
        assert tr.stop_reason == ref_stop
        # rounding moves the stop iteration by a few (survey §8c: C1 24-30 vs 26-29)
        assert abs(res.iterations - ref_iters) <= max(3, 0.15 * ref_iters), (res.iterations, ref_iters)
    if name in STRICT_EXCEPTIONS:
        kind = STRICT_EXCEPTIONS[name][0]
        if kind == "order_of_magnitude":
            assert tr.fe[-1] <= 50 * fe_ref[-1], (tr.fe[-1], fe_ref[-1])
        else:  # "rounding_floor": both runs at kappa*u; the bar is the floor
            floor = 10 * truth.kappa * U
            assert tr.fe[-1] <= max(2 * fe_ref[-1], floor), (tr.fe[-1], fe_ref[-1], floor)
            assert tr.re[-1] <= max(2 * re_ref[-1], floor), (tr.re[-1], re_ref[-1], floor)
        return
    # the north-star bar, strict: FE and RE within 2x of the reference's own
    # final values (one-sided; + a few u of absolute slack for u-level errors)
    assert tr.fe[-1] <= 2 * fe_ref[-1] + 4 * U, (tr.fe[-1], fe_ref[-1])
    assert tr.re[-1] <= 2 * re_ref[-1] + 4 * U, (tr.re[-1], re_ref[-1])
    if len(g[f"{name}_be"]):
        assert tr.be[-1] <= 2 * g[f"{name}_be"][-1] + 4 * U
    x_ref = g[f"{name}_solution"]
    dev_x = np.linalg.norm(res.solution - x_ref) / np.linalg.norm(x_ref)
    # triangle inequality always holds for two accurate solutions
    assert dev_x <= tr.fe[-1] + fe_ref[-1] + 4 * U


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_c2_shape_parity_and_stated_bound(pkg, orc, seed):
    """C2 shape (200000 x 200, kappa 1e10, beta 1e-12, d = 20n): the stated
    bound ||x - x_ref||/||x_ref|| <= 10 kappa u + FE_ref holds with margin."""
    a, b, truth = orc.gen_randsvd(200000, 200, 1e10, 1e-12, seed)
    cfg = orc.Config(d=4000, rng_seed=seed)
    x_ref, tr_ref = orc.iterative_sketching(a, b, cfg, truth)
    t = pkg.Truth(x=truth.x, r=truth.r, kappa=truth.kappa, beta=truth.beta)
    res = pkg.iterative_sketching(a, b, pkg.SolverConfig(d=4000, rng_seed=seed), t)
    assert res.trace.stop_reason == tr_ref.stop_reason
    assert res.trace.fe[-1] <= 2 * tr_ref.fe[-1]
    assert res.trace.re[-1] <= 2 * tr_ref.re[-1]
    dev_x = np.linalg.norm(res.solution - x_ref) / np.linalg.norm(x_ref)
    assert dev_x <= 10 * truth.kappa * U + tr_ref.fe[-1]


def test_update_identity_bit_for_bit(pkg):
    """GPU analogue of test_update_identity_bit_for_bit (test_solvers.py:223-233):
    x_{i+1} == fl(x_i + R^{-1}R^{-T}A'r_i) with the device's own kernels."""
    p = pkg.gen_randsvd(500, 12, 1e4, 1e-3, 3)
    res = pkg.iterative_sketching(p.a, p.b, pkg.SolverConfig(d=240, max_iters=6, rng_seed=3), p.truth)
    s = pkg.sparse_sign_new(240, 500, 8, 3)
    f = pkg.householder_qr_econ(s.apply_dense(p.a))
    dev = torch.device("cuda")
    at = torch.from_numpy(p.a).to(dev)
    r_dev = torch.from_numpy(f.r).to(dev)
    tr = res.trace
    for i in range(len(tr.iterates) - 1):
        c = at.T @ torch.from_numpy(tr.residual_vectors[i]).to(dev)
        d = pkg.tri_solve_upper(r_dev, pkg.tri_solve_upper_transpose(r_dev, c))
        # c from cuBLAS here vs the fused pass in the solver: compare to rounding
        step = tr.iterates[i + 1] - tr.iterates[i]
        np.testing.assert_allclose(step, d.cpu().numpy(), rtol=1e-9, atol=1e-15)


def test_bitwise_determinism_and_graph_equivalence(pkg):
    p = pkg.gen_randsvd(600, 15, 1e6, 1e-4, 5)
    cfg = pkg.SolverConfig(d=300, max_iters=40, rng_seed=5)
    r1 = pkg.iterative_sketching(p.a, p.b, cfg, p.truth)
    r2 = pkg.iterative_sketching(p.a, p.b, cfg, p.truth)
    r3 = pkg.iterative_sketching(p.a, p.b, cfg, p.truth, use_graph=False)
    for r in (r2, r3):
        assert np.array_equal(r1.solution, r.solution)
        assert r1.trace.fe == r.trace.fe
        assert r1.trace.residual_changes == r.trace.residual_changes
        assert r1.trace.stop_reason == r.trace.stop_reason


def test_device_tensor_inputs_zero_copy(pkg):
    p = pkg.gen_randsvd(3000, 40, 1e8, 1e-6, 2)
    cfg = pkg.SolverConfig(d=800, variant="momentum", rng_seed=2)
    r_host = pkg.iterative_sketching(p.a, p.b, cfg)
    at = torch.from_numpy(p.a).cuda()
    bt = torch.from_numpy(p.b).cuda()
    r_dev = pkg.iterative_sketching(at, bt, cfg)
    assert np.array_equal(r_host.solution, r_dev.solution)
    # a strided view (lda > n) is used in place
    big = torch.zeros((3000, 48), dtype=torch.float64, device="cuda")
    big[:, :40] = at
    r_view = pkg.iterative_sketching(big[:, :40], bt, cfg)
    assert np.array_equal(r_host.solution, r_view.solution)


@pytest.mark.parametrize("m,n,kappa,d", [(4000, 50, 1e10, 1000), (20000, 200, 1e10, 4000), (20000, 100, 1e15, 2000),
                                         (6000, 257, 1e6, 2000), (30000, 1000, 1e8, 12000), (100, 1, 1.0, 10),
                                         (300, 33, 1e3, 100)])
def test_condest_inverse_operator_matches_trsv_operator(pkg, orc, m, n, kappa, d):
    """itsk_condest_ws (Lanczos on X X' with X = R^-1 formed once) against
    itsk_condest (two triangular solves per step) and the exact kappa."""
    from paper_2311_04362_b200 import _lib
    from paper_2311_04362_b200 import device as dv

    if n == 1:
        a = np.random.default_rng(0).standard_normal((m, 1))
    else:
        a, _, _ = orc.gen_randsvd(m, n, kappa, 1e-6, 1)
    _, r = orc.householder_qr_econ(orc.sketch_apply(orc.sparse_sign_pattern(d, m, 8, 1), a))
    dev = dv.current_device()
    rt = torch.from_numpy(np.ascontiguousarray(r)).to(dev)
    lib = dv.lib(dev)
    v0 = torch.from_numpy(np.random.default_rng(1).standard_normal(n)).to(dev)
    o1 = torch.empty(1, dtype=torch.float64, device=dev)
    o2 = torch.empty(1, dtype=torch.float64, device=dev)
    import ctypes

    nws = ctypes_i64()
    lib.itsk_condest_workspace(n, ctypes.byref(nws))
    ws = torch.empty(nws.value, dtype=torch.float64, device=dev)
    rp = torch.empty(_rp_len(lib, n), dtype=torch.float64, device=dev)
    _lib.check(lib.itsk_pack_upper(dv.ptr(rt), n, dv.ptr(rp), dv.stream_ptr()))
    _lib.check(lib.itsk_condest(dv.ptr(rt), n, dv.ptr(v0), dv.ptr(o1), dv.ptr(rp), dv.stream_ptr()))
    _lib.check(lib.itsk_condest_ws(dv.ptr(rt), n, dv.ptr(v0), dv.ptr(o2), dv.ptr(rp), dv.ptr(ws), ws.numel(),
                                   dv.stream_ptr()))
    c1, c2 = float(o1.item()), float(o2.item())
    exact = orc.cond_est(r)
    assert c2 == pytest.approx(c1, rel=1e-10)
    assert c2 == pytest.approx(exact, rel=1e-9)
    # X really is R^-1 (upper triangle)
    x = np.triu(ws[: n * n].view(n, n).cpu().numpy())
    assert np.linalg.norm(x @ r - np.eye(n)) <= 1e3 * n * U * np.linalg.norm(x) * np.linalg.norm(r)


def ctypes_i64():
    import ctypes

    return ctypes.c_int64()


def _rp_len(lib, n):
    import ctypes

    v = ctypes.c_int64()
    lib.itsk_pack_upper_doubles(n, ctypes.byref(v))
    return v.value


def test_chunked_upload_and_sketch_windows_bitwise(pkg, orc):
    """A host A >= 32 MB is uploaded in row chunks and sketched window by
    window as it lands (itsk_sketch_rows): the solve is bitwise the one from
    the device-resident A, and any row windows taken in order reproduce the
    one-shot sketch bit for bit."""
    import ctypes

    from paper_2311_04362_b200 import _lib
    from paper_2311_04362_b200 import device as dv

    m, n = 40000, 120  # 38 MB -> the pipelined path
    rng = np.random.default_rng(7)
    a = rng.standard_normal((m, n)) / np.sqrt(m)
    b = rng.standard_normal(m)
    cfg = pkg.SolverConfig(d=2400, max_iters=12, rng_seed=7)
    pinned = torch.from_numpy(a).pin_memory()
    r_host = pkg.iterative_sketching(pinned.numpy(), b, cfg)
    r_page = pkg.iterative_sketching(a, b, cfg)
    r_dev = pkg.iterative_sketching(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), cfg)
    assert np.array_equal(r_host.solution, r_dev.solution)
    assert np.array_equal(r_page.solution, r_dev.solution)
    # windows
    s = pkg.sparse_sign_new(500, 3000, 8, 3)
    a2 = torch.from_numpy(rng.standard_normal((3000, 37))).cuda()
    b2 = torch.from_numpy(rng.standard_normal(3000)).cuda()
    ref = s.apply_dense(a2, b2)
    lib = dv.lib(a2.device)
    for cuts in ([0, 3000], [0, 1, 1500, 1501, 3000], [0, 700, 700, 2999, 3000]):
        w = torch.full((500, 38), float("nan"), dtype=torch.float64, device=a2.device)
        for k in range(len(cuts) - 1):
            _lib.check(lib.itsk_sketch_rows(dv.ptr(a2), 3000, 37, 37, dv.ptr(b2), dv.ptr(s.ptr_dev), dv.ptr(s.src_dev),
                                            500, 8, dv.ptr(w), 38, cuts[k], cuts[k + 1], 1 if k else 0,
                                            dv.stream_ptr()))
        assert torch.equal(w, ref), cuts
    assert lib.itsk_sketch_rows(dv.ptr(a2), 3000, 37, 37, dv.ptr(b2), dv.ptr(s.ptr_dev), dv.ptr(s.src_dev), 500, 8,
                                dv.ptr(w), 38, 10, 5, 0, dv.stream_ptr()) == _lib.ITSK_EINVAL
    del ctypes


def test_pageable_upload_staging_is_exact(pkg):
    """A pageable host matrix >= 32 MB goes through two pinned 64 MB staging
    buffers (device.upload_rows_staged); several pieces per call and two
    calls back to back (the buffers and their events are reused): the device
    copy equals the plain one bit for bit, also for a strided source."""
    from paper_2311_04362_b200 import device as dv

    dev = dv.current_device()
    rng = np.random.default_rng(3)
    big = rng.standard_normal((70000, 401))          # 224 MB: 4 pieces
    strided = rng.standard_normal((30000, 500))[:, :333]  # rows of a wider array
    for arr in (big, strided, big[:12345]):
        t, lda = dv.as_device_matrix(arr, dev)
        torch.cuda.synchronize()
        assert lda == arr.shape[1]
        assert torch.equal(t.cpu(), torch.from_numpy(np.ascontiguousarray(arr)))


def test_edge_configs(pkg, orc):
    # zeta == d, zeta == 1, odd n, residuals="last", extra_iters
    for (m, n, d, zeta) in [(300, 7, 10, 10), (500, 9, 40, 1), (2001, 33, 300, 3)]:
        a, b, truth = orc.gen_randsvd(m, n, 1e3, 1e-3, 1)
        cfg_o = orc.Config(d=d, zeta=zeta, rng_seed=1, max_iters=60)
        x_ref, tr_ref = orc.iterative_sketching(a, b, cfg_o, truth)
        t = pkg.Truth(x=truth.x, r=truth.r, kappa=truth.kappa, beta=truth.beta)
        res = pkg.iterative_sketching(a, b, pkg.SolverConfig(d=d, zeta=zeta, rng_seed=1, max_iters=60), t,
                                      residuals="last")
        assert res.trace.stop_reason == tr_ref.stop_reason
        assert res.trace.fe[-1] <= 2 * tr_ref.fe[-1] + 4 * U
        np.testing.assert_allclose(res.trace.residual_vectors[-1], b - a @ res.solution, atol=1e-13)
        if res.iterations >= 2:
            with pytest.raises(IndexError):
                res.trace.residual_vectors[0]


def test_validation_and_singular(pkg):
    p = pkg.gen_randsvd(100, 10, 10.0, 0.1, 0)
    with pytest.raises(ValueError):
        pkg.iterative_sketching(p.a, p.b, pkg.SolverConfig(d=5))
    with pytest.raises(ValueError):
        pkg.iterative_sketching(p.a, p.b, pkg.SolverConfig(d=50, variant="bogus"))
    a = p.a.copy()
    a[:, 4] = 0.0
    with pytest.raises(pkg.SingularMatrixError):
        pkg.iterative_sketching(a, p.b, pkg.SolverConfig(d=50))


@pytest.mark.parametrize("shape", [(400, 10, 200), (6000, 130, 2600), (20000, 400, 8000)])
def test_nonfinite_inputs_raise_like_the_reference(pkg, orc, shape):
    """NaN / Inf in A or b: the reference fails in sketch_and_solve's
    triangular solve (scipy solve_triangular's check_finite, linalg.py:59-62)
    with ValueError("array must not contain infs or NaNs") — the oracle does
    the same here — and so does the device path (a flag bit set by the QR's
    finish kernel, read with the results), in iterative_sketching,
    sketch_and_precondition, sketch_and_solve and the triangular solves;
    householder_qr_econ itself returns the NaNs like LAPACK's QR (linalg.py:42).
    A zero pivot still wins over a non-finite entry (_check_square_upper first)."""
    m, n, d = shape
    p = pkg.gen_randsvd(m, n, 10.0, 0.1, 0)
    cfg = pkg.SolverConfig(d=d)
    for what, val in (("a", np.nan), ("a", np.inf), ("b", np.nan), ("b", -np.inf)):
        a, b = p.a.copy(), p.b.copy()
        (a if what == "a" else b)[m // 3, ...] = val
        with pytest.raises(ValueError, match="infs or NaNs"):
            orc.iterative_sketching(a, b, orc.Config(d=d))
        with pytest.raises(ValueError, match="infs or NaNs"):
            pkg.iterative_sketching(a, b, cfg)
        with pytest.raises(ValueError, match="infs or NaNs"):
            pkg.sketch_and_precondition(a, b, cfg)
        with pytest.raises(ValueError, match="infs or NaNs"):
            pkg.sketch_and_solve(a, b, pkg.sparse_sign_new(d, m, 8, 0))
    a = p.a.copy()
    a[5, 2] = np.nan
    f = pkg.householder_qr_econ(a)
    assert not np.all(np.isfinite(f.r))
    with pytest.raises(ValueError, match="infs or NaNs"):
        pkg.tri_solve_upper(f.r, np.ones(n))
    with pytest.raises(ValueError, match="infs or NaNs"):
        pkg.tri_solve_upper_transpose(np.eye(3), np.array([1.0, np.inf, 0.0]))
    # the workspace is reusable after the error, and a clean solve is unaffected
    res = pkg.iterative_sketching(p.a, p.b, cfg)
    x_ref, tr_ref = orc.iterative_sketching(p.a, p.b, orc.Config(d=d))
    it_ref = len(tr_ref.iterates) - 1
    assert res.trace.stop_reason == tr_ref.stop_reason and abs(res.iterations - it_ref) <= max(3, 0.15 * it_ref)
    assert np.linalg.norm(res.solution - x_ref) <= 1e-8 * np.linalg.norm(x_ref)
    a = p.a.copy()
    a[:, 4] = 0.0
    a[7, 1] = np.nan  # a zero column AND a NaN: R has a NaN pivot row, not a zero pivot -> ValueError
    with pytest.raises((ValueError, pkg.SingularMatrixError)):
        pkg.iterative_sketching(a, p.b, cfg)


def test_wide_problem_parity(pkg, orc):
    """n beyond the staged pass kernels' 2048 columns (the CTA-per-row pass,
    the cluster tail and the global-R estimates): 15000 x 2100, momentum,
    against the oracle on the same bytes — FE / RE within 2x, the stated
    bound on x, the estimates to rounding."""
    m, n, kappa, beta, d = 15000, 2100, 1e6, 1e-8, 16800
    a, b, t = orc.gen_randsvd(m, n, kappa, beta, 0)
    x_ref, tr = orc.iterative_sketching(a, b, orc.Config(d=d, variant="momentum"), t)
    truth = pkg.Truth(x=t.x, r=t.r, kappa=t.kappa, beta=t.beta)
    res = pkg.iterative_sketching(a, b, pkg.SolverConfig(d=d, variant="momentum"), truth)
    it_ref = len(tr.iterates) - 1
    # as at C4 (tests/test_gpu_c4.py): with 2100-term dots the rule's threshold
    # lies under OpenBLAS's dgemv noise, so the oracle may run to max_iters where
    # the device path stops by the rule; never the other way round
    assert res.trace.stop_reason == "stopped_by_rule", res.trace.stop_reason
    assert tr.stop_reason == "max_iters" or abs(res.iterations - it_ref) <= max(3, 0.15 * it_ref), (
        res.iterations, it_ref, tr.stop_reason)
    assert res.trace.fe[-1] <= 2 * tr.fe[-1] and res.trace.re[-1] <= 2 * tr.re[-1]
    assert np.linalg.norm(res.solution - x_ref) / np.linalg.norm(x_ref) <= 10 * kappa * U + tr.fe[-1]
    assert res.trace.normest == pytest.approx(tr.normest, rel=1e-10)
    assert res.trace.condest == pytest.approx(tr.condest, rel=1e-8)


def test_input_forms(pkg, orc):
    """np.asarray(a, dtype=float) semantics of the reference's entry point
    (solvers.py:323-329): Fortran-ordered, column-strided, row-sliced and
    non-contiguous device inputs and a list b give the contiguous float64
    solve bit for bit; float32 / integer A are converted like the reference
    converts them; a wrong-length b and a 1-D A raise ValueError."""
    a, b, _ = orc.gen_randsvd(4000, 50, 1e6, 1e-6, 0)
    cfg = pkg.SolverConfig(d=1000)
    ref = pkg.iterative_sketching(a, b, cfg).solution
    forms = {
        "fortran": (np.asfortranarray(a), b),
        "column-strided": (np.ascontiguousarray(np.hstack([a, a]))[:, :50], b),
        "row-sliced": (np.vstack([a, a])[:4000], b),
        "list b": (a, list(b)),
        "device, non-contiguous": (torch.from_numpy(np.asfortranarray(a)).cuda(), torch.from_numpy(b).cuda()),
    }
    for name, (aa, bb) in forms.items():
        x = pkg.iterative_sketching(aa, bb, cfg).solution
        x = x.cpu().numpy() if isinstance(x, torch.Tensor) else x
        assert np.array_equal(x, ref), name
    for aa in (a.astype(np.float32), np.round(a * 1e3).astype(np.int64)):
        x = pkg.iterative_sketching(aa, b, cfg).solution
        x_ref, _ = orc.iterative_sketching(np.asarray(aa, dtype=float), b, orc.Config(d=1000))
        assert np.linalg.norm(x - x_ref) <= 1e-9 * np.linalg.norm(x_ref), aa.dtype
    with pytest.raises(ValueError):
        pkg.iterative_sketching(a, b[:-1], cfg)
    with pytest.raises(ValueError):
        pkg.iterative_sketching(a[:, 0], b, cfg)


def test_residual_vectors_survive_workspace_reuse(pkg):
    p = pkg.gen_randsvd(800, 10, 1e3, 1e-3, 4)
    cfg = pkg.SolverConfig(d=200, rng_seed=4)
    r1 = pkg.iterative_sketching(p.a, p.b, cfg)
    q = pkg.gen_randsvd(800, 10, 1e3, 1e-3, 5)
    pkg.iterative_sketching(q.a, q.b, cfg)
    np.testing.assert_allclose(r1.trace.residual_vectors[-1], p.b - p.a @ r1.solution, atol=1e-12)
    np.testing.assert_allclose(r1.trace.residual_vectors[0], p.b - p.a @ r1.trace.iterates[0], atol=1e-12)


@pytest.mark.slow
@pytest.mark.parametrize("seed", [0, 1])
def test_c3_full_size_parity(pkg, orc, seed):
    """C3 at full size (1e6 x 500, kappa 1e15, beta 1e-3, d = 20n): the
    device-built instance (instances.gen_randsvd_device; the host generator
    takes minutes here) is copied to the host and both sides solve the same
    bytes.  S·[A|b] bitwise; FE/RE one-sided within 2x; the stated bound."""
    from paper_2311_04362_b200.instances import gen_randsvd_device

    p = gen_randsvd_device(1_000_000, 500, 1e15, 1e-3, seed)
    a_h, b_h = p.a.cpu().numpy(), p.b.cpu().numpy()
    r_h = p.truth.r.cpu().numpy()
    otruth = orc.Truth(x=p.truth.x, r=r_h, kappa=1e15, beta=1e-3)
    # the sketch, bitwise, on the full instance
    s = pkg.sparse_sign_new(10000, 1_000_000, 8, seed)
    sab = s.apply_dense(p.a, p.b).cpu().numpy()
    pat = orc.sparse_sign_pattern(10000, 1_000_000, 8, seed)
    assert np.array_equal(sab, orc.sketch_apply(pat, np.column_stack([a_h, b_h])))
    del sab
    cfg = orc.Config(d=10000, rng_seed=seed)
    x_ref, tr_ref = orc.iterative_sketching(a_h, b_h, cfg, otruth)
    res = pkg.iterative_sketching(p.a, p.b, pkg.SolverConfig(d=10000, rng_seed=seed), p.truth, residuals="last")
    tr = res.trace
    dev_x = np.linalg.norm(res.solution - x_ref) / np.linalg.norm(x_ref)
    print(f"C3 seed {seed}: iters {res.iterations} vs {len(tr_ref.iterates) - 1}, FE {tr.fe[-1]:.3e} vs "
          f"{tr_ref.fe[-1]:.3e}, RE {tr.re[-1]:.3e} vs {tr_ref.re[-1]:.3e}, |x-x_ref|/|x_ref| {dev_x:.3e}")
    # kappa u = 0.11: R carries O(1) relative perturbations, so the contraction
    # rate — and the stop iteration — is rounding-driven here (not compared)
    assert tr.stop_reason == tr_ref.stop_reason
    assert tr.fe[-1] <= 2 * tr_ref.fe[-1], (tr.fe[-1], tr_ref.fe[-1])
    assert tr.re[-1] <= 2 * tr_ref.re[-1], (tr.re[-1], tr_ref.re[-1])
    assert dev_x <= 10 * 1e15 * U + tr_ref.fe[-1]


@pytest.mark.parametrize("n,kappa,illblock", [(500, 1e8, False), (1000, 1e10, False), (2000, 1e8, False),
                                              (2047, 1e6, True), (4096, 1e4, False), (777, 1e12, True)])
def test_trsv_pair_cluster(pkg, n, kappa, illblock):
    """The cluster solve pair (itsk_trsv_pair_cl, the loop tail's solves for
    large n) against a float64 reference solve: residual-based bar as the
    single-CTA TRSV tests; with `illblock` some diagonal blocks are made
    ill conditioned so the register substitution path runs instead of the
    stored inverse.  Bitwise reproducible across runs."""
    from paper_2311_04362_b200 import _lib
    from paper_2311_04362_b200 import device as dv

    rng = np.random.default_rng(n)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    s = kappa ** (-np.arange(n) / (n - 1))
    r = np.linalg.qr((q * s) @ np.linalg.qr(rng.standard_normal((n, n)))[0].T, mode="r")
    r = r * np.sign(np.diag(r))[:, None]
    if illblock:
        # two diagonal blocks made ill conditioned (kappa_1 past the inverse's
        # threshold): their solves take the register substitution chain
        for b0 in (64, 32 * (n // 64)):
            r[b0 + 5, b0 + 5] *= 1e-6
    c = rng.standard_normal(n)
    dev = torch.device("cuda")
    R = torch.from_numpy(np.ascontiguousarray(r)).to(dev)
    nb = ctypes.c_int64()
    lib = dv.lib(dev)
    _lib.check(lib.itsk_pack_upper_doubles(n, ctypes.byref(nb)))
    Rp = torch.empty(nb.value, dtype=torch.float64, device=dev)
    _lib.check(lib.itsk_pack_upper(dv.ptr(R), n, dv.ptr(Rp), dv.stream_ptr()))
    ct = torch.from_numpy(c).to(dev)
    outs = []
    for rep in range(3):
        d = torch.full((n,), float("nan"), dtype=torch.float64, device=dev)
        _lib.check(lib.itsk_trsv_pair_cl(dv.ptr(R), dv.ptr(Rp), n, dv.ptr(ct), dv.ptr(d), dv.stream_ptr()))
        outs.append(d.cpu().numpy())
    assert all(np.array_equal(o, outs[0]) for o in outs[1:])
    d = outs[0]
    assert np.isfinite(d).all()
    # backward-error form: R' R d = c to ~ n u ||R||^2 ||d||
    res = r.T @ (r @ d) - c
    assert np.linalg.norm(res) <= 100 * n * U * np.linalg.norm(r, 2) ** 2 * np.linalg.norm(d) + 100 * n * U * np.linalg.norm(c)
    import scipy.linalg as sl
    ref = sl.solve_triangular(r, sl.solve_triangular(r, c, trans="T"))
    cond = np.linalg.cond(r)
    assert np.linalg.norm(d - ref) <= 1e3 * n * U * cond ** 2 * np.linalg.norm(ref) + 1e-300
