"""C5 (BASELINE configs[4]: the sketch-only sweep) at its own cell sizes: the
kernel the library chooses by itself for every m = 2^20 cell (n in {100, 500,
2000} x d in {4n, 12n, 20n} x zeta in {4, 8, 16}: ring, one- and two-column
register gather, materialised and direct window sweep) is bitwise equal to
the plain one-column register gather, and a column subset — the fused b
column included — is bitwise equal to the CPU oracle's sequential sum
(scipy's csc_matvecs order, oracle.sketch_apply) on the same bytes.  Two
larger cells cover the choices that depend on the size of A (the direct sweep
from 16 GB, the two-column gather on 13 GB).  Seeded Gaussian A on the device
stands in for the sweep's inputs."""

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


@pytest.fixture(scope="module")
def orc():
    from oracle import itsketch_oracle as o

    return o


def _check_cell(pkg, orc, monkeypatch, a, b, d, zeta, seed):
    m, n = a.shape
    s = pkg.sparse_sign_new(d, m, zeta, seed)
    for k in ("ITSK_SKETCH_SWEEP", "ITSK_SKETCH_RING", "ITSK_SKETCH_GCPL", "ITSK_SKETCH_UNR", "ITSK_SKETCH_DIRECT"):
        monkeypatch.delenv(k, raising=False)
    got = s.apply_dense(a, b)  # the automatic choice
    monkeypatch.setenv("ITSK_SKETCH_SWEEP", "0")
    monkeypatch.setenv("ITSK_SKETCH_RING", "0")
    monkeypatch.setenv("ITSK_SKETCH_GCPL", "1")
    plain = s.apply_dense(a, b)
    assert torch.equal(got, plain), (m, n, d, zeta)
    # the oracle on a column subset: first, an interior pair, the last column of A, and b
    cols = sorted({0, n // 2, n // 2 + 1, n - 1})
    sub = np.column_stack([a[:, cols].cpu().numpy(), b.cpu().numpy()])
    pat = orc.Pattern(d=d, m=m, zeta=zeta, rows=np.asarray(s.rows).astype(np.int64),
                      signs=np.asarray(s.signs).astype(np.float64), scale=s.scale)
    ref = orc.sketch_apply(pat, sub)
    assert np.array_equal(got[:, cols + [n]].cpu().numpy(), ref), (m, n, d, zeta)


@pytest.mark.parametrize("n", [100, 500, 2000])
def test_c5_cells_at_2_to_20_bitwise(pkg, orc, monkeypatch, n):
    m = 1 << 20
    g = torch.Generator(device="cuda").manual_seed(n)
    a = torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g)
    b = torch.randn(m, dtype=torch.float64, device="cuda", generator=g)
    for d in (4 * n, 12 * n, 20 * n):
        for zeta in (4, 8, 16):
            _check_cell(pkg, orc, monkeypatch, a, b, d, zeta, seed=d + zeta)


@pytest.mark.parametrize("m,n,d,zeta", [(1 << 24, 100, 2000, 8), (1 << 24, 500, 2000, 8)])
def test_c5_large_cells_bitwise(pkg, orc, monkeypatch, m, n, d, zeta):
    free, _ = torch.cuda.mem_get_info()
    if free < 8 * m * n * 1.3:
        pytest.skip("not enough free device memory for this cell")
    g = torch.Generator(device="cuda").manual_seed(m + n)
    a = torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g)
    b = torch.randn(m, dtype=torch.float64, device="cuda", generator=g)
    _check_cell(pkg, orc, monkeypatch, a, b, d, zeta, seed=3)
    del a, b
    torch.cuda.empty_cache()
