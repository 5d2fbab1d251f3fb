"""GPU: problem ingestion on the device (ingest.cu) on awkward shapes — empty
rows and columns, rows at and just past the long-row threshold (256), one
very long row, all-long matrices, no nonzeros — checked bit for bit against
the oracle's CSR-ordered matvec / matvec_transpose (SERIAL layouts) and the
first iterates of a TREE solve (its own layouts, split factors and SELL-σ)."""
import ctypes as C

import numpy as np
import pytest

from oracle.pyoracle import Oracle
from paper_2508_08062_b200 import (Method, ProblemData, Solver, SolverConfig, SparseMatrix,
                                   _abi)
from paper_2508_08062_b200.api import check, errbuf

pytestmark = pytest.mark.gpu


def lp_from_rows(row_cols, n, seed):
    """LP with the given column sets per row, N(0,1) values, planted-ish data."""
    rng = np.random.default_rng(seed)
    rows, cols = [], []
    for r, cs in enumerate(row_cols):
        cs = np.unique(np.asarray(cs, dtype=np.int64))
        rows += [r] * len(cs)
        cols += list(cs)
    m = len(row_cols)
    vals = rng.standard_normal(len(rows))
    k = SparseMatrix.from_triplets(m, n, np.array(rows, dtype=np.int64),
                                   np.array(cols, dtype=np.int64), vals)
    c = rng.random(n)
    q = rng.standard_normal(m)
    return ProblemData(k, m // 3, c, q, np.zeros(n), np.where(rng.random(n) < 0.5, 3.0, np.inf))


def shapes():
    rng = np.random.default_rng(11)
    n = 700
    out = {}
    # empty rows and columns, rows of 256 and 257 entries (threshold), short rows
    rc = [[] for _ in range(5)] + [rng.choice(n - 50, 256, replace=False),
                                   rng.choice(n - 50, 257, replace=False)]
    rc += [rng.choice(n - 50, int(rng.integers(1, 30)), replace=False) for _ in range(90)]
    out["edges"] = (rc, n)
    # one very long row among length-1 rows (Zipf-like extremes)
    rc = [np.arange(0, n, 1)] + [[int(rng.integers(0, n))] for _ in range(200)]
    out["one_long"] = (rc, n)
    # every row long
    out["all_long"] = ([rng.choice(n, 300 + 40 * i, replace=False) for i in range(9)], n)
    # rows at and past the CTA-per-row threshold (1024) beside warp-per-row
    # and short rows
    nh = 6000
    rc = [rng.choice(nh, L, replace=False) for L in (5000, 1024, 1023, 2000, 300)]
    rc += [rng.choice(nh, int(rng.integers(1, 40)), replace=False) for _ in range(60)]
    out["huge"] = (rc, nh)
    return out


@pytest.fixture(scope="module")
def port():
    return Oracle("port")


@pytest.mark.parametrize("name", ["edges", "one_long", "all_long", "huge"])
def test_device_layouts_bitwise(name, port):
    rc, n = shapes()[name]
    p = lp_from_rows(rc, n, seed=len(name))
    rng = np.random.default_rng(1)
    x = rng.standard_normal(p.n())
    y = rng.standard_normal(p.k.nrows)
    y[::7] = 0.0  # matvec_transpose skips zero y entries
    with Solver(p) as s:
        err = errbuf()
        kx = np.empty(p.k.nrows)
        check(s.lib.aapdhg_cuda_matvec(s.h, _abi.dptr(x), _abi.dptr(kx), err, len(err)), err)
        kty = np.empty(p.n())
        check(s.lib.aapdhg_cuda_matvec_transpose(s.h, _abi.dptr(y), _abi.dptr(kty), err,
                                                 len(err)), err)
        assert np.array_equal(kx, port.matvec(p, x))
        assert np.array_equal(kty, port.matvec_transpose(p, y))
        for red in ("serial", "tree"):
            cfg = SolverConfig(method=Method.AA_PDHG, m=5, toll=1e-12, max_iters=40, tau=0.01,
                               sigma=0.01, reduction=red)
            got = s.solve(cfg)
            ref = port.solve(p, cfg)
            if red == "serial":
                assert np.array_equal(got.trajectory["g_norm"], ref.trajectory["g_norm"])
            else:
                np.testing.assert_allclose(got.trajectory["g_norm"][:30],
                                           ref.trajectory["g_norm"][:30], rtol=1e-10)


@pytest.mark.parametrize("name", ["huge", "all_long", "one_long"])
def test_long_row_paths_agree(name, monkeypatch, port):
    """The TREE long-row paths — a CTA per row (AAPDHG_HUGE), a warp per row,
    a warp per 512-entry chunk with the last chunk adding the chunk sums in
    order (AAPDHG_LONG_CHUNK=1, opt-in) — on rows of 300..5000 entries, the
    first 30 iterates against the oracle at 1e-10."""
    rc, n = shapes()[name]
    p = lp_from_rows(rc, n, seed=len(name))
    cfg = SolverConfig(method=Method.AA_PDHG, m=5, toll=1e-12, max_iters=40, tau=0.01,
                       sigma=0.01, reduction="tree")
    ref = port.solve(p, cfg)
    for huge, chunk in (("1", "0"), ("0", "0"), ("0", "1")):
        monkeypatch.setenv("AAPDHG_HUGE", huge)
        monkeypatch.setenv("AAPDHG_LONG_CHUNK", chunk)
        with Solver(p) as s:
            got = s.solve(cfg)
            got2 = s.solve(cfg)  # (the chunk tickets reset for the next launch)
        np.testing.assert_allclose(got.trajectory["g_norm"][:30], ref.trajectory["g_norm"][:30],
                                   rtol=1e-10, err_msg=f"HUGE={huge} LONG_CHUNK={chunk}")
        assert np.array_equal(got.trajectory["g_norm"], got2.trajectory["g_norm"])


def test_no_nonzeros(port):
    m, n = 4, 6
    k = SparseMatrix(m, n, np.zeros(m + 1, dtype=np.int32), np.zeros(0, dtype=np.int32),
                     np.zeros(0))
    p = ProblemData(k, 1, np.linspace(-1, 1, n), np.arange(m, dtype=float), np.zeros(n),
                    np.full(n, 2.0))
    cfg = SolverConfig(method=Method.PDHG, toll=1e-9, max_iters=30, reduction="serial")
    with Solver(p) as s:
        got = s.solve(cfg)
    ref = port.solve(p, cfg)
    assert got.result.status == ref.result.status
    assert np.array_equal(got.trajectory["g_norm"], ref.trajectory["g_norm"])
    assert got.result.steps.tau == ref.result.steps.tau == 1.0  # all-zero K


def test_unsorted_columns_rejected():
    from paper_2508_08062_b200 import DimensionError
    k = SparseMatrix(1, 3, np.array([0, 2], dtype=np.int32), np.array([2, 0], dtype=np.int32),
                     np.array([1.0, 2.0]))
    p = ProblemData(k, 0, np.zeros(3), np.ones(1), np.zeros(3), np.full(3, np.inf))
    with pytest.raises(DimensionError):
        Solver(p)
