"""Host <-> device plumbing of round 2 (paper_2508_08062_b200/csrc/memory.cu,
engine.cu): the device block cache reused across handles of different
shapes, page-locked and pageable host buffers, the lazily grown safeguard
table, and max_iters at the top of the size_t range. Every case must give
the bit-identical SERIAL trajectory of a fresh reference solve."""
import numpy as np
import pytest

from oracle.pyoracle import Oracle
from paper_2508_08062_b200 import Method, Solver, SolverConfig, problems

pytestmark = pytest.mark.gpu


def cfg(max_iters=300, **kw):
    return SolverConfig(method=Method.AA_PDHG, m=5, toll=1e-7, max_iters=max_iters,
                        reduction="serial", **kw)


def same(a, b):
    assert a.result.iterations == b.result.iterations
    assert np.array_equal(a.trajectory["g_norm"], b.trajectory["g_norm"])
    assert np.array_equal(a.result.u.x, b.result.u.x)
    assert np.array_equal(a.result.u.y, b.result.u.y)


def test_block_cache_across_handles_of_different_shapes():
    port = Oracle("port")
    shapes = [0.1, 0.2, 0.1, 0.15, 0.2, 0.1]
    want = {sc: port.solve(problems.make_config(0, scale=sc), cfg()) for sc in set(shapes)}
    for sc in shapes:  # handles come and go; their blocks are reused in between
        p = problems.make_config(0, scale=sc)
        with Solver(p) as s:
            same(s.solve(cfg()), want[sc])


@pytest.mark.parametrize("blocks", [False, True])
def test_pinned_and_pageable_inputs_and_outputs_agree(blocks, monkeypatch):
    """Page-locked inputs take the two-phase ingestion (the values over PCIe on
    a side stream while every layout's structure is built, then the value
    fills); pageable ones the one-phase path: identical solves. `blocks`: with
    L2 column blocks (tiny ones) so the blocks' structure / value split runs."""
    import torch
    if blocks:
        monkeypatch.setenv("AAPDHG_L2_BLOCK_MIN_KB", "0")
        monkeypatch.setenv("AAPDHG_L2_BLOCK_KB", "16")
    p = problems.make_config(1, scale=0.05)
    with Solver(p) as s:
        a = s.solve(cfg())
    keep = []

    def pin(x):
        t = torch.empty(x.shape, dtype=torch.from_numpy(np.empty(0, x.dtype)).dtype, pin_memory=True)
        keep.append(t)
        v = t.numpy()
        v[...] = x
        return v

    from paper_2508_08062_b200.api import ProblemData, SparseMatrix
    k = SparseMatrix(p.k.nrows, p.k.ncols, pin(p.k.row_ptr), pin(p.k.col_idx), pin(p.k.vals))
    hp = ProblemData(k, p.m1, pin(p.c), pin(p.q), pin(p.l), pin(p.u))
    outs = (pin(np.empty(p.n())), pin(np.empty(p.k.nrows)), pin(np.empty(p.n())))
    with Solver(hp) as s:
        b = s.solve(cfg(), out=outs)
    same(a, b)
    assert b.result.u.x is outs[0]
    assert np.array_equal(a.result.lambda_, b.result.lambda_)


@pytest.mark.parametrize("blocks", [False, True])
@pytest.mark.parametrize("method", [Method.AA_PDHG, Method.PDHG])
def test_result_download_beside_the_last_iteration(blocks, method, monkeypatch):
    """Page-locked x / y of a large LP leave on a side stream while the last
    iteration runs (engine.cu: the launches stop one short of max_iters);
    forced on a small LP (AAPDHG_OUT_OVERLAP_MB=0). TREE solves that stop on
    max_iters (0, 1, 7, 40), on the residual, or on KKT must equal the same
    solves into pageable buffers bit for bit (the overlap off)."""
    import torch
    if blocks:
        monkeypatch.setenv("AAPDHG_L2_BLOCK_MIN_KB", "0")
        monkeypatch.setenv("AAPDHG_L2_BLOCK_KB", "16")
    p = problems.make_config(1, scale=0.05)
    n, m = p.n(), p.k.nrows
    outs = tuple(torch.empty(k, dtype=torch.float64, pin_memory=True).numpy() for k in (n, m, n))
    cases = [dict(max_iters=mi) for mi in (0, 1, 7, 40)]
    cases += [dict(max_iters=5000, toll=1e-4), dict(max_iters=5000, kkt_terminate=True, kkt_eps=1e-3)]
    with Solver(p) as s:
        for kw in cases:
            c = SolverConfig(method=method, m=5, reduction="tree", **{"toll": 1e-12, **kw})
            monkeypatch.setenv("AAPDHG_OUT_OVERLAP_MB", "1000000")
            a = s.solve(c)
            monkeypatch.setenv("AAPDHG_OUT_OVERLAP_MB", "0")
            for v in outs:
                v[...] = np.nan
            b = s.solve(c, out=outs)
            assert a.result.status == b.result.status, kw
            assert a.result.iterations == b.result.iterations, kw
            assert np.array_equal(a.trajectory["g_norm"], b.trajectory["g_norm"]), kw
            assert np.array_equal(a.result.u.x, b.result.u.x), kw
            assert np.array_equal(a.result.u.y, b.result.u.y), kw
            assert np.array_equal(a.result.lambda_, b.result.lambda_), kw
            assert a.result.g_norm == b.result.g_norm and a.result.objective == b.result.objective


def test_safeguard_table_grows_and_max_iters_saturates():
    """A 7,575-iteration solve with 473 AA steps (config 0 at scale 0.1,
    toll 1e-5): launches after the first grow the table; then the same solve
    with max_iters = 2^64 - 1 (no wrap, the table still sized lazily). Both
    equal the oracle bit for bit."""
    port = Oracle("port")
    p = problems.make_config(0, scale=0.1)
    c1 = SolverConfig(method=Method.AA_PDHG, m=5, toll=1e-5, max_iters=60000, reduction="serial")
    huge = SolverConfig(method=Method.AA_PDHG, m=5, toll=1e-5, max_iters=2**64 - 1,
                        reduction="serial")
    want = port.solve(p, c1)
    assert want.result.status.name == "RESIDUAL_TOL" and want.result.i > 400
    with Solver(p) as s:
        got = s.solve(c1)
        got2 = s.solve(huge)
    same(got, want)
    same(got2, want)
