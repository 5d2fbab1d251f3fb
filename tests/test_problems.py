"""Synthetic stand-ins for BASELINE.json's configs and the
host-side model types. CPU only."""
import numpy as np
import pytest

from paper_2508_08062_b200 import problems
from paper_2508_08062_b200.api import (DimensionError, InputError, Method, ProblemData,
                                       SolverConfig, SparseMatrix, vstack)


def _rows(k):
    return np.repeat(np.arange(k.nrows), np.diff(k.row_ptr))


def _check_csr(k):
    assert k.row_ptr[0] == 0 and k.row_ptr[-1] == k.nnz
    assert np.all(np.diff(k.row_ptr) >= 0)
    r = _rows(k)
    key = r.astype(np.int64) * k.ncols + k.col_idx
    assert np.all(np.diff(key) > 0), "columns strictly increasing within rows"


def test_config0_shape_and_planted_optimum():
    p = problems.make_config(0)
    assert (p.k.nrows, p.k.ncols, p.k.nnz, p.m1) == (1000, 2000, 20000, 0)
    _check_csr(p.k)
    assert np.all(p.l == 0) and np.all(np.isinf(p.u))
    # b = A x*, c = A'y* + s*, s* complementary to x*  =>  c'x* = b'y*
    assert abs(p.c @ p.planted_x - p.q @ p.planted_y) < 1e-9 * abs(p.c @ p.planted_x)
    assert np.all(p.planted_x[p.c - p.k.transpose().dense() @ p.planted_y > 1e-12] == 0)


def test_config1_distinct_rows_per_column():
    p = problems.make_config(1, scale=0.02)
    _check_csr(p.k)
    assert np.all(np.bincount(p.k.col_idx, minlength=p.n()) == 20)


def test_transport_structure():
    p = problems.make_config(2, scale=0.01)  # 20 x 20
    S = T = 20
    _check_csr(p.k)
    assert p.k.nrows == S + T and p.n() == S * T and p.k.nnz == 2 * S * T
    assert np.all(np.bincount(p.k.col_idx) == 2)
    assert abs(p.q[:S].sum() - p.q[S:].sum()) < 1e-9
    assert np.all(np.diff(p.k.row_ptr) == np.r_[np.full(S, T), np.full(T, S)])


def test_zipf_row_lengths():
    p = problems.make_config(3, scale=0.002)
    _check_csr(p.k)
    lens = np.diff(p.k.row_ptr)
    assert lens.min() >= 1 and (lens == 1).mean() > 0.3


def test_from_triplets_sums_duplicates_in_order():
    k = SparseMatrix.from_triplets(2, 3, [1, 0, 1, 1], [2, 1, 2, 0], [0.1, 5.0, 0.2, 7.0])
    assert k.row_ptr.tolist() == [0, 1, 3]
    assert k.col_idx.tolist() == [1, 0, 2]
    assert k.vals.tolist() == [5.0, 7.0, 0.1 + 0.2]
    with pytest.raises(DimensionError):
        SparseMatrix.from_triplets(1, 1, [1], [0], [1.0])


def test_transpose_keeps_row_order():
    p = problems.make_config(0, scale=0.1)
    kt = p.k.transpose()
    _check_csr(kt)
    np.testing.assert_array_equal(kt.dense(), p.k.dense().T)


def test_vstack_and_problem_validation():
    a = SparseMatrix.from_triplets(1, 2, [0], [1], [2.0])
    b = SparseMatrix.from_triplets(2, 2, [0, 1], [0, 0], [1.0, 3.0])
    k = vstack(a, b)
    assert k.dense().tolist() == [[0, 2], [1, 0], [3, 0]]
    with pytest.raises(DimensionError):
        ProblemData(k, 1, np.zeros(3), np.zeros(3), np.zeros(2), np.ones(2))


def test_config_params_validation():
    cfg = SolverConfig(method=Method.AA_PDHG, reduction="bogus")
    with pytest.raises(InputError):
        cfg.to_params(4)
    cfg = SolverConfig(aa=type(SolverConfig().aa)(d_hat=np.ones(3)))
    with pytest.raises(DimensionError):
        cfg.to_params(4)


def test_instance_cache_round_trip(tmp_path, monkeypatch):
    """problems.cached_config: generated once into .npy files (a completion
    marker written last), memory-mapped afterwards; identical to make_config."""
    monkeypatch.setenv("AAPDHG_INSTANCE_CACHE", str(tmp_path))
    a = problems.cached_config(1, 0.05)
    d = problems.cache_dir(1, 0.05)
    assert (d / "complete").exists()
    b = problems.cached_config(1, 0.05, generate=False)  # mapped, not regenerated
    ref = problems.make_config(1, 0.05)
    for x in (a, b):
        assert np.array_equal(x.k.row_ptr, ref.k.row_ptr)
        assert np.array_equal(x.k.col_idx, ref.k.col_idx)
        assert np.array_equal(x.k.vals, ref.k.vals)
        for f in ("c", "q", "l", "u"):
            assert np.array_equal(getattr(x, f), getattr(ref, f))
        assert x.planted_objective == ref.planted_objective
    with pytest.raises(FileNotFoundError):
        problems.cached_config(1, 0.07, generate=False)


def test_bench_iteration_bytes_and_workload_selection():
    import argparse
    import bench
    p = problems.make_config(1, 0.05)
    n, m, nnz = p.n(), p.k.nrows, p.k.nnz
    plain = bench.kernel_bytes(p, "k_plain_loop")
    # (the ring history: g_k stored, 8 bytes per element and iteration)
    assert plain == (12 * nnz + 4 * (n + 1) + 8 * m + 48 * n) + (12 * nnz + 4 * (m + 1) + 8 * n + 48 * m)
    N = n + m
    aa = 8 * N * 11 + 8 * N * 14 + 12 * nnz + 4 * (m + 1) + 8 * n + 8 * m
    assert bench.iteration_bytes(p, 20, 3) == 20 * plain + 3 * aa
    # configs[4] at every N (BENCH and the scaling curve share the LP)
    args = argparse.Namespace(workload="config4", loopback=0)
    bench.select_workload(args, 1)
    assert bench.CONFIG_ID == 4 and "configs[4]" in bench.METRIC
    bench.select_workload(args, 8)
    assert bench.CONFIG_ID == 4 and "configs[4]" in bench.METRIC
    bench.select_workload(argparse.Namespace(workload="config1", loopback=0), 1)
    assert bench.CONFIG_ID == 1 and "configs[1]" in bench.METRIC
    # the column-pass bytes of configs[4]'s layout (K': 3 blocks of y, K: 5 of x)
    class _K:
        nrows, nnz = 20_000_000, 400_000_000
    class _P:
        k = _K()
        def n(self):
            return 40_000_000
    pb = bench.kernel_bytes(_P(), "k_spmv_pass")
    assert 1.0e9 < pb < 2.5e9


def test_stable_argsort_paths_agree():
    """problems._argsort_stable: the torch path (used on a GPU box for the
    150-400M-key sorts of configs 3 and 4) gives numpy's stable permutation,
    equal keys included, and np.lexsort((val, grp)) equals the combined-key
    sort the generator uses."""
    rng = np.random.default_rng(11)
    grp = np.repeat(np.arange(3000, dtype=np.int64), rng.integers(1, 60, 3000))
    val = rng.integers(0, 40, grp.size)
    key = grp * np.int64(40) + val
    want = np.lexsort((val, grp))
    assert np.array_equal(problems._argsort_stable(key, use_torch=False), want)
    assert np.array_equal(problems._argsort_stable(key, use_torch=True), want)
