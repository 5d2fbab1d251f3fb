"""The drop-in C++ API (include/aapdhg/*.hpp, lib/libaapdhg.so) used the way
a reference user would: reference known answers through solve()."""
import json
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
EXE = ROOT / "paper_2508_08062_b200" / "lib" / "dropin_check"


@pytest.mark.gpu
def test_cpp_dropin_end_to_end():
    assert EXE.exists(), "build first: __graft_entry__.build()"
    out = subprocess.run([str(EXE)], check=True, capture_output=True, text=True, timeout=600)
    r = json.loads(out.stdout.strip().splitlines()[-1])
    # proj/test_output.txt:21 — toy: PDHG 274 (RESIDUAL_TOL), AA-PDHG 47
    assert r["toy_pdhg_iterations"] == 274 and r["toy_pdhg_status"] == "RESIDUAL_TOL"
    assert r["toy_aa_iterations"] == 47
    assert r["toy_faa_iterations"] <= 100
    assert abs(float(r["toy_aa_x"]) - 3.0) < 1e-3
    assert r["mps_roundtrip_iterations"] == 274
    assert r["bookkeeping_ok"] and r["accel_records"] >= 2
    assert r["transport_nnz"] >= 3200 and float(r["transport_best_ratio"]) <= 0.1
    assert r["csv_rows"] == 48 + 1 and r["summary_has_status"]
    assert r["input_error_thrown"]
    assert r["sweep_ok"] and r["sweep_names"] == "D1_m2,D1_m5,D1e-300_m2,D1e-300_m5"


def test_dropin_library_exports_api():
    lib = ROOT / "paper_2508_08062_b200" / "lib" / "libaapdhg.so"
    if not lib.exists():
        pytest.fail("libaapdhg.so not built")
    syms = subprocess.run(["nm", "-DC", "--defined-only", str(lib)], check=True,
                          capture_output=True, text=True).stdout
    for name in ("aapdhg::solve(aapdhg::ProblemData const&, aapdhg::SolverConfig const&)",
                 "aapdhg::select_step_sizes(", "aapdhg::kkt_metrics(", "aapdhg::safeguard_pass(",
                 "aapdhg::pdhg_step(", "aapdhg::parse_mps(", "aapdhg::to_standard_form(",
                 "aapdhg::trajectory_csv", "aapdhg::summary_json", "aapdhg::solve_sweep",
                 "aapdhg::sweep_cases"):
        assert name in syms, name


@pytest.mark.gpu
def test_mps_front_end_round_trip_10m_nonzeros(tmp_path):
    """f3 at scale: a 500k x 1M LP with 10^7 nonzeros (E / G / L rows, every
    bound type) written with emit_mps, read back by the mmap + threaded
    parse_mps_file and assembled by to_standard_form on the device: the
    four-block form must come back bit for bit (lib/mps_check)."""
    exe = ROOT / "paper_2508_08062_b200" / "lib" / "mps_check"
    assert exe.exists(), "build first: __graft_entry__.build()"
    out = subprocess.run([str(exe), "500000", "1000000", "10", "7", str(tmp_path / "rt.mps")],
                         capture_output=True, text=True, timeout=900)
    r = json.loads(out.stdout.strip().splitlines()[-1])
    assert out.returncode == 0 and r["identical"], out.stdout + out.stderr
    assert r["nnz"] == 10_000_000


@pytest.mark.gpu
def test_from_triplets_on_device_matches_definition():
    """SparseMatrix::from_triplets semantics on the device entry
    (aapdhg_cuda_csr_from_triplets): sorted (row, col), duplicates summed
    left to right in input order, cancellations kept, ranges checked, and the
    standard-form row map / negation."""
    import ctypes as C

    import numpy as np

    from paper_2508_08062_b200 import _abi
    lib = _abi.cuda_lib()
    rng = np.random.default_rng(5)
    cnt, nr, nc = 200_000, 3_000, 2_000
    trip = np.zeros(cnt, dtype=[("row", "<i4"), ("col", "<i4"), ("val", "<f8")])
    trip["row"] = rng.integers(0, nr, cnt)
    trip["col"] = rng.integers(0, nc, cnt)  # many duplicates
    trip["val"] = rng.standard_normal(cnt)
    rmap = rng.permutation(nr).astype(np.int32)
    neg = (rng.random(nr) < 0.3).astype(np.uint8)
    rp = np.zeros(nr + 1, dtype=np.int32)
    ci = np.zeros(cnt, dtype=np.int32)
    va = np.zeros(cnt)
    nnz = C.c_int64()
    err = C.create_string_buffer(512)
    rc = lib.aapdhg_cuda_csr_from_triplets(0, nr, nr, nc, cnt, trip.ctypes.data,
                                           _abi.iptr(rmap), neg.ctypes.data, _abi.iptr(rp),
                                           _abi.iptr(ci), _abi.dptr(va), C.byref(nnz), err, 512)
    assert rc == 0, err.value
    # the definition, in numpy: stable order of (mapped row, col), left-to-right sums
    r2 = rmap[trip["row"]]
    v2 = np.where(neg[trip["row"]] == 1, -trip["val"], trip["val"])
    order = np.lexsort((trip["col"], r2))  # stable
    key = r2[order].astype(np.int64) * nc + trip["col"][order]
    heads = np.flatnonzero(np.r_[True, key[1:] != key[:-1]])
    sums = np.empty(heads.size)
    for t, h in enumerate(heads):
        e = heads[t + 1] if t + 1 < heads.size else key.size
        acc = 0.0
        for x in v2[order][h:e]:
            acc += x
        sums[t] = acc
    assert nnz.value == heads.size
    assert np.array_equal(ci[: nnz.value], (key[heads] % nc).astype(np.int32))
    assert np.array_equal(va[: nnz.value], sums)
    assert np.array_equal(rp, np.r_[0, np.cumsum(np.bincount(key[heads] // nc, minlength=nr))])
    bad = trip.copy()
    bad["col"][7] = nc
    rc = lib.aapdhg_cuda_csr_from_triplets(0, nr, nr, nc, cnt, bad.ctypes.data, None, None,
                                           _abi.iptr(rp), _abi.iptr(ci), _abi.dptr(va),
                                           C.byref(nnz), err, 512)
    assert rc == 2  # AAPDHG_ERR_DIMENSION
