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
