"""The C-ABI library loads, exports every symbol include/aapdhg_cuda.h
declares, and its struct layouts match the ctypes mirror. No compute calls
(this runs on the CPU-only driver box too)."""
import ctypes as C
import re
import subprocess
import textwrap
from pathlib import Path

import numpy as np
import pytest

from paper_2508_08062_b200 import _abi

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "aapdhg_cuda.h"


def declared_functions():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(aapdhg_cuda_\w+)\s*\(", text)))


def test_header_matches_mirror():
    assert declared_functions() == sorted(_abi.CUDA_SYMBOLS)


def test_library_exports_every_symbol():
    if not _abi.CUDA_LIB.exists():
        pytest.fail(f"{_abi.CUDA_LIB} not built — run __graft_entry__.build()")
    out = subprocess.run(["nm", "-D", "--defined-only", str(_abi.CUDA_LIB)], check=True,
                         capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (aapdhg_cuda_\w+)", out))
    missing = set(declared_functions()) - exported
    assert not missing, missing


def test_library_loads_and_reports_abi():
    lib = _abi.cuda_lib()
    assert lib.aapdhg_cuda_abi_version() == _abi.ABI_VERSION


def test_struct_layouts_match_header(tmp_path):
    structs = {"aapdhg_csr_view": _abi.CsrView, "aapdhg_problem_view": _abi.ProblemView,
               "aapdhg_solve_params": _abi.SolveParams, "aapdhg_record": _abi.Record,
               "aapdhg_solve_result": _abi.SolveResultC}
    lines = []
    for cname, py in structs.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            lines.append(f'printf("{cname}.{fname} %zu\\n", offsetof({cname}, {fname}));')
    src = tmp_path / "layout.c"
    src.write_text(textwrap.dedent("""
        #include <stdio.h>
        #include <stddef.h>
        #include "aapdhg_cuda.h"
        int main(void) {
        """) + "\n".join(lines) + "\nreturn 0; }\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c11", "-I", str(ROOT / "include"), str(src), "-o", str(exe)],
                   check=True)
    got = dict(l.split() for l in subprocess.run([str(exe)], check=True, capture_output=True,
                                                 text=True).stdout.splitlines())
    for cname, py in structs.items():
        assert int(got[cname]) == C.sizeof(py), cname
        for fname, _ in py._fields_:
            assert int(got[f"{cname}.{fname}"]) == getattr(py, fname).offset, (cname, fname)


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU failure mode")
def test_no_gpu_fails_loudly():
    """No CPU fallback: without a device the product path raises CudaError."""
    from paper_2508_08062_b200 import CudaError, Solver, problems
    with pytest.raises(CudaError):
        Solver(problems.toy())


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    monkeypatch.setattr(_abi, "_cuda_lib", None)
    monkeypatch.setenv("AAPDHG_CUDA_LIB", str(tmp_path / "nope.so"))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _abi.cuda_lib()


def test_balance_partition_follows_the_sm_rates():
    """k_plain_loop's calibrated partition (engine.cu rebalance_partition, host
    only): from a proportional start and per-SM rates spread +-20%, the new
    slice starts cover every slice once, give no worker more than 8, share
    the work per SM in proportion to the rates (work = slice lengths), and
    cut the slowest SM's predicted time below the proportional partition's."""
    lib = _abi.cuda_lib()
    rng = np.random.default_rng(5)
    nsm, per_sm, ns = 148, 6, 6250
    workers = nsm * per_sm - 1                      # (the control CTA takes a slot)
    sm = np.array([w % nsm for w in range(workers)], dtype=np.int32)
    work = rng.integers(15, 26, ns).astype(np.int32)  # slice lengths
    cur = np.array([w * ns // workers for w in range(workers + 1)], dtype=np.int32)
    rate = rng.uniform(0.8, 1.2, nsm)                # work per ns, per SM

    def sm_time(starts):
        w_sm = np.zeros(nsm)
        for w in range(workers):
            w_sm[sm[w]] += work[starts[w]:starts[w + 1]].sum()
        return w_sm / rate, w_sm

    t0, _ = sm_time(cur)
    phase = np.array([t0[sm[w]] for w in range(workers)], dtype=np.float64)
    new = np.empty(workers + 1, dtype=np.int32)
    rc = lib.aapdhg_cuda_balance_partition(
        workers, ns, cur.ctypes.data_as(C.POINTER(C.c_int32)),
        phase.ctypes.data_as(C.POINTER(C.c_double)), sm.ctypes.data_as(C.POINTER(C.c_int32)),
        work.ctypes.data_as(C.POINTER(C.c_int32)), new.ctypes.data_as(C.POINTER(C.c_int32)))
    assert rc == 0
    assert new[0] == 0 and new[-1] == ns
    d = np.diff(new)
    assert d.min() >= 0 and d.max() <= 8
    t1, w_sm = sm_time(new)
    assert np.corrcoef(w_sm, rate)[0, 1] > 0.9
    assert t1.max() < 0.95 * t0.max()
