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
