"""The reference's OWN test files, unmodified (proj/tests/test_solver.cpp,
test_pdhg_core.cpp, test_lp_model.cpp), compiled against the B200 drop-in
headers (include/aapdhg/) and linked to the drop-in library
(paper_2508_08062_b200/lib/libaapdhg.so -> the sm_100a C-ABI), with a
minimal doctest stand-in (tests/reftests/doctest.h). Built by
`make -C oracle reftests` when /root/reference is present (the binaries
travel to the GPU box in oracle/_ref/reftests)."""
import os
import re
import subprocess
from pathlib import Path

import pytest

BIN = Path(__file__).resolve().parents[1] / "oracle" / "_ref" / "reftests"


def run_suite(name, skip=""):
    exe = BIN / name
    if not exe.exists():
        pytest.skip(f"{exe} not built (needs /root/reference at build time)")
    env = dict(os.environ, DOCTEST_SKIP=skip)
    r = subprocess.run([str(exe)], capture_output=True, text=True, env=env, timeout=600)
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed \| (\d+) skipped",
                  r.stdout)
    assert m, r.stdout + r.stderr
    total, passed, failed, skipped = map(int, m.groups())
    assert r.returncode == 0 and failed == 0, r.stderr[-3000:]
    return total, passed, skipped


@pytest.mark.gpu
def test_reference_solver_suite_passes_on_dropin():
    total, passed, skipped = run_suite("test_solver")
    assert total == 23 and passed == 23 and skipped == 0


@pytest.mark.gpu
def test_reference_pdhg_core_suite_passes_on_dropin():
    total, passed, skipped = run_suite("test_pdhg_core")
    assert passed == total and skipped == 0


@pytest.mark.gpu
def test_reference_lp_model_suite_passes_on_dropin():
    # the one case that reads proj/data/toy.mps needs the reference checkout
    data = Path("/root/reference/proj/data/toy.mps").exists()
    total, passed, skipped = run_suite("test_lp_model", skip="" if data else "toy instance parses")
    assert passed == total - skipped and skipped <= 1
