"""summary_json / trajectory_csv of the drop-in (host/report.cpp) against
the reference's own report.cpp (proj/src/report.cpp:18-104, built with its
nlohmann::ordered_json dependency from the venv's copy), byte for byte, on
18 results whose numbers cover the shortest-round-trip formats (1.0, 0.9,
1e-06, 0.0001, 1e+16, -0.0, NaN -> null ...), d_hat arrays and string
escapes (tests/reftests/summary_main.cpp; built by `make -C oracle reftests`
when /root/reference is present)."""
import subprocess
from pathlib import Path

import pytest

BIN = Path(__file__).resolve().parents[1] / "oracle" / "_ref" / "reftests"


def test_summary_json_and_csv_bytes_match_reference():
    ref, ours = BIN / "summary_ref", BIN / "summary_dropin"
    if not ref.exists() or not ours.exists():
        pytest.skip("summary_ref / summary_dropin not built (needs /root/reference at build time)")
    a = subprocess.run([str(ref)], capture_output=True, check=True, timeout=60).stdout
    b = subprocess.run([str(ours)], capture_output=True, check=True, timeout=60).stdout
    assert a == b
    assert b.count(b'"config": {') == 18 and b"null" in b and b'"D": 1.0' in b
