"""The drop-in's MPS reader (paper_2508_08062_b200/host/mps.cpp: mmap +
threaded COLUMNS tokenising) on CPU, through `lib/mps_check parse` (host
only). Each file is also read by the small one-pass reader below (test
infrastructure); the two must agree on every field `mps_check` reports.
Files large enough to be cut into several COLUMNS chunks (> 65,536 lines
per thread) check that the threaded reader keeps file order: columns in
order of first appearance (a column may reappear later), entries in file
order, objective coefficients summed in file order, integer markers."""
import json
import math
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
EXE = ROOT / "paper_2508_08062_b200" / "lib" / "mps_check"


def run_parse(path):
    if not EXE.exists():
        pytest.skip("lib/mps_check not built")
    out = subprocess.run([str(EXE), "parse", str(path)], capture_output=True, text=True,
                         timeout=300)
    return json.loads(out.stdout.strip().splitlines()[-1])


def reference_read(text):
    """One-pass reader of the same MPS subset (for the comparison only)."""
    name, obj, maximize, sense_next = "", "", False, False
    rows, senses, rhs, cols, colidx = {}, [], [], [], {}
    objc, lower, upper, integer = [], [], [], []
    entries = []
    sec, in_int = None, False
    for raw in text.splitlines():
        line = raw.rstrip("\r")
        if not line.strip() or line.startswith("*"):
            continue
        f = line.split()
        if not line[0].isspace():
            sense_next = False
            if f[0] == "NAME":
                name = f[1] if len(f) > 1 else ""
            elif f[0] == "OBJSENSE":
                if len(f) > 1:
                    maximize = f[1] in ("MAX", "MAXIMIZE")
                else:
                    sense_next = True
            elif f[0] == "ENDATA":
                break
            else:
                sec = f[0]
            continue
        if sense_next:
            maximize = f[0] in ("MAX", "MAXIMIZE")
            sense_next = False
            continue
        if sec == "ROWS":
            if f[0] == "N":
                obj = obj or f[1]
            else:
                rows[f[1]] = len(senses)
                senses.append(f[0])
                rhs.append(0.0)
        elif sec == "COLUMNS":
            if len(f) >= 3 and f[1] == "'MARKER'":
                in_int = f[2] == "'INTORG'"
                continue
            if f[0] not in colidx:
                colidx[f[0]] = len(cols)
                cols.append(f[0])
                objc.append(0.0)
                lower.append(0.0)
                upper.append(math.inf)
                integer.append(False)
            c = colidx[f[0]]
            integer[c] = integer[c] or in_int
            for k in range(1, len(f) - 1, 2):
                v = float(f[k + 1])
                if f[k] == obj:
                    objc[c] += v
                else:
                    entries.append((rows[f[k]], c, v))
        elif sec == "RHS":
            for k in range(1, len(f) - 1, 2):
                if f[k] != obj:
                    rhs[rows[f[k]]] = float(f[k + 1])
        elif sec == "BOUNDS":
            c = colidx[f[2]]
            v = float(f[3]) if len(f) > 3 else 0.0
            if f[0] in ("UP", "UI"):
                upper[c] = v
            elif f[0] in ("LO", "LI"):
                lower[c] = v
            elif f[0] == "FX":
                lower[c] = upper[c] = v
            elif f[0] == "FR":
                lower[c], upper[c] = -math.inf, math.inf
            elif f[0] == "MI":
                lower[c] = -math.inf
            elif f[0] == "PL":
                upper[c] = math.inf
            elif f[0] == "BV":
                lower[c], upper[c] = 0.0, 1.0

    def fsum(vals):  # left-to-right double sums, as mps_check prints them
        s = 0.0
        for v in vals:
            s += v
        return s

    return {"name": name, "objective": obj, "maximize": maximize, "rows": len(senses),
            "cols": len(cols), "entries": len(entries), "senses": "".join(senses),
            "obj_sum": fsum(objc), "entry_sum": fsum(e[2] for e in entries),
            "rhs_sum": fsum(rhs), "row_index_sum": sum(e[0] for e in entries),
            "col_index_sum": sum(e[1] for e in entries), "integer": sum(integer),
            "inf_lower": sum(math.isinf(v) for v in lower),
            "inf_upper": sum(math.isinf(v) for v in upper),
            "first_col": cols[0] if cols else "", "last_col": cols[-1] if cols else ""}


SMALL = """* a comment before NAME
NAME   MIXED
OBJSENSE
    MAX
ROWS
 N  PROFIT
 N  FREEROW
 L  CAP1
 G  DEM1
 E  BAL1
COLUMNS
    MARKER                 'MARKER'                 'INTORG'
    A      PROFIT   3.5   CAP1   1.0
    A      DEM1     2.0
    MARKER                 'MARKER'                 'INTEND'
* a comment inside COLUMNS
    B      CAP1    -1.25   BAL1   4e-1
    C      PROFIT  +2      DEM1    9.0
    B      PROFIT   0.5
RHS
    RHS    CAP1     10     PROFIT 7.0
    RHS    BAL1     -3.5
BOUNDS
 UP BND A 4
 MI BND B
 FX BND C 1.5
 BV BND A
ENDATA
"""


def test_small_file_every_record_kind(tmp_path):
    f = tmp_path / "small.mps"
    f.write_text(SMALL.replace("\n", "\r\n"))  # CRLF line ends
    got = run_parse(f)
    assert got == reference_read(SMALL)
    assert got["maximize"] and got["integer"] == 1 and got["senses"] == "LGE"


@pytest.mark.parametrize("ncols,per,seed", [(60_000, 4, 1), (150_000, 3, 2)])
def test_large_file_threaded_chunks_keep_file_order(tmp_path, ncols, per, seed):
    rng = np.random.default_rng(seed)
    m = 5_000
    lines = ["NAME BIG", "ROWS", " N COST"]
    lines += [f" {'EGL'[r % 3]} R{r}" for r in range(m)]
    lines.append("COLUMNS")
    order = list(range(ncols))
    # a few columns reappear later (their index is the first appearance's)
    extra = rng.choice(ncols, size=ncols // 50, replace=False)
    for j in order:
        rows_j = rng.choice(m, size=per, replace=False)
        vals = rng.standard_normal(per)
        lines.append(f"    X{j} COST {rng.standard_normal():.17g}")
        for r, v in zip(rows_j, vals):
            lines.append(f"    X{j} R{r} {v:.17g}")
        if j % 20_000 == 0:
            lines.append("    M 'MARKER' 'INTORG'" if (j // 20_000) % 2 == 0
                         else "    M 'MARKER' 'INTEND'")
    for j in extra:
        lines.append(f"    X{j} COST {rng.standard_normal():.17g} R{int(rng.integers(m))} 1.5")
    lines += ["RHS", "    RHS R0 1.0 R1 -2.0", "BOUNDS", f" FR BND X{ncols - 1}", "ENDATA"]
    text = "\n".join(lines) + "\n"
    f = tmp_path / "big.mps"
    f.write_text(text)
    got = run_parse(f)
    want = reference_read(text)
    assert got == want
    assert got["entries"] > 65_536  # several chunks


@pytest.mark.parametrize("text,kind", [
    ("NAME X\nROWS\n N OBJ\nCOLUMNS\n X OBJ 1.0 NOPE 2.0\nENDATA\n", "InputError"),
    ("NAME X\nROWS\n G R1\nCOLUMNS\n X R1 1.0\nENDATA\n", "InputError"),
    ("NAME X\nCOLUMNS\n X OBJ 1.0\nENDATA\n", "InputError"),
    (" X OBJ 1.0\n", "InputError"),
    ("NAME X\nROWS\n Z R1\nENDATA\n", "InputError"),
    ("NAME X\nROWS\n N OBJ\n G R1\n G R1\nENDATA\n", "InputError"),
    ("NAME X\nROWS\n N OBJ\nCOLUMNS\n X OBJ 1.0\nBOUNDS\n UP BND X\nENDATA\n", "InputError"),
    ("NAME X\nROWS\n N OBJ\nCOLUMNS\n X OBJ 1.0x\nENDATA\n", "InputError"),
    ("NAME R\nROWS\n N C\n G R1\nCOLUMNS\n X C 1.0 R1 1.0\nRANGES\n RNG R1 4.0\nENDATA\n",
     "UnsupportedError"),
])
def test_malformed_inputs(tmp_path, text, kind):
    f = tmp_path / "bad.mps"
    f.write_text(text)
    got = run_parse(f)
    assert got.get("error") == kind, got


def test_error_in_a_later_chunk_is_reported_with_its_line(tmp_path):
    lines = ["NAME E", "ROWS", " N OBJ", " E R0", "COLUMNS"]
    lines += [f" X{j} R0 1.0" for j in range(200_000)]
    bad = len(lines) + 1
    lines.append(" XBAD UNDECLARED 1.0")
    lines += [f" Y{j} R0 1.0" for j in range(10)]
    lines.append("ENDATA")
    f = tmp_path / "late.mps"
    f.write_text("\n".join(lines) + "\n")
    got = run_parse(f)
    assert got["error"] == "InputError" and f"line {bad}:" in got["what"]
