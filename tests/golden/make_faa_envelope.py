"""The reference's own iteration-count envelope on the FAA golden solves
(test infrastructure): the unmodified reference built three ways
(oracle/Makefile `ref` + `variants`: strict, FMA-contracted, reassociated
sums) solves each FAA case of golden.json; FAA-PDHG is chaotic under
rounding, so a count is judged against this spread,
and so are the first 50 iterates (g_norm_spread_50: the largest relative
g_norm difference of a variant from the strict build).
    python tests/golden/make_faa_envelope.py  ->  tests/golden/faa_envelope.json"""
import json
import sys

import numpy as np
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE.parents[1]))

from golden_io import config_for, golden, problem  # noqa: E402
from oracle.pyoracle import Oracle  # noqa: E402
from paper_2508_08062_b200 import Method  # noqa: E402

out = {}
for case in golden()["solves"]:
    if Method(case["config"]["method"]) != Method.FAA_PDHG:
        continue
    p = problem(case["problem"])
    cfg = config_for(case, "serial")
    runs = {k: Oracle(k).solve(p, cfg) for k in ("ref", "ref-fast", "ref-assoc")}
    counts = {k: r.result.iterations for k, r in runs.items()}
    # the first 50 iterates of the variants against the strict build
    g0 = runs["ref"].trajectory["g_norm"][:50]
    spread = max(float(np.max(np.abs(r.trajectory["g_norm"][:len(g0)] - g0) / np.abs(g0)))
                 for r in runs.values())
    out[case["name"]] = dict(counts, g_norm_spread_50=spread)
    print(case["name"], out[case["name"]])
(HERE / "faa_envelope.json").write_text(json.dumps(out, indent=1))
