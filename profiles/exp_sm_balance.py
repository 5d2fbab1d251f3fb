"""Experiment (not a benchmark): is the k_plain_loop barrier wait a per-SM
property? Per worker CTA K1 / K2 phase averages (globaltimer stamps of an
EXTRA=-DAAPDHG_PLAIN_STAMPS build) grouped by SM, over two separate solves:
if the slow SMs of solve A are the slow SMs of solve B, a static per-SM
share of the slices can remove the wait."""
import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2508_08062_b200 import Method, Solver, SolverConfig, problems  # noqa: E402

p = problems.make_config(1)
res = []
with Solver(p) as s:
    cfg = SolverConfig(method=Method.PDHG, toll=1e-12, max_iters=3000, tau=0.0775, sigma=0.0775,
                       reduction="tree")
    buf = (C.c_double * 4096)()
    s.solve(cfg)
    s.lib.aapdhg_cuda_plain_stamps_cta(buf)
    for rep in range(2):
        s.solve(cfg)
        s.lib.aapdhg_cuda_plain_stamps_cta(buf)
        a = np.frombuffer(buf, dtype=np.float64).reshape(1024, 4).copy()
        res.append(a)
for rep, a in enumerate(res):
    live = a[:, 2] > 0
    k1 = a[live, 0] / a[live, 2] / 1e3
    k2 = a[live, 1] / a[live, 2] / 1e3
    sm = a[live, 3].astype(int)
    print(f"solve {rep}: {live.sum()} CTAs; K1 mean {k1.mean():.2f} us p99 {np.percentile(k1, 99):.2f}"
          f" max {k1.max():.2f}; K2 mean {k2.mean():.2f} p99 {np.percentile(k2, 99):.2f} max {k2.max():.2f}")
    per_sm1 = np.array([k1[sm == q].mean() if (sm == q).any() else np.nan for q in range(148)])
    per_sm2 = np.array([k2[sm == q].mean() if (sm == q).any() else np.nan for q in range(148)])
    print("  per-SM K1 mean: min %.2f max %.2f; K2 min %.2f max %.2f" % (
        np.nanmin(per_sm1), np.nanmax(per_sm1), np.nanmin(per_sm2), np.nanmax(per_sm2)))
    res[rep] = (per_sm1, per_sm2, sm, k1, k2)
(a1, a2, sma, k1a, k2a), (b1, b2, smb, k1b, k2b) = res
print("per-SM correlation across solves: K1 %.3f K2 %.3f" % (
    np.corrcoef(a1, b1)[0, 1], np.corrcoef(a2, b2)[0, 1]))
print("same CTA->SM map across solves:", bool((sma == smb).all()))
print(json.dumps({"per_sm_k1": [round(v, 2) for v in a1], "per_sm_k2": [round(v, 2) for v in a2]}))
print(json.dumps({"cta_sm": [int(v) for v in sma], "cta_k1": [round(v, 3) for v in k1a],
                  "cta_k2": [round(v, 3) for v in k2a]}))
