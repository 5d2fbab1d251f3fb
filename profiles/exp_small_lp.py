"""Small-LP path (BASELINE config 0: 1,000 x 2,000, AA-PDHG m=5, toll 1e-6):
SERIAL (bit-identical to the reference) through the persistent plain-step
grid (the control CTA runs the index-ordered chains) against the per-kernel
graph (AAPDHG_SERIAL_PERSIST=0), and TREE for comparison. One JSON line per
arm: iterations, status, time, microseconds per iteration.
  python profiles/exp_small_lp.py"""
import json
import os
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def arm(name, reduction, env):
    code = f"""
import json, sys, time
sys.path.insert(0, {str(ROOT)!r})
from paper_2508_08062_b200 import Method, Solver, SolverConfig, problems
p = problems.make_config(0)
cfg = SolverConfig(method=Method.AA_PDHG, m=5, toll=1e-6, max_iters=400000, reduction={reduction!r})
with Solver(p) as s:
    s.solve(SolverConfig(method=Method.AA_PDHG, m=5, toll=1e-6, max_iters=50, reduction={reduction!r}))
    t0 = time.perf_counter()
    r = s.solve(cfg)
    dt = time.perf_counter() - t0
g = r.trajectory["g_norm"]
print(json.dumps({{"arm": {name!r}, "iterations": r.result.iterations, "aa_steps": r.result.i,
                  "status": r.result.status.name, "seconds": dt,
                  "us_per_iteration": 1e6 * dt / r.result.iterations,
                  "objective": r.result.objective.hex(), "g_last": float(g[-1]).hex()}}))
"""
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         env=dict(os.environ, **env))
    print(out.stdout.strip() or out.stderr[-2000:], flush=True)


arm("serial-persist", "serial", {"AAPDHG_SERIAL_PERSIST": "1"})
arm("serial-per-kernel", "serial", {"AAPDHG_SERIAL_PERSIST": "0"})
arm("tree-persist", "tree", {})
