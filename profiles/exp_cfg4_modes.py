"""Experiment (not a benchmark): config 4 per-iteration wall time in graph
mode against eager stream launches (AAPDHG_EAGER=1), 100 and 200 iterations
(the difference removes the fixed cost of a solve call)."""
import os
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, str(ROOT))
    from paper_2508_08062_b200 import Method, Solver, SolverConfig, problems
    p = problems.make_config(4)
    with Solver(p) as s:
        t = {}
        for it in (100, 200):
            cfg = SolverConfig(method=Method.AA_PDHG, m=10, toll=1e-12, max_iters=it, tau=0.0905,
                               sigma=0.0905, reduction="tree")
            if it == 100:
                s.solve(cfg)
            t0 = time.perf_counter()
            o = s.solve(cfg)
            t[it] = time.perf_counter() - t0
            print(f"EAGER={os.environ.get('AAPDHG_EAGER', '0')} {it} its {t[it]:.3f} s "
                  f"({o.result.i} AA steps)", flush=True)
        print(f"EAGER={os.environ.get('AAPDHG_EAGER', '0')} marginal "
              f"{1e3 * (t[200] - t[100]) / 100:.2f} ms/iteration", flush=True)
    sys.exit(0)
for eager in ("0", "1"):
    subprocess.run([sys.executable, __file__, "child"], env=dict(os.environ, AAPDHG_EAGER=eager))
