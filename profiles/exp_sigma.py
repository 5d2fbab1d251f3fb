"""Experiment (not a benchmark): SELL-sigma window of the TREE layout
(AAPDHG_SIGMA, rows sorted by length inside windows of sigma rows) against
the persistent plain-step time on configs[1], PDHG and AA-PDHG m=10,
3000 iterations, explicit step size."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2508_08062_b200 import Method, Solver, SolverConfig, problems  # noqa: E402

p = problems.make_config(int(os.environ.get("CFG", "1")))
for sigma in sys.argv[1:] or ["1", "128", "512", "2048", "100000"]:
    os.environ["AAPDHG_SIGMA"] = sigma
    with Solver(p) as s:
        for meth in (Method.PDHG, Method.AA_PDHG):
            cfg = SolverConfig(method=meth, m=10, toll=1e-12, max_iters=3000, tau=0.0775,
                               sigma=0.0775, reduction="tree")
            s.solve(cfg)
            t = time.perf_counter()
            o = s.solve(cfg)
            dt = time.perf_counter() - t
            print(f"sigma {sigma:>7s} {meth.name:8s} {1e6 * dt / o.result.iterations:7.2f} us/it",
                  flush=True)
