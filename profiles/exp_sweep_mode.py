"""Experiment: sweep-mode throughput on a small LP (configs[0], SERIAL, full
solves to 1e-6): the same 8 cases on 1 worker vs 8 concurrent workers (one
resident handle and stream each) on one GPU."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2508_08062_b200 import Method, SolverConfig, problems, solve_sweep, sweep_cases  # noqa

p = problems.make_config(0)
base = SolverConfig(method=Method.AA_PDHG, m=5, toll=1e-6, max_iters=200000)
cases = sweep_cases(base, d=[1.0, 0.1], eps=[1.0, 0.5], m=[5, 10])
for w in (1, 8):
    t0 = time.perf_counter()
    out = solve_sweep(p, cases, workers=w)
    dt = time.perf_counter() - t0
    its = sum(o[2].result.iterations for o in out if o[0])
    print(f"workers={w} cases={len(cases)} wall={dt:.2f}s iterations={its} "
          f"aggregate={its / dt:,.0f} it/s ok={all(o[0] for o in out)}", flush=True)
