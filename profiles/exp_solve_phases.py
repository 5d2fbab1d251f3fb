"""Where a short configs[1] solve spends its time (the driver's bench runs
20 iterations): AAPDHG_TIMING=1 phase stamps from engine.cu on stderr, plus
the Python-side wall time of the same calls.
  python profiles/exp_solve_phases.py [iters] [reps]"""
import os
import sys
import time
from pathlib import Path

os.environ.setdefault("AAPDHG_TIMING", "1")
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

from paper_2508_08062_b200 import Method, Solver, SolverConfig, problems  # noqa: E402


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    iters = int(args[0]) if len(args) > 0 else 20
    reps = int(args[1]) if len(args) > 1 else 3
    p = problems.make_config(1)
    n, m = p.n(), p.k.nrows
    import torch
    outs = tuple(torch.empty(k, dtype=torch.float64, pin_memory=True).numpy() for k in (n, m, n))
    with Solver(p) as s:
        tau = s.select_step_sizes(SolverConfig(reduction="tree")).tau
        cfg = SolverConfig(method=Method.AA_PDHG, m=10, toll=1e-6, max_iters=iters, tau=tau,
                           sigma=tau)
        s.solve(cfg, out=outs)
        for r in range(reps):
            print(f"--- rep {r}", file=sys.stderr, flush=True)
            t0 = time.perf_counter()
            out = s.solve(cfg, out=outs)
            dt = time.perf_counter() - t0
            print(f"python wall {1e6 * dt:.1f} us, {out.result.iterations} it, "
                  f"{out.result.i} aa, {iters / dt:.0f} it/s", file=sys.stderr, flush=True)
    if "--pinned" in sys.argv:  # the bench's e2e: the LP in page-locked buffers
        sys.path.insert(0, str(ROOT))
        import bench
        p, _ = bench.pinned_problem(torch, p)
    for r in range(reps):
        t0 = time.perf_counter()
        with Solver(p) as s2:
            t1 = time.perf_counter()
            s2.solve(cfg, out=outs)
            t2 = time.perf_counter()
        print(f"e2e create {1e6 * (t1 - t0):.0f} us solve {1e6 * (t2 - t1):.0f} us "
              f"destroy {1e6 * (time.perf_counter() - t2):.0f} us", file=sys.stderr, flush=True)


if __name__ == "__main__":
    main()
