"""Experiment (not a benchmark): k_plain_loop with the calibrated per-SM
partition (AAPDHG_BALANCE=1, per-slice partials) against the proportional
per-CTA partition (AAPDHG_BALANCE=0) on configs[1]: microseconds per
iteration over 3,000 PDHG / AA-PDHG iterations and the 20-iteration solve the
driver's bench times; with balancing, the trajectory before calibration (the
first solve of the process, proportional partition) must equal the one after
it bit for bit (the partials are per slice)."""
import os
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, str(ROOT))
    import numpy as np
    from paper_2508_08062_b200 import Method, Solver, SolverConfig, problems
    p = problems.make_config(1)
    tag = f"BALANCE={os.environ.get('AAPDHG_BALANCE', '1')}"
    with Solver(p) as s:
        tau = 0.0775
        def cfg(meth, it):
            return SolverConfig(method=meth, m=10, toll=1e-12, max_iters=it, tau=tau, sigma=tau,
                                reduction="tree")
        first = s.solve(cfg(Method.AA_PDHG, 300))
        for _ in range(3):
            s.solve(cfg(Method.PDHG, 300))
        again = s.solve(cfg(Method.AA_PDHG, 300))
        same = (np.array_equal(first.trajectory["g_norm"], again.trajectory["g_norm"]) and
                np.array_equal(first.result.u.x, again.result.u.x))
        print(f"{tag}: trajectory before / after calibration bitwise equal: {same}", flush=True)
        for meth in (Method.PDHG, Method.AA_PDHG):
            t0 = time.perf_counter()
            o = s.solve(cfg(meth, 3000))
            dt = time.perf_counter() - t0
            print(f"{tag}: {meth.name} 3000 iterations {1e6 * dt / 3000:.2f} us/iteration "
                  f"({o.result.i} AA steps)", flush=True)
        ts = []
        for _ in range(10):
            t0 = time.perf_counter()
            s.solve(cfg(Method.AA_PDHG, 20))
            ts.append(time.perf_counter() - t0)
        print(f"{tag}: 20-iteration AA-PDHG solve median {1e3 * sorted(ts)[5]:.3f} ms "
              f"({20 / sorted(ts)[5]:.0f} it/s)", flush=True)
    sys.exit(0)
for bal in (sys.argv[1:] or ["0", "1"]):
    subprocess.run([sys.executable, __file__, "child"], env=dict(os.environ, AAPDHG_BALANCE=bal))
