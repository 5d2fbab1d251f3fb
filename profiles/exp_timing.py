"""Experiment (not a benchmark): iteration rate of config 1 under graph vs
eager launch and PDHG vs AA, to separate kernel time from launch overhead."""
import os
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

if len(sys.argv) > 1 and sys.argv[1] == "child":
    from paper_2508_08062_b200 import Method, Solver, SolverConfig, problems
    import numpy as np
    p = problems.make_config(1, scale=float(sys.argv[3]) if len(sys.argv) > 3 else 1.0)
    meth = Method[sys.argv[2]]
    with Solver(p) as s:
        tau = s.select_step_sizes(SolverConfig(reduction="tree")).tau
        cfg = SolverConfig(method=meth, m=10, toll=1e-6, max_iters=2000, tau=tau, sigma=tau,
                           reduction="tree")
        s.solve(SolverConfig(method=meth, m=10, toll=1e-6, max_iters=50, tau=tau, sigma=tau,
                             reduction="tree"))
        t0 = time.perf_counter()
        out = s.solve(cfg)
        dt = time.perf_counter() - t0
    print(f"eager={os.environ.get('AAPDHG_EAGER','0')} pdl={os.environ.get('AAPDHG_PDL','1')} {meth.name:9s} scale={sys.argv[3] if len(sys.argv)>3 else 1} "
          f"{out.result.iterations/dt:10.1f} it/s  {1e6*dt/out.result.iterations:8.1f} us/it  aa={out.result.i}")
    sys.exit(0)

# usage: exp_timing.py [eager,pdl ...]   e.g. 0,1 0,0 1,1
combos = sys.argv[1:] or ["0,1", "0,0", "1,1"]
for combo in combos:
    eager, pdl = combo.split(",")
    for meth in ("PDHG", "AA_PDHG"):
        for scale in ("1", "0.01"):
            env = dict(os.environ, AAPDHG_EAGER=eager, AAPDHG_PDL=pdl)
            subprocess.run([sys.executable, __file__, "child", meth, scale], env=env)
