"""Experiment (not a benchmark): config-1 PDHG iteration time across the
SpMV layout knobs (AAPDHG_SF = lanes per row, AAPDHG_SPMV_WARPS = warps per
CTA)."""
import os
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

if len(sys.argv) > 1 and sys.argv[1] == "child":
    from paper_2508_08062_b200 import Method, Solver, SolverConfig, problems
    p = problems.make_config(1)
    with Solver(p) as s:
        cfg = SolverConfig(method=Method[sys.argv[2]], m=10, toll=1e-6, max_iters=1500,
                           tau=0.0775, sigma=0.0775, reduction="tree")
        s.solve(SolverConfig(method=Method.PDHG, max_iters=20, tau=0.0775, sigma=0.0775,
                             reduction="tree"))
        t0 = time.perf_counter()
        out = s.solve(cfg)
        dt = time.perf_counter() - t0
    print(f"sf={os.environ.get('AAPDHG_SF')} warps={os.environ.get('AAPDHG_SPMV_WARPS')} "
          f"{sys.argv[2]:8s} {1e6 * dt / out.result.iterations:7.1f} us/it", flush=True)
    sys.exit(0)

for sf in ("1", "2", "4"):
    for w in ("2", "4", "8"):
        env = dict(os.environ, AAPDHG_SF=sf, AAPDHG_SPMV_WARPS=w)
        subprocess.run([sys.executable, __file__, "child", "PDHG"], env=env)
