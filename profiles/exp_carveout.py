"""Experiment (not a benchmark): L1 / shared-memory carveout of the gather
kernels (AAPDHG_CARVEOUT = percent of the maximum shared memory, -1 = driver
default) against the persistent plain-step time on configs[1]."""
import os
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, str(ROOT))
    from paper_2508_08062_b200 import Method, Solver, SolverConfig, problems
    p = problems.make_config(1)
    with Solver(p) as s:
        for meth in (Method.PDHG, Method.AA_PDHG):
            cfg = SolverConfig(method=meth, m=10, toll=1e-12, max_iters=3000, tau=0.0775,
                               sigma=0.0775, reduction="tree")
            s.solve(cfg)
            t = time.perf_counter()
            o = s.solve(cfg)
            dt = time.perf_counter() - t
            import ctypes as C
            pi, ps, pl = C.c_uint64(), C.c_double(), C.c_uint64()
            s.lib.aapdhg_cuda_last_plain_loop(s.h, C.byref(pi), C.byref(ps), C.byref(pl))
            print(f"carveout {os.environ.get('AAPDHG_CARVEOUT')} {meth.name:8s} "
                  f"{1e6 * dt / o.result.iterations:7.2f} us/it  final |g| "
                  f"{o.result.g_norm:.6e}  persistent launches {pl.value}", flush=True)
    sys.exit(0)
for c in sys.argv[1:] or ["-1", "0", "5", "10", "14", "20", "28"]:
    subprocess.run([sys.executable, __file__, "child"], env=dict(os.environ, AAPDHG_CARVEOUT=c))
