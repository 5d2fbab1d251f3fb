"""Experiment (not a benchmark): configs[4] plain PDHG iteration time in graph
mode under L2 settings: column-block size (AAPDHG_L2_BLOCK_KB) and the
persisting set-aside with evict_last gathers (AAPDHG_L2_PERSIST=1).
Marginal ms per iteration = (t(N2) - t(N1)) / (N2 - N1)."""
import os
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, str(ROOT))
    from paper_2508_08062_b200 import Method, Solver, SolverConfig, problems
    p = problems.cached_config(4)
    t0 = time.perf_counter()
    with Solver(p) as s:
        create = time.perf_counter() - t0
        t = {}
        for it in (5, 10, 40):
            cfg = SolverConfig(method=Method.PDHG, toll=1e-12, max_iters=it, tau=0.0905,
                               sigma=0.0905, reduction="tree")
            t0 = time.perf_counter()
            s.solve(cfg)
            t[it] = time.perf_counter() - t0
        tag = " ".join(f"{k}={os.environ.get(k, '-')}" for k in (
            "AAPDHG_L2_BLOCK_KB", "AAPDHG_L2_BLOCK_MIN_KB", "AAPDHG_L2_PERSIST",
            "AAPDHG_SPLIT_EPI"))
        print(f"{tag}: create {create:.2f} s, marginal PDHG "
              f"{1e3 * (t[40] - t[10]) / 30:.2f} ms/iteration", flush=True)
    sys.exit(0)
# KB[,PERSIST[,MIN_KB]]: MIN_KB = the vector size blocking starts above (the
# default 64 MB blocks both y (156,250 KB) and x (312,500 KB); 200000 leaves
# K'y unblocked)
combos = [a.split(",") for a in (sys.argv[1:] or ["65536,0", "65536,1", "81920,0", "81920,1"])]
for c in combos:
    kb, persist, mn = (c + ["0", "65536"])[:3] if len(c) == 1 else (c + ["65536"])[:3]
    subprocess.run([sys.executable, __file__, "child"],
                   env=dict(os.environ, AAPDHG_L2_BLOCK_KB=kb, AAPDHG_L2_PERSIST=persist,
                            AAPDHG_L2_BLOCK_MIN_KB=mn))
