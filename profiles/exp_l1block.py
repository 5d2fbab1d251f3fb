"""Experiment (not a benchmark): does column blocking sized for L1 (the L2
blocking mechanism, build_blocks, with small blocks) raise the gather hit
rate enough to pay for the extra passes on configs[1]? Per-kernel graph
(AAPDHG_PERSIST=0) with and without blocks; PDHG, 2,000 iterations."""
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
        cfg = SolverConfig(method=Method.PDHG, toll=1e-12, max_iters=2000, tau=0.0775,
                           sigma=0.0775, reduction="tree")
        s.solve(cfg)
        t = time.perf_counter()
        o = s.solve(cfg)
        dt = time.perf_counter() - t
    print(f"block_kb={os.environ.get('AAPDHG_L2_BLOCK_KB', 'off'):>6}  "
          f"{1e6 * dt / o.result.iterations:7.2f} us/it  |g| {o.result.g_norm:.6e}", flush=True)
    sys.exit(0)
for kb in ["off", "800", "400", "200", "100"]:
    env = dict(os.environ, AAPDHG_PERSIST="0")
    if kb != "off":
        env.update(AAPDHG_L2_BLOCK_KB=kb, AAPDHG_L2_BLOCK_MIN_KB="0")
    subprocess.run([sys.executable, __file__, "child"], env=env)
