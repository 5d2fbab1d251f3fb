"""Short, deterministic workload for ncu captures: BASELINE configs[1]
(100k x 200k, 4M nnz), AA-PDHG m=10, explicit step size (no power
iteration), 40 iterations through the C-ABI. Not a benchmark."""
import os
import sys
from pathlib import Path

os.environ.setdefault("AAPDHG_EAGER", "1")  # ncu cannot see kernels of conditional graphs

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2508_08062_b200 import Method, Solver, SolverConfig, problems  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 40
p = problems.make_config(1)
with Solver(p) as s:
    out = s.solve(SolverConfig(method=Method.AA_PDHG, m=10, toll=1e-6, max_iters=iters,
                               tau=0.0775, sigma=0.0775, reduction="tree"))
print("iterations", out.result.iterations, "aa", out.result.i)
