"""Short, deterministic workload for ncu captures of another config:
profile_cfg.py CFG SCALE ITERS (AA/FAA as the config says, explicit tau,
eager launches). Not a benchmark."""
import os
import sys
from pathlib import Path

os.environ.setdefault("AAPDHG_EAGER", "1")
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2508_08062_b200 import FilterParams, Method, Solver, SolverConfig, problems  # noqa: E402

cfg, scale, iters = int(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3])
spec = problems.CONFIGS[cfg]
p = (problems.cached_config(cfg) if cfg == 4 and scale == 1.0
     else problems.make_config(cfg, scale=scale))
meth = {"aa": Method.AA_PDHG, "faa": Method.FAA_PDHG}[spec["method"]]
with Solver(p) as s:
    out = s.solve(SolverConfig(method=meth, m=spec["memory"], toll=1e-9, max_iters=iters,
                               tau=0.05, sigma=0.05, reduction="tree",
                               filter=FilterParams(c_s=spec.get("c_s", 0.2),
                                                   kappa_bar=spec.get("kappa_bar", 1e9))))
print("nnz", p.k.nnz, "iterations", out.result.iterations)
