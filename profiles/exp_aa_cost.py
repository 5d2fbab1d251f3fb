"""Experiment: what the AA machinery costs per iteration on configs[1]:
PDHG vs AA-PDHG with D = 1e-300 (history push + IF node, never an attempt)
vs AA-PDHG with D = 1 (the bench setting)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2508_08062_b200 import Method, Solver, SolverConfig, problems  # noqa: E402

p = problems.make_config(1)
with Solver(p) as s:
    tau = s.select_step_sizes(SolverConfig(reduction="tree")).tau
    for name, meth, d in (("pdhg", Method.PDHG, 1.0), ("aa D=1e-300", Method.AA_PDHG, 1e-300),
                          ("aa D=1", Method.AA_PDHG, 1.0)):
        cfg = SolverConfig(method=meth, m=10, safeguard_d=d, toll=1e-9, max_iters=5000, tau=tau,
                           sigma=tau, reduction="tree")
        s.solve(SolverConfig(method=meth, m=10, safeguard_d=d, toll=1e-9, max_iters=20, tau=tau,
                             sigma=tau, reduction="tree"))
        t0 = time.perf_counter()
        r = s.solve(cfg)
        dt = time.perf_counter() - t0
        print(f"{name:12s} {1e6 * dt / r.result.iterations:7.2f} us/iteration  aa_steps={r.result.i}"
              f"  attempts={r.result.i + r.result.aa_failures}", flush=True)
