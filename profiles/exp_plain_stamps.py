"""Experiment (not a benchmark): where a k_plain_loop iteration goes on
configs[1] (PDHG, graph path), from globaltimer stamps compiled in with
  make -C paper_2508_08062_b200/csrc EXTRA=-DAAPDHG_PLAIN_STAMPS
Averages over workers and iterations: K1 phase, barrier-1 wait, K2 phase,
barrier-2 wait; the waits show how far the slowest CTA trails the average."""
import ctypes as C
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2508_08062_b200 import Method, Solver, SolverConfig, problems  # noqa: E402

p = problems.make_config(1)
with Solver(p) as s:
    for meth in (Method.PDHG, Method.AA_PDHG):
        cfg = SolverConfig(method=meth, m=10, toll=1e-12, max_iters=3000, tau=0.0775, sigma=0.0775,
                           reduction="tree")
        out = (C.c_double * 7)()
        s.solve(cfg)
        s.lib.aapdhg_cuda_plain_stamps(out)
        s.solve(cfg)
        s.lib.aapdhg_cuda_plain_stamps(out)
        print(meth.name)
        for nm, v in zip(["K1 phase", "bar 1 wait", "K2 phase", "bar 2 wait", "max K1 phase",
                          "max K2 phase"], out):
            print(f"  {nm:14s} {v / 1e3:8.2f} us")
        print(f"  worker-iterations {out[6]:.0f}")
