"""Experiment (not a benchmark): phase times of K2's fused control tail on
config 1 (AA-PDHG m=10, graph path), from globaltimer stamps compiled in with
  make -C paper_2508_08062_b200/csrc EXTRA=-DAAPDHG_TAIL_STAMPS
(the stamps add a few hundred ns; phases only, not a speed)."""
import ctypes as C
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2508_08062_b200 import Method, Solver, SolverConfig, problems  # noqa: E402

p = problems.make_config(1)
names = ["K1 phase+barrier", "K2 phase->elected", "->partials reduced", "->decided",
         "->tail end", "->next K1 start (plain)", "->next K1 start (after AA)", "iterations",
         "plain", "after AA"]
with Solver(p) as s:
    for meth in (Method.AA_PDHG, Method.PDHG):
        cfg = SolverConfig(method=meth, m=10, toll=1e-6, max_iters=3000, tau=0.0775,
                           sigma=0.0775, reduction="tree")
        s.solve(cfg)
        out = (C.c_double * 10)()
        s.lib.aapdhg_cuda_debug_stamps(out)
        s.solve(cfg)
        s.lib.aapdhg_cuda_debug_stamps(out)
        print(meth.name)
        for nm, v in zip(names, out):
            print(f"  {nm:28s} {v:10.0f}")
