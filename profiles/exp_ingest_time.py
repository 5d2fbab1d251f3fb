import os, sys, time
os.environ["AAPDHG_TIMING"] = "2"
sys.path.insert(0, ".")
import torch
from paper_2508_08062_b200 import Solver, problems
import bench
p = problems.cached_config(4)
hp, hout = bench.pinned_problem(torch, p)
for r in range(2):
    t0 = time.perf_counter()
    s = Solver(hp)
    print("create", time.perf_counter() - t0, file=sys.stderr, flush=True)
    s.close()
