"""Experiment (not a benchmark): where a short solve spends its time.
The driver's bench times 20 AA-PDHG iterations; this prints the host phase
timers (AAPDHG_TIMING=1, engine.cu PhaseTimer) and the CUDA-event time of
solves of several lengths with page-locked result buffers (as the bench), so
the fixed per-solve cost is the intercept.
usage: exp_fixed_cost.py [cfg=1] [lengths=20,20,100,1000,20] [ENV=a/b ...]
(ENV=a/b: each length runs once per value of that environment switch, in turn)"""
import ctypes as C
import os
import sys
import time
from pathlib import Path

os.environ.setdefault("AAPDHG_TIMING", "1")
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2508_08062_b200 import Method, Solver, SolverConfig  # noqa: E402

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 1
lengths = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "20,20,100,1000,20").split(",")]
p = bench.load_workload(cfg_id)
hp, hout = bench.pinned_problem(torch, p)
dev = torch.device("cuda:0")
stream = torch.cuda.Stream(dev)
with Solver(p) as s:
    s.lib.aapdhg_cuda_set_stream(s.h, C.c_void_p(stream.cuda_stream))
    tau = s.select_step_sizes(bench.solver_config()).tau if cfg_id == 4 else 0.0775

    def cfg(it):
        return SolverConfig(method=Method.AA_PDHG, m=10, toll=1e-12, max_iters=it, tau=tau,
                            sigma=tau, reduction="tree")

    for _ in range(3 if cfg_id == 1 else 1):
        s.solve(cfg(64 if cfg_id == 1 else 5), out=hout)
    ab = [a.split("=", 1) for a in sys.argv[3:]]
    variants = [[]]
    for k, vals in ab:
        variants = [v + [(k, x)] for v in variants for x in vals.split("/")]
    for it, var in [(it, var) for it in lengths for var in variants]:
        for k, x in var:
            os.environ[k] = x
        print(f"--- solve of {it} iterations {var}", file=sys.stderr, flush=True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        with torch.cuda.stream(stream):
            e0.record(stream)
            out = s.solve(cfg(it), out=hout)
            e1.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        print(f"iters {out.result.iterations} aa {out.result.i}: events {e0.elapsed_time(e1):.3f} ms, "
              f"wall {wall * 1e3:.3f} ms", file=sys.stderr, flush=True)
    # page-locked D2H rate of the result sizes
    n, m = p.n(), p.k.nrows
    d = torch.empty(n, dtype=torch.float64, device=dev)
    h = torch.empty(n, dtype=torch.float64, pin_memory=True)
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        h.copy_(d, non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"D2H page-locked {n * 8 / 1e6:.1f} MB: {dt * 1e3:.3f} ms ({n * 8 / dt / 1e9:.1f} GB/s)",
          file=sys.stderr, flush=True)
