"""Experiment (not a benchmark): where a short configs[1] solve spends its time.
The driver's bench times 20 AA-PDHG iterations (3 AA steps) at ~1.9 ms while a
plain iteration costs ~45 us; this prints the host phase timers
(AAPDHG_TIMING=1, engine.cu PhaseTimer) and the CUDA-event time of solves of
20 / 100 / 1000 iterations, so the fixed per-solve cost is the intercept."""
import os
import sys
import time
from pathlib import Path

os.environ.setdefault("AAPDHG_TIMING", "1")
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2508_08062_b200 import Method, Solver, SolverConfig, problems  # noqa: E402

p = problems.make_config(1)
dev = torch.device("cuda:0")
stream = torch.cuda.Stream(dev)
with Solver(p) as s:
    import ctypes as C
    s.lib.aapdhg_cuda_set_stream(s.h, C.c_void_p(stream.cuda_stream))
    tau = 0.0775

    def cfg(it):
        return SolverConfig(method=Method.AA_PDHG, m=10, toll=1e-12, max_iters=it, tau=tau,
                            sigma=tau, reduction="tree")

    for _ in range(3):
        s.solve(cfg(64))
    for it in (20, 20, 100, 1000, 20):
        print(f"--- solve of {it} iterations", file=sys.stderr, flush=True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        with torch.cuda.stream(stream):
            e0.record(stream)
            out = s.solve(cfg(it))
            e1.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        print(f"iters {out.result.iterations} aa {out.result.i}: events {e0.elapsed_time(e1):.3f} ms, "
              f"wall {wall * 1e3:.3f} ms", file=sys.stderr, flush=True)
