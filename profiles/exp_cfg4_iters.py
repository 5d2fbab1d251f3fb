"""Experiment (not a benchmark): per-iteration device timestamps (record.elapsed_s) of the
configs[4] solve the bench times (20 and 60 AA-PDHG iterations, explicit tau, page-locked
result buffers), with the host phase timers (AAPDHG_TIMING=1) and the CUDA-event total."""
import ctypes as C
import os
import sys
from pathlib import Path

os.environ.setdefault("AAPDHG_TIMING", "1")
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2508_08062_b200 import Solver  # noqa: E402

p = bench.load_workload(4)
hp, hout = bench.pinned_problem(torch, p)
dev = torch.device("cuda:0")
stream = torch.cuda.Stream(dev)
with Solver(p) as s:
    s.lib.aapdhg_cuda_set_stream(s.h, C.c_void_p(stream.cuda_stream))
    tau = s.select_step_sizes(bench.solver_config()).tau
    s.solve(bench.solver_config(tau=tau, max_iters=5), out=hout)
    for it in (20, 20, 60):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            out = s.solve(bench.solver_config(tau=tau, max_iters=it), out=hout)
            e1.record(stream)
        torch.cuda.synchronize()
        tr = out.trajectory
        el = [float(r["elapsed_s"]) for r in tr]
        aa = [int(r["aa_step"]) for r in tr]
        print(f"--- {it} iterations: events {e0.elapsed_time(e1):.2f} ms, records {len(tr)}, "
              f"AA steps {out.result.i}, rejected {out.result.j}", flush=True)
        prev = 0.0
        for k, (t, a) in enumerate(zip(el, aa)):
            print(f"  k={k:3d} aa={a} elapsed {1e3 * t:9.3f} ms  +{1e3 * (t - prev):8.3f}")
            prev = t
