"""FAA cost on BASELINE config 2 (transport 2000 x 2000, FAA m=10): device
time per iteration and per FAA attempt with the double-double Gram on the
warp-per-item dots (default) or on the register Gram (AAPDHG_FAA_GRAM=1).
  python profiles/exp_faa_cost.py [iters]"""
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2508_08062_b200 import FilterParams, Method, Solver, SolverConfig, problems  # noqa

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 300
p = problems.make_config(2)
spec = problems.CONFIGS[2]
with Solver(p) as s:
    tau = s.select_step_sizes(SolverConfig()).tau
    for meth in (Method.FAA_PDHG, Method.PDHG):
        cfg = SolverConfig(method=meth, m=10, toll=1e-12, max_iters=iters, tau=tau, sigma=tau,
                           filter=FilterParams(c_s=spec["c_s"], kappa_bar=spec["kappa_bar"]))
        s.solve(cfg)
        t0 = time.perf_counter()
        r = s.solve(cfg)
        dt = time.perf_counter() - t0
        print(json.dumps({"method": meth.name, "faa_gram": os.environ.get("AAPDHG_FAA_GRAM", "0"),
                          "iterations": r.result.iterations, "aa_steps": r.result.i,
                          "us_per_iteration": 1e6 * dt / r.result.iterations}), flush=True)

# per-kernel device times (eager launches with events, aapdhg_cuda_kernel_times)
import ctypes as C  # noqa: E402

with Solver(p) as s:
    lib = s.lib
    cfg = SolverConfig(method=Method.FAA_PDHG, m=10, toll=1e-12, max_iters=iters, tau=tau,
                       sigma=tau, filter=FilterParams(c_s=spec["c_s"], kappa_bar=spec["kappa_bar"]))
    lib.aapdhg_cuda_set_profiling(s.h, 1)
    s.solve(cfg)
    names = C.create_string_buffer(4096)
    msa = (C.c_double * 64)()
    la = (C.c_uint64 * 64)()
    cnt = C.c_int32()
    lib.aapdhg_cuda_kernel_times(s.h, names, 4096, msa, la, 64, C.byref(cnt))
    kn = names.value.decode().split("\n")[: cnt.value]
    print(json.dumps({k: round(1e3 * msa[i] / max(la[i], 1), 1) for i, k in enumerate(kn)}))
