"""Experiment (not a benchmark): L2 column-block size for the SpMVs of a large
config (default configs[4]): iterations/s and per-kernel times for each
AAPDHG_L2_BLOCK_KB value. usage: exp_block.py CFG KB [KB ...]  (KB 0 = off)"""
import ctypes as C
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2508_08062_b200 import Method, Solver, SolverConfig, problems  # noqa: E402

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 4
kbs = [int(v) for v in sys.argv[2:]] or [0, 40960, 65536, 98304]
p = problems.make_config(cfg_id)
tau = None
for kb in kbs:
    os.environ["AAPDHG_L2_BLOCK_KB"] = str(kb)
    t0 = time.perf_counter()
    s = Solver(p)
    create = time.perf_counter() - t0
    if tau is None:
        tau = s.select_step_sizes(SolverConfig(reduction="tree")).tau
    cfg = SolverConfig(method=Method.AA_PDHG, m=10, toll=1e-9, max_iters=60, tau=tau, sigma=tau,
                       reduction="tree")
    s.solve(SolverConfig(method=Method.AA_PDHG, m=10, toll=1e-9, max_iters=3, tau=tau, sigma=tau,
                         reduction="tree"))
    t0 = time.perf_counter()
    r = s.solve(cfg)
    dt = time.perf_counter() - t0
    s.lib.aapdhg_cuda_set_profiling(s.h, 1)
    s.solve(SolverConfig(method=Method.AA_PDHG, m=10, toll=1e-9, max_iters=20, tau=tau,
                         sigma=tau, reduction="tree"))
    names = C.create_string_buffer(4096)
    ms = (C.c_double * 64)()
    la = (C.c_uint64 * 64)()
    cnt = C.c_int32()
    s.lib.aapdhg_cuda_kernel_times(s.h, names, 4096, ms, la, 64, C.byref(cnt))
    kn = names.value.decode().split("\n")[: cnt.value]
    s.close()
    print(json.dumps({"config": cfg_id, "block_kb": kb, "create_s": create,
                      "us_per_iter": 1e6 * dt / r.result.iterations,
                      "kernels": {kn[i]: [round(1e3 * ms[i] / max(la[i], 1), 1), int(la[i])]
                                  for i in range(cnt.value)}}), flush=True)
