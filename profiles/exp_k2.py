"""Experiment (not a benchmark): per-kernel event times of config 1 (AA-PDHG
m=10, eager launches with CUDA events) under AAPDHG_* switches, to attribute
the k_primal_side time. usage: exp_k2.py "FUSED=1,PDL=1" "FUSED=0,PDL=0" ..."""
import ctypes as C
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

if len(sys.argv) > 1 and sys.argv[1] == "child":
    from paper_2508_08062_b200 import Method, Solver, SolverConfig, problems
    p = problems.make_config(1)
    with Solver(p) as s:
        cfg = SolverConfig(method=Method.AA_PDHG, m=10, toll=1e-6, max_iters=400, tau=0.0775,
                           sigma=0.0775, reduction="tree")
        s.solve(cfg)
        s.lib.aapdhg_cuda_set_profiling(s.h, 1)
        s.solve(cfg)
        names = C.create_string_buffer(4096)
        ms = (C.c_double * 64)()
        la = (C.c_uint64 * 64)()
        cnt = C.c_int32()
        s.lib.aapdhg_cuda_kernel_times(s.h, names, 4096, ms, la, 64, C.byref(cnt))
    kn = names.value.decode().split("\n")[: cnt.value]
    print(sys.argv[2], " ".join(f"{kn[i]}={1e3 * ms[i] / max(la[i], 1):.2f}"
                                for i in range(cnt.value)), flush=True)
    sys.exit(0)

for combo in sys.argv[1:] or ["FUSED=1,PDL=1", "FUSED=1,PDL=0", "FUSED=0,PDL=0"]:
    env = dict(os.environ)
    for kv in combo.split(","):
        k, v = kv.split("=")
        env["AAPDHG_" + k] = v
    subprocess.run([sys.executable, __file__, "child", combo], env=env)
