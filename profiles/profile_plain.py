"""Short, deterministic workload for ncu captures of k_plain_loop, the
persistent plain-step grid: BASELINE configs[1] (100k x 200k, 4M nnz),
AA-PDHG m=10 (the PUSH variant the bench runs), explicit step size, launched
on the stream instead of the conditional graph (ncu cannot profile kernels of
graphs with conditional nodes). D = 1e-300 keeps every step plain, so the
launches run the iteration batches 8, 16, 32, ... (plus no-op launches past
each batch's end): `-k regex:k_plain_loop -c 1` captures an 8-iteration
launch. Not a benchmark."""
import os
import sys
from pathlib import Path

os.environ.setdefault("AAPDHG_EAGER", "1")
os.environ.setdefault("AAPDHG_PERSIST_EAGER", "1")

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2508_08062_b200 import Method, Solver, SolverConfig, problems  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 24
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 0  # calibration solves of 64 iterations first
p = problems.make_config(1)
with Solver(p) as s:
    for _ in range(warm):  # (each: 4 k_plain_loop launches, batches 8+16+32+64 -> ncu --launch-skip 4*warm)
        s.solve(SolverConfig(method=Method.AA_PDHG, m=10, safeguard_d=1e-300, toll=1e-12,
                             max_iters=64, tau=0.0775, sigma=0.0775, reduction="tree"))
    out = s.solve(SolverConfig(method=Method.AA_PDHG, m=10, safeguard_d=1e-300, toll=1e-12,
                               max_iters=iters, tau=0.0775, sigma=0.0775, reduction="tree"))
    import ctypes as C
    pi, ps, pl = C.c_uint64(), C.c_double(), C.c_uint64()
    s.lib.aapdhg_cuda_last_plain_loop(s.h, C.byref(pi), C.byref(ps), C.byref(pl))
print("iterations", out.result.iterations, "aa", out.result.i, "plain-loop iterations",
      pi.value, "launches that ran", pl.value, "device s", ps.value)
