"""Measurement of every BASELINE config on one B200, beside
the reference CPU solve() (oracle/_ref) on the same host. Not the bench line
(bench.py measures configs[1]); one JSON object per config on stdout.

usage: exp_configs.py CFG[:ITERS[:CPU_ITERS[:TTT_CAP]]] ...
  ITERS      iterations timed on the GPU (explicit tau, after one warm-up solve)
  CPU_ITERS  iterations of the reference solve() timed on the host (0 = skip)
  TTT_CAP    wall cap (s) of a full solve to toll 1e-6 on the GPU (0 = skip)
"""
import ctypes as C
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

from paper_2508_08062_b200 import (FilterParams, Method, Solver, SolverConfig,  # noqa: E402
                                   problems)


def config_for(cfg, tau=0.0, max_iters=100000, wall=3600.0, toll=1e-6):
    spec = problems.CONFIGS[cfg]
    meth = {"aa": Method.AA_PDHG, "faa": Method.FAA_PDHG}[spec["method"]]
    filt = FilterParams(c_s=spec.get("c_s", FilterParams().c_s),
                        kappa_bar=spec.get("kappa_bar", FilterParams().kappa_bar))
    return SolverConfig(method=meth, m=spec["memory"], toll=toll, max_iters=max_iters, tau=tau,
                        sigma=tau, max_wall_seconds=wall, filter=filt)


def kernel_profile(s, cfg, tau, iters):
    s.lib.aapdhg_cuda_set_profiling(s.h, 1)
    s.solve(config_for(cfg, tau, iters))
    names = C.create_string_buffer(4096)
    ms = (C.c_double * 64)()
    la = (C.c_uint64 * 64)()
    cnt = C.c_int32()
    s.lib.aapdhg_cuda_kernel_times(s.h, names, 4096, ms, la, 64, C.byref(cnt))
    s.lib.aapdhg_cuda_set_profiling(s.h, 0)
    kn = names.value.decode().split("\n")[: cnt.value]
    return {kn[i]: {"us": 1e3 * ms[i] / max(la[i], 1), "launches": int(la[i])}
            for i in range(cnt.value)}


def run(cfg, iters, cpu_iters, ttt_cap):
    out = {"config": cfg, "spec": {k: v for k, v in problems.CONFIGS[cfg].items()}}
    t0 = time.perf_counter()
    p = problems.cached_config(4) if cfg == 4 else problems.make_config(cfg)
    out["generate_s"] = time.perf_counter() - t0
    out["shape"] = {"m": p.k.nrows, "n": p.n(), "nnz": int(p.k.nnz)}
    t0 = time.perf_counter()
    s = Solver(p)
    out["problem_create_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    tau = s.select_step_sizes(config_for(cfg)).tau
    out["step_sizes_s"] = time.perf_counter() - t0
    out["tau"] = tau
    s.solve(config_for(cfg, tau, 5))  # warm-up (graph instantiation)
    t0 = time.perf_counter()
    r = s.solve(config_for(cfg, tau, iters))
    dt = time.perf_counter() - t0
    out["gpu"] = {"iterations": r.result.iterations, "aa_steps": r.result.i, "seconds": dt,
                  "iter_per_s": r.result.iterations / dt,
                  "us_per_iter": 1e6 * dt / max(r.result.iterations, 1)}
    out["kernels_us"] = kernel_profile(s, cfg, tau, min(iters, 200))
    if ttt_cap > 0:
        t0 = time.perf_counter()
        full = s.solve(config_for(cfg, wall=ttt_cap))
        tr = full.trajectory
        mk = np.maximum(np.maximum(tr["r_gap"], tr["r_primal"]), tr["r_dual"])
        hit = np.flatnonzero(mk <= 1e-6)
        out["gpu_time_to_tol"] = {
            "seconds": time.perf_counter() - t0, "status": full.result.status.name,
            "iterations": full.result.iterations, "aa_steps": full.result.i,
            "objective": full.result.objective,
            "planted_objective": getattr(p, "planted_objective", None),
            "max_kkt": full.result.kkt.max(),
            "first_kkt_le_1e-6": ({"k": int(tr["k"][hit[0]]),
                                   "elapsed_s": float(tr["elapsed_s"][hit[0]])}
                                  if hit.size else None)}
    s.close()
    if cpu_iters > 0:
        from oracle.pyoracle import Oracle, ref_available
        kind = "reference" if ref_available() else "port"
        orc = Oracle("ref" if kind == "reference" else "port")
        t0 = time.perf_counter()
        rr = orc.solve(p, config_for(cfg, tau, cpu_iters))
        dt = time.perf_counter() - t0
        out["cpu"] = {"kind": kind, "threads": 1, "iterations": rr.result.iterations,
                      "seconds": dt, "iter_per_s": rr.result.iterations / dt,
                      "cores_on_host": os.cpu_count()}
        out["speedup_per_iteration"] = out["gpu"]["iter_per_s"] / out["cpu"]["iter_per_s"]
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    for arg in sys.argv[1:]:
        parts = [float(v) for v in arg.split(":")]
        cfg = int(parts[0])
        iters = int(parts[1]) if len(parts) > 1 else 2000
        cpu_iters = int(parts[2]) if len(parts) > 2 else 0
        ttt = parts[3] if len(parts) > 3 else 0.0
        run(cfg, iters, cpu_iters, ttt)
