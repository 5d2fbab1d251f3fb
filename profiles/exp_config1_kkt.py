"""Parity item 4 of SURVEY.md §8(c) on BASELINE configs[1] (100k x 200k, AA-PDHG
m=10): iterations until max KKT <= 1e-6 (kkt_terminate, the metric's
"time-to-1e-6 KKT"), from the reference itself under three rounding regimes
(oracle/_ref and its variants) and from the sm_100a path in SERIAL and TREE
order. All arms use the reference's own step size (select_step_sizes).
  python profiles/exp_config1_kkt.py ref|ref-fast|ref-assoc   (CPU: ~30 min each)
  python profiles/exp_config1_kkt.py gpu                       (the B200 arms)
  python profiles/exp_config1_kkt.py ref@+1 ref@-2 ...         (the reference at tau shifted
                                                                by +1 / -2 ulp: the spread of
                                                                its own count under a last-bit
                                                                change of tau)
  python profiles/exp_config1_kkt.py gpu@-3:3                  (the B200 TREE arm at each
                                                                shift in -3..3 ulp)
Each arm prints one JSON line."""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2508_08062_b200 import Method, SolverConfig, problems  # noqa: E402


def cfg(tau, reduction="auto"):
    return SolverConfig(method=Method.AA_PDHG, m=10, toll=1e-12, kkt_eps=1e-6,
                        kkt_terminate=True, max_iters=200000, max_wall_seconds=36000.0,
                        tau=tau, sigma=tau, reduction=reduction)


def row(arm, r, dt):
    return {"arm": arm, "iterations": r.result.iterations, "aa_steps": r.result.i,
            "status": r.result.status.name, "objective": r.result.objective,
            "kkt": [r.result.kkt.r_gap, r.result.kkt.r_primal, r.result.kkt.r_dual], "seconds": dt}


def shifted(tau, ulps):
    import numpy as np
    for _ in range(abs(ulps)):
        tau = float(np.nextafter(tau, np.inf if ulps > 0 else -np.inf))
    return tau


def main():
    arm = sys.argv[1]
    p = problems.make_config(1)
    if arm.startswith("gpu@"):
        from paper_2508_08062_b200 import Solver
        lo, hi = (int(v) for v in arm[4:].split(":"))
        with Solver(p) as s:
            tau0 = s.select_step_sizes(SolverConfig(reduction="serial")).tau
            for u in range(lo, hi + 1):
                tau = shifted(tau0, u)
                t0 = time.perf_counter()
                r = s.solve(cfg(tau, "tree"))
                print(json.dumps(dict(row(f"gpu-tree@{u:+d}", r, time.perf_counter() - t0),
                                      tau=tau)), flush=True)
        return
    if "@" in arm:
        from oracle.pyoracle import Oracle
        kind, u = arm.split("@")
        orc = Oracle(kind)
        tau = shifted(orc.select_step_sizes(p, SolverConfig()).tau, int(u))
        t0 = time.perf_counter()
        r = orc.solve(p, cfg(tau))
        print(json.dumps(dict(row(arm, r, time.perf_counter() - t0), tau=tau)), flush=True)
        return
    if arm == "gpu":
        from paper_2508_08062_b200 import Solver
        with Solver(p) as s:
            tau = s.select_step_sizes(SolverConfig(reduction="serial")).tau
            for red in ("tree", "serial"):
                t0 = time.perf_counter()
                r = s.solve(cfg(tau, red))
                print(json.dumps(dict(row("gpu-" + red, r, time.perf_counter() - t0), tau=tau)),
                      flush=True)
        return
    from oracle.pyoracle import Oracle
    orc = Oracle(arm)
    tau = orc.select_step_sizes(p, SolverConfig()).tau
    t0 = time.perf_counter()
    r = orc.solve(p, cfg(tau))
    print(json.dumps(dict(row(arm, r, time.perf_counter() - t0), tau=tau)), flush=True)


if __name__ == "__main__":
    main()
