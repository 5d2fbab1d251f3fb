"""Parity item 4 of SURVEY.md §8(c) on BASELINE configs[1] (100k x 200k, AA-PDHG
m=10): iterations until max KKT <= 1e-6 (kkt_terminate, the metric's
"time-to-1e-6 KKT"), from the reference itself under three rounding regimes
(oracle/_ref and its variants) and from the sm_100a path in SERIAL and TREE
order. All arms use the reference's own step size (select_step_sizes).
  python profiles/exp_config1_kkt.py ref|ref-fast|ref-assoc   (CPU: ~30 min each)
  python profiles/exp_config1_kkt.py gpu                       (the B200 arms)
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


def main():
    arm = sys.argv[1]
    p = problems.make_config(1)
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
