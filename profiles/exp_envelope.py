"""Parity item 4 of SURVEY.md §8(c): iteration counts to toll = 1e-6 of the
reference itself under three rounding regimes (strict Release build; FMA
contraction; reassociated sums — oracle/Makefile `variants`), the C port,
and the sm_100a path in SERIAL and TREE order. AA-PDHG is chaotic under
rounding, so TREE is judged against the reference's own envelope.
usage: exp_envelope.py [CFG[:SCALE] ...]   (default: configs[0])"""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle.pyoracle import Oracle  # noqa: E402
from paper_2508_08062_b200 import Method, Solver, SolverConfig, problems  # noqa: E402


def cfg_for(spec, reduction="auto"):
    meth = {"aa": Method.AA_PDHG, "faa": Method.FAA_PDHG}[spec["method"]]
    return SolverConfig(method=meth, m=spec["memory"], toll=1e-6, max_iters=300000,
                        max_wall_seconds=600.0, reduction=reduction)


def main():
    args = sys.argv[1:] or ["0"]
    for a in args:
        cfg_id, scale = (a.split(":") + ["1.0"])[:2]
        cfg_id, scale = int(cfg_id), float(scale)
        p = problems.make_config(cfg_id, scale=scale)
        spec = problems.CONFIGS[cfg_id]
        rows = []
        for kind in ("ref", "ref-fast", "ref-assoc", "port"):
            try:
                orc = Oracle(kind)
            except FileNotFoundError as e:
                rows.append({"arm": kind, "error": str(e)})
                continue
            t0 = time.perf_counter()
            r = orc.solve(p, cfg_for(spec))
            rows.append({"arm": kind, "iterations": r.result.iterations, "aa_steps": r.result.i,
                         "status": r.result.status.name, "objective": r.result.objective,
                         "tau": r.result.steps.tau, "seconds": time.perf_counter() - t0})
        try:
            for red in ("serial", "tree"):
                with Solver(p) as s:
                    t0 = time.perf_counter()
                    r = s.solve(cfg_for(spec, red))
                    rows.append({"arm": "gpu-" + red, "iterations": r.result.iterations,
                                 "aa_steps": r.result.i, "status": r.result.status.name,
                                 "objective": r.result.objective, "tau": r.result.steps.tau,
                                 "seconds": time.perf_counter() - t0})
        except Exception as e:  # no GPU here
            rows.append({"arm": "gpu", "error": str(e)[:200]})
        ref_its = [r["iterations"] for r in rows if r["arm"].startswith("ref") and "iterations" in r]
        out = {"config": cfg_id, "scale": scale, "arms": rows,
               "reference_envelope": [min(ref_its), max(ref_its)] if ref_its else None}
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
