"""Full-size parity fixtures for BASELINE.json configs 1-4, made by the
REFERENCE ITSELF (test infrastructure; VERDICT r01 "Next round" item 1,
SURVEY.md §8(c) item 5).

Run here, where /root/reference exists and oracle/_ref is built:

    python tests/golden/make_fullsize.py 2 3        # ~10 min
    python tests/golden/make_fullsize.py 4          # ~30 GB RAM, ~30 min

For each config the instance comes from paper_2508_08062_b200.problems
(seeded; the GPU test regenerates it on the box and checks the input
digest below first). The step size is the reference's own
``select_step_sizes`` (its seeded power iteration,
proj/src/solver.cpp:112-123); the first K iterates of the reference's
``solve()`` (proj/src/solver.cpp:125-253) at that explicit tau are recorded:

* every trajectory record (g_norm, objective, r_gap, r_primal, r_dual as C99
  hex; aa_step, i, j) — solver.cpp:138-149 fills them;
* the final iterate u_K: ||x||, ||y||, sum x, sum y, and x/y at 4096 fixed
  indices, hex.

Output: tests/golden/fullsize_cfg<N>.json (small; the instance is not stored).
"""
from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))

from oracle.pyoracle import Oracle  # noqa: E402
from paper_2508_08062_b200 import problems  # noqa: E402
from paper_2508_08062_b200.api import FilterParams, Method, SolverConfig  # noqa: E402

ITERATES = {1: 50, 2: 50, 3: 50, 4: 20}
SAMPLES = 4096


def hx(a):
    return [float(v).hex() for v in np.asarray(a, dtype=np.float64).ravel()]


def digest(p) -> str:
    """sha256 over the instance arrays (CSR + c, q, l, u) — pins the generator."""
    h = hashlib.sha256()
    for a in (p.k.row_ptr, p.k.col_idx, p.k.vals, p.c, p.q, p.l, p.u):
        h.update(np.ascontiguousarray(a).view(np.uint8))
    return h.hexdigest()


def sample_index(size: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(size, size=min(SAMPLES, size), replace=False))


def solver_config(cfg_id: int, tau: float, iters: int) -> SolverConfig:
    spec = problems.CONFIGS[cfg_id]
    meth = {"aa": Method.AA_PDHG, "faa": Method.FAA_PDHG}[spec["method"]]
    filt = FilterParams(c_s=spec.get("c_s", 0.2), kappa_bar=spec.get("kappa_bar", 1e9))
    # toll far below reach: exactly `iters` iterations (MAX_ITERS)
    return SolverConfig(method=meth, m=spec["memory"], toll=1e-300, max_iters=iters, tau=tau,
                        sigma=tau, filter=filt, max_wall_seconds=1e9)


def make(cfg_id: int) -> dict:
    t0 = time.perf_counter()
    p = problems.make_config(cfg_id)
    tgen = time.perf_counter() - t0
    dig = digest(p)
    print(f"cfg{cfg_id}: generated {p.k.nrows}x{p.n()} nnz={p.k.nnz} in {tgen:.0f}s", flush=True)
    ref = Oracle("ref")
    t0 = time.perf_counter()
    st = ref.select_step_sizes(p, SolverConfig())
    tpow = time.perf_counter() - t0
    print(f"cfg{cfg_id}: tau={st.tau!r} ({tpow:.0f}s)", flush=True)
    iters = ITERATES[cfg_id]
    cfg = solver_config(cfg_id, st.tau, iters)
    t0 = time.perf_counter()
    out = ref.solve(p, cfg)
    tsol = time.perf_counter() - t0
    tr = out.trajectory
    x, y = out.result.u.x, out.result.u.y
    ix, iy = sample_index(x.size, 1), sample_index(y.size, 2)
    fx = {
        "config": cfg_id,
        "source": "oracle/_ref (reference sources compiled unmodified), make_fullsize.py",
        "dims": [int(p.k.nrows), int(p.n()), int(p.k.nnz)],
        "input_sha256": dig,
        "method": int(cfg.method), "memory": cfg.m, "c_s": cfg.filter.c_s,
        "kappa_bar": cfg.filter.kappa_bar,
        "tau": float(st.tau).hex(), "sigma": float(st.sigma).hex(),
        "iterations": int(out.result.iterations), "status": out.result.status.name,
        "traj": {f: hx(tr[f]) for f in ("g_norm", "objective", "r_gap", "r_primal", "r_dual")},
        "aa_step": [int(v) for v in tr["aa_step"]],
        "i": [int(v) for v in tr["i"]], "j": [int(v) for v in tr["j"]],
        "final": {"x_norm": float(np.linalg.norm(x)).hex(), "y_norm": float(np.linalg.norm(y)).hex(),
                  "x_sum": float(np.sum(x)).hex(), "y_sum": float(np.sum(y)).hex(),
                  "x_idx": ix.tolist(), "x_val": hx(x[ix]), "y_idx": iy.tolist(),
                  "y_val": hx(y[iy])},
        "seconds": {"generate": tgen, "power": tpow, "solve": tsol},
        "planted_objective": (float(p.planted_objective).hex()
                              if getattr(p, "planted_objective", None) is not None else None),
    }
    print(f"cfg{cfg_id}: {iters} iterates in {tsol:.0f}s, aa steps {int(out.result.i)}",
          flush=True)
    return fx


def main():
    for a in sys.argv[1:] or ["2", "3"]:
        fx = make(int(a))
        (HERE / f"fullsize_cfg{a}.json").write_text(json.dumps(fx, indent=0))


if __name__ == "__main__":
    main()
