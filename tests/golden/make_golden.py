"""Generates the committed golden fixtures from the REFERENCE ITSELF.

Run here (where /root/reference exists) after `make -C oracle ref`:

    python tests/golden/make_golden.py

Every number below comes from oracle/_ref/libaapdhg_ref.so — the unmodified
reference sources (proj/src/*.cpp + proj/tests/support/test_support.cpp)
compiled by oracle/Makefile. Floats are stored as C99 hex strings so the
fixtures pin results bit for bit. Problems are stored with their arrays
(golden_problems.npz) so the fixtures do not depend on any generator.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))

from oracle.pyoracle import Oracle, ref_generate  # noqa: E402
from paper_2508_08062_b200 import problems  # noqa: E402
from paper_2508_08062_b200.api import (AAParams, FilterParams, Iterate, Method,  # noqa: E402
                                       SolverConfig, StepSizes)


def hx(a):
    return [float(v).hex() for v in np.asarray(a, dtype=np.float64).ravel()]


def cfg_dict(c: SolverConfig):
    return dict(method=int(c.method), m=c.m, D=c.safeguard_d, eps=c.safeguard_eps,
                beta=c.aa.beta, eta=c.aa.eta, c_s=c.filter.c_s, kappa_bar=c.filter.kappa_bar,
                toll=c.toll, kkt_eps=c.kkt_eps, kkt_terminate=c.kkt_terminate,
                max_iters=c.max_iters, tau=c.tau, sigma=c.sigma)


def main():
    ref = Oracle("ref")
    probs = {}
    probs["toy"] = ref_generate("toy")
    for idx in range(6):
        probs[f"randbox{idx}"] = ref_generate("random_box", seed=99, index=idx)
    probs["transport20"] = ref_generate("transport", 20, 20, seed=7, slack=1.3)
    probs["setcover"] = ref_generate("setcover", 60, 120, 9, seed=5)
    probs["config0_s02"] = problems.make_config(0, scale=0.2)

    arrays = {}
    for name, p in probs.items():
        arrays[f"{name}.row_ptr"] = p.k.row_ptr
        arrays[f"{name}.col_idx"] = p.k.col_idx
        arrays[f"{name}.vals"] = p.k.vals
        for f in ("c", "q", "l", "u"):
            arrays[f"{name}.{f}"] = getattr(p, f)
        arrays[f"{name}.dims"] = np.array([p.k.nrows, p.k.ncols, p.m1], dtype=np.int64)
    np.savez_compressed(HERE / "golden_problems.npz", **arrays)

    solves = []

    def add(name, pname, cfg, keep=None):
        out = ref.solve(probs[pname], cfg)
        t = out.trajectory if keep is None else out.trajectory[:keep]
        r = out.result
        solves.append(dict(
            name=name, problem=pname, config=cfg_dict(cfg), status=int(r.status),
            iterations=r.iterations, i=r.i, j=r.j, aa_failures=r.aa_failures,
            g_norm=float(r.g_norm).hex(), objective=float(r.objective).hex(),
            kkt=hx([r.kkt.r_gap, r.kkt.r_primal, r.kkt.r_dual]), tau=float(r.steps.tau).hex(),
            x=hx(r.u.x) if r.u.x.size <= 64 else None, y=hx(r.u.y) if r.u.y.size <= 64 else None,
            n_records=int(out.trajectory.size),
            traj=dict(g_norm=hx(t["g_norm"]), aa_step=t["aa_step"].tolist(), i=t["i"].tolist(),
                      j=t["j"].tolist(), r_gap=hx(t["r_gap"]), r_primal=hx(t["r_primal"]),
                      r_dual=hx(t["r_dual"]), objective=hx(t["objective"]))))

    # proj/test_output.txt:21 — toy PDHG 274, AA 47 (tau = sigma = 0.25, toll 1e-4)
    for meth in (Method.PDHG, Method.AA_PDHG, Method.FAA_PDHG):
        add(f"toy_{meth.name}", "toy", SolverConfig(method=meth, m=5, toll=1e-4, tau=0.25,
                                                    sigma=0.25, max_iters=1000))
    add("toy_AA_auto_tau", "toy", SolverConfig(method=Method.AA_PDHG, toll=1e-9, max_iters=5000))
    add("toy_PDHG_kkt_terminate", "toy", SolverConfig(method=Method.PDHG, toll=1e-12, tau=0.25,
                                                      sigma=0.25, kkt_terminate=True,
                                                      kkt_eps=1e-3, max_iters=5000))
    for idx in range(6):
        for meth in (Method.AA_PDHG, Method.FAA_PDHG):
            add(f"randbox{idx}_{meth.name}", f"randbox{idx}",
                SolverConfig(method=meth, toll=1e-8, m=5, safeguard_d=0.1, max_iters=300000),
                keep=400)
    add("transport20_FAA", "transport20",
        SolverConfig(method=Method.FAA_PDHG, m=5, safeguard_d=10.0, safeguard_eps=0.01,
                     toll=1e-14, max_iters=600))
    add("setcover_AA_dhat", "setcover",
        SolverConfig(method=Method.AA_PDHG, m=7, toll=1e-10, max_iters=800,
                     aa=AAParams(beta=0.8, d_hat=np.linspace(0.5, 1.5, 60 + 120))))
    add("config0_s02_AA", "config0_s02",
        SolverConfig(method=Method.AA_PDHG, m=5, toll=1e-6, max_iters=20000), keep=2000)

    # single-op vectors (pdhg_core / anderson / filtering / sparse_linalg)
    ops = []
    rng = np.random.default_rng(1234)
    for pname in ("randbox0", "randbox3", "transport20"):
        p = probs[pname]
        n, m = p.n(), p.k.nrows
        x = rng.standard_normal(n)
        y = rng.standard_normal(m)
        ts = StepSizes(0.3, 0.2)
        step = ref.pdhg_step(p, Iterate(x, y), ts)
        kkt, lam, cx = ref.kkt_metrics(p, Iterate(np.abs(x), y))
        ops.append(dict(problem=pname, x=hx(x), y=hx(y), Kx=hx(ref.matvec(p, x)),
                        KTy=hx(ref.matvec_transpose(p, y)), tau=ts.tau, sigma=ts.sigma,
                        step_x=hx(step.x), step_y=hx(step.y),
                        kkt=hx([kkt.r_gap, kkt.r_primal, kkt.r_dual, cx]), lam=hx(lam),
                        power=float(ref.power_norm(p)[0]).hex()))
    aa_ops = []
    for t, (p_, N) in enumerate([(1, 7), (3, 11), (5, 40), (8, 40)]):
        du = rng.standard_normal((p_, N))
        dg = rng.standard_normal((p_, N))
        u = rng.standard_normal(N)
        g = rng.standard_normal(N)
        rc, out = ref.aa_apply(du, dg, u, g, beta=0.9, eta=1e-10)
        rc2, out2, kept = ref.filtered_aa_apply(du, dg, u, g, c_s=0.2, kappa_bar=1e9)
        aa_ops.append(dict(du=hx(du), dg=hx(dg), u=hx(u), g=hx(g), p=p_, N=N, beta=0.9, eta=1e-10,
                           rc=rc, out=hx(out) if rc == 0 else None, frc=rc2,
                           fout=hx(out2) if rc2 == 0 else None, kept=kept.tolist()))
    # crafted filter cases: near-collinear columns (angle filter drops) and a
    # small kappa_bar (length filter truncates), c_s as in config 2
    for t, (kb, cs) in enumerate([(1e9, 0.2), (30.0, 0.2), (1e4, float(np.sqrt(1 - 0.99 ** 2)))]):
        N = 25
        base = rng.standard_normal((6, N))
        f = base.copy()
        f[2] = base[1] + 0.05 * base[2]        # sine ~ 0.05 against column 1
        f[4] = base[0] - base[3] + 1e-3 * base[4]
        e = rng.standard_normal((6, N))
        u = rng.standard_normal(N)
        g = rng.standard_normal(N)
        rc2, out2, kept = ref.filtered_aa_apply(e, f, u, g, c_s=cs, kappa_bar=kb, beta=0.7)
        aa_ops.append(dict(du=hx(e), dg=hx(f), u=hx(u), g=hx(g), p=6, N=N, beta=0.7, eta=1e-10,
                           rc=None, out=None, frc=rc2, fout=hx(out2) if rc2 == 0 else None,
                           kept=kept.tolist(), c_s=cs, kappa_bar=kb))
    # rank-deficient memory with eta = 0 -> SingularError (test_anderson.cpp:159-172)
    col = rng.standard_normal(9)
    du = np.stack([col, 2 * col])
    rc, _ = ref.aa_apply(du, du, np.zeros(9), np.ones(9), eta=0.0)
    aa_ops.append(dict(du=hx(du), dg=hx(du), u=hx(np.zeros(9)), g=hx(np.ones(9)), p=2, N=9,
                       beta=1.0, eta=0.0, rc=rc, out=None, frc=None, fout=None, kept=None))

    doc = dict(generated_by="oracle/_ref (reference sources, unmodified)", solves=solves,
               ops=ops, aa_ops=aa_ops)
    with open(HERE / "golden.json", "w") as f:
        json.dump(doc, f, separators=(",", ":"))
    print("wrote", HERE / "golden.json", (HERE / "golden.json").stat().st_size, "bytes")


if __name__ == "__main__":
    main()
