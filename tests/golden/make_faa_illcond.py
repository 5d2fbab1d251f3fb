"""Ill-conditioned FAA per-op fixtures (test infrastructure).

The reference's FAA solve is a Householder QR (filtering.cpp:25-50,
sparse_linalg.cpp:131-192): its error grows like kappa(F) u. This script
builds histories F with prescribed condition numbers 1e2 .. 1e8, runs the
REFERENCE's build_filtered_memory + filtered_aa_apply (oracle/_ref) on them,
and records, next to the reference's output, the exact candidate
(mpmath, 250-bit normal equations on the kept columns) so the GPU test can
hold the device to the exact answer and show the reference's own distance
from it.

    python tests/golden/make_faa_illcond.py   ->  tests/golden/faa_illcond.json
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import mpmath as mp
import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))

from oracle.pyoracle import Oracle  # noqa: E402


def hx(a):
    return [float(v).hex() for v in np.asarray(a, dtype=np.float64).ravel()]


def exact_candidate(E, F, u, g, beta=1.0):
    mp.mp.prec = 250
    Fm = mp.matrix(F.T.tolist())
    gm = mp.matrix(g.tolist())
    w = mp.lu_solve(Fm.T * Fm, Fm.T * gm)
    out = []
    for t in range(len(u)):
        v = mp.mpf(u[t]) + beta * mp.mpf(g[t])
        for j in range(F.shape[0]):
            v -= w[j] * (mp.mpf(E[j, t]) + beta * mp.mpf(F[j, t]))
        out.append(float(v))
    return np.array(out)


def main():
    ref = Oracle("ref")
    rng = np.random.default_rng(20250808)
    cases = []
    for p in (6, 10):
        for kappa in (1e2, 1e4, 1e6, 1e8):
            N = 160
            Q, _ = np.linalg.qr(rng.standard_normal((N, p)))
            V, _ = np.linalg.qr(rng.standard_normal((p, p)))
            F = ((Q * np.logspace(0, -np.log10(kappa), p)) @ V.T).T.copy()  # p x N
            E = rng.standard_normal((p, N))
            u = rng.standard_normal(N)
            g = 0.1 * rng.standard_normal(N) + F.T @ rng.standard_normal(p)
            for c_s, kb in ((1e-12, 1e300), (0.2, 1e9)):
                rc, out, kept = ref.filtered_aa_apply(E, F, u, g, c_s=c_s, kappa_bar=kb)
                kept = kept.astype(bool)
                ex = exact_candidate(E[kept], F[kept], u, g) if rc == 0 and kept.any() else None
                cases.append(dict(p=p, N=N, kappa=kappa, c_s=c_s, kappa_bar=kb, rc=int(rc),
                                  kept=kept.astype(int).tolist(), du=hx(E), dg=hx(F), u=hx(u),
                                  g=hx(g), ref=hx(out) if rc == 0 else None,
                                  exact=hx(ex) if ex is not None else None))
                if ex is not None:
                    sc = np.max(np.abs(ex))
                    print(f"p={p} kappa={kappa:.0e} c_s={c_s} kept={kept.sum()} "
                          f"|ref-exact|/|exact|={np.max(np.abs(out - ex)) / sc:.2e}")
    (HERE / "faa_illcond.json").write_text(json.dumps(
        {"generated_by": "tests/golden/make_faa_illcond.py (oracle/_ref + mpmath)",
         "cases": cases}))


if __name__ == "__main__":
    main()
