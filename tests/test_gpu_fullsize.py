"""Full-size parity on BASELINE.json configs 1-4 against fixtures the
REFERENCE ITSELF produced (tests/golden/make_fullsize.py runs oracle/_ref,
the unmodified reference sources, on the same seeded instance).

For each config: the instance is regenerated here and its sha256 must match
the fixture's (the generator is pinned); the solve runs on the sm_100a path
in its default (AUTO -> TREE) reduction order at the reference's own tau
(select_step_sizes of the reference, proj/src/solver.cpp:112-123) for the
fixture's iteration count, and is held to the north-star bar
(BASELINE.json): every one of the first K iterates within 1e-10 relative
(g_norm and objective of each record), the same AA step pattern (aa_step,
i, j), and the final iterate within 1e-10 relative (norms and 4096 sampled
entries of x and y). The KKT residuals of each record are derived
quantities with cancellation (r_gap = |dual - primal| / ...): they are held
to 1e-8 relative or 1e-12 absolute. The device's own step size must agree
with the reference's to 1e-10 (same seeded power iteration,
sparse_linalg.cpp:95-123).

Config 4 (20M x 40M, 400M nnz) needs ~35 GB of host RAM and ~3 minutes
(instance generation); its fixture holds the first 20 iterates (the
reference takes ~40 s per iteration on one core).
"""
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from paper_2508_08062_b200 import FilterParams, Method, Solver, SolverConfig, problems

pytestmark = pytest.mark.gpu

GOLDEN = Path(__file__).resolve().parent / "golden"
CONFIGS = [c for c in (1, 2, 3, 4) if (GOLDEN / f"fullsize_cfg{c}.json").exists()]


def unhex(v):
    return np.array([float.fromhex(s) for s in v], dtype=np.float64)


def digest(p) -> str:
    h = hashlib.sha256()
    for a in (p.k.row_ptr, p.k.col_idx, p.k.vals, p.c, p.q, p.l, p.u):
        h.update(np.ascontiguousarray(a).view(np.uint8))
    return h.hexdigest()


def rel_err(got, want):
    got, want = np.asarray(got), np.asarray(want)
    return float(np.max(np.abs(got - want) / np.maximum(np.abs(want), 1e-300)))


@pytest.mark.parametrize("cfg_id", CONFIGS)
def test_fullsize_first_iterates_match_reference(cfg_id):
    fx = json.loads((GOLDEN / f"fullsize_cfg{cfg_id}.json").read_text())
    p = problems.make_config(cfg_id)
    assert [p.k.nrows, p.n(), p.k.nnz] == fx["dims"]
    assert digest(p) == fx["input_sha256"], "instance generator drifted from the fixture"
    tau = float.fromhex(fx["tau"])
    iters = fx["iterations"]
    cfg = SolverConfig(method=Method(fx["method"]), m=fx["memory"], toll=1e-300,
                       max_iters=iters, tau=tau, sigma=float.fromhex(fx["sigma"]),
                       filter=FilterParams(c_s=fx["c_s"], kappa_bar=fx["kappa_bar"]),
                       max_wall_seconds=1e9)
    with Solver(p) as s:
        got = s.solve(cfg)
        own_tau = s.select_step_sizes(SolverConfig()).tau
    tr = got.trajectory
    assert got.result.status.name == fx["status"]
    assert got.result.iterations == iters
    k = len(fx["aa_step"])
    assert tr.size == k
    # the AA step pattern and counters, exactly
    assert tr["aa_step"].tolist() == fx["aa_step"]
    assert tr["i"].tolist() == fx["i"] and tr["j"].tolist() == fx["j"]
    # every iterate: g_norm and objective within the north-star 1e-10
    for f in ("g_norm", "objective"):
        want = unhex(fx["traj"][f])
        assert rel_err(tr[f], want) <= 1e-10, (f, rel_err(tr[f], want))
    for f in ("r_gap", "r_primal", "r_dual"):
        want = unhex(fx["traj"][f])
        np.testing.assert_allclose(tr[f], want, rtol=1e-8, atol=1e-12, err_msg=f)
    # the final iterate
    fin = fx["final"]
    x, y = got.result.u.x, got.result.u.y
    for v, key in ((x, "x"), (y, "y")):
        nrm = float.fromhex(fin[f"{key}_norm"])
        assert abs(np.linalg.norm(v) - nrm) <= 1e-10 * nrm
        idx = np.array(fin[f"{key}_idx"])
        want = unhex(fin[f"{key}_val"])
        assert np.max(np.abs(v[idx] - want)) <= 1e-10 * max(np.max(np.abs(want)), 1e-300)
    # the device's own step size (seeded power iteration) agrees with the reference's
    assert abs(own_tau - tau) <= 1e-10 * tau, (own_tau, tau)


def test_config1_iterations_to_kkt_1e6_within_reference_envelope():
    """BASELINE configs[1] to max KKT <= 1e-6 (the metric's time-to-1e-6 KKT),
    TREE order (the bench path), at the reference's tau and at tau shifted by
    +-1 ulp. AA-PDHG is chaotic under rounding: the reference's own count
    spans [32,566, 35,588] over its strict / FMA / reassociated builds and
    +-1-2 ulp changes of tau (tests/golden/config1_envelope.json). Every GPU
    count must fall within that envelope widened by the north-star 2%, with
    KKT <= 1e-6 and the objective within 1e-6 of the planted optimum
    (c'x* = b'y*) and of the reference's final objective."""
    env = json.loads((GOLDEN / "config1_envelope.json").read_text())
    lo, hi = env["envelope"]
    ref = env["arms"]["ref"]
    p = problems.make_config(1)
    counts = []
    with Solver(p) as s:
        tau0 = ref["tau"]
        for ulps in (0, 1, -1):
            tau = float(np.nextafter(tau0, np.inf if ulps > 0 else -np.inf)) if ulps else tau0
            cfg = SolverConfig(method=Method.AA_PDHG, m=10, toll=1e-12, kkt_eps=1e-6,
                               kkt_terminate=True, max_iters=200000, max_wall_seconds=600.0,
                               tau=tau, sigma=tau, reduction="tree")
            r = s.solve(cfg).result
            assert r.status.name == "KKT_TOL"
            assert r.kkt.max() <= 1e-6
            assert abs(r.objective - p.planted_objective) <= 1e-6 * abs(p.planted_objective)
            assert abs(r.objective - ref["objective"]) <= 1e-6 * abs(ref["objective"])
            counts.append(r.iterations)
    for c in counts:
        assert 0.98 * lo <= c <= 1.02 * hi, (counts, env["envelope"])
