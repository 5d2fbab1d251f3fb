"""Loads the committed golden fixtures (made by tests/golden/make_golden.py
from the reference itself) — test infrastructure."""
from __future__ import annotations

import json
from functools import lru_cache
from pathlib import Path

import numpy as np

from paper_2508_08062_b200.api import (AAParams, FilterParams, Method, ProblemData,
                                       SolverConfig, SparseMatrix)

GOLDEN = Path(__file__).resolve().parent / "golden"


def unhex(v):
    return np.array([float.fromhex(s) for s in v], dtype=np.float64)


@lru_cache(maxsize=1)
def golden():
    with open(GOLDEN / "golden.json") as f:
        return json.load(f)


@lru_cache(maxsize=1)
def _arrays():
    return dict(np.load(GOLDEN / "golden_problems.npz"))


def problem(name: str) -> ProblemData:
    a = _arrays()
    m, n, m1 = (int(v) for v in a[f"{name}.dims"])
    k = SparseMatrix(m, n, a[f"{name}.row_ptr"], a[f"{name}.col_idx"], a[f"{name}.vals"])
    return ProblemData(k, m1, a[f"{name}.c"], a[f"{name}.q"], a[f"{name}.l"], a[f"{name}.u"],
                       name=name)


def config(d: dict, reduction: str = "serial") -> SolverConfig:
    cfg = SolverConfig(method=Method(d["method"]), m=d["m"], safeguard_d=d["D"],
                       safeguard_eps=d["eps"], aa=AAParams(beta=d["beta"], eta=d["eta"]),
                       filter=FilterParams(c_s=d["c_s"], kappa_bar=d["kappa_bar"]),
                       toll=d["toll"], kkt_eps=d["kkt_eps"], kkt_terminate=d["kkt_terminate"],
                       max_iters=d["max_iters"], tau=d["tau"], sigma=d["sigma"],
                       reduction=reduction)
    return cfg


def config_for(case: dict, reduction: str = "serial") -> SolverConfig:
    cfg = config(case["config"], reduction)
    if case["name"] == "setcover_AA_dhat":
        p = problem(case["problem"])
        cfg.aa.d_hat = np.linspace(0.5, 1.5, p.n() + p.k.nrows)
    return cfg


TRAJ_FLOAT = ("g_norm", "r_gap", "r_primal", "r_dual", "objective")


def assert_traj_equal(traj, case, exact=True, rtol=0.0):
    t = case["traj"]
    k = len(t["g_norm"])
    assert traj.size >= k, (traj.size, k)
    for f in TRAJ_FLOAT:
        want = unhex(t[f])
        got = traj[f][:k]
        if exact:
            assert np.array_equal(got, want), (f, np.flatnonzero(got != want)[:5])
        else:
            np.testing.assert_allclose(got, want, rtol=rtol, atol=0, err_msg=f)
    for f in ("aa_step", "i", "j"):
        assert np.array_equal(traj[f][:k], np.array(t[f])), f
