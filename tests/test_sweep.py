"""Sweep mode (proj/src/cli.cpp:142-214): the case cross
product and names (CPU), and concurrent solves on resident handles (GPU)."""
import numpy as np
import pytest

from paper_2508_08062_b200 import (FilterParams, Method, Solver, SolverConfig, problems,
                                   solve_sweep, sweep_cases)


def test_sweep_case_names_and_order():
    base = SolverConfig(method=Method.FAA_PDHG, m=7, filter=FilterParams(c_s=0.3, kappa_bar=5.0))
    cs = sweep_cases(base, d=[1.0, 0.25], eps=[1e-3], m=[3, 10], kappa_bar=[1e4])
    assert [c.name for c in cs] == ["D1_eps0.001_m3_kappa10000", "D1_eps0.001_m10_kappa10000",
                                    "D0.25_eps0.001_m3_kappa10000",
                                    "D0.25_eps0.001_m10_kappa10000"]
    assert cs[2].cfg.safeguard_d == 0.25 and cs[2].cfg.m == 3
    assert cs[0].cfg.filter.c_s == 0.3 and cs[0].cfg.filter.kappa_bar == 1e4
    assert base.m == 7 and base.filter.kappa_bar == 5.0  # base untouched
    assert [c.name for c in sweep_cases(base)] == [""]


@pytest.mark.gpu
def test_solve_sweep_matches_sequential_solves():
    p = problems.make_config(0, scale=0.3)
    base = SolverConfig(method=Method.AA_PDHG, toll=1e-6, max_iters=3000, tau=0.1, sigma=0.1)
    cases = sweep_cases(base, d=[1.0, 1e-2], eps=[1.0, 0.5], m=[3, 5])
    got = solve_sweep(p, cases, workers=4)
    assert len(got) == len(cases)
    with Solver(p) as s:
        for (ok, err, out), c in zip(got, cases):
            assert ok, err
            ref = s.solve(c.cfg)
            assert out.result.iterations == ref.result.iterations, c.name
            assert np.array_equal(out.trajectory["g_norm"], ref.trajectory["g_norm"]), c.name
            assert np.array_equal(out.result.u.x, ref.result.u.x)


@pytest.mark.gpu
def test_solve_sweep_reports_case_errors():
    p = problems.make_config(0, scale=0.2)
    good = SolverConfig(method=Method.PDHG, toll=1e-4, max_iters=50, tau=0.1, sigma=0.1)
    bad = SolverConfig(method=Method.AA_PDHG, m=0)
    got = solve_sweep(p, [good, bad, good], workers=2)
    assert got[0][0] and got[2][0] and not got[1][0]
    assert "m must be >= 1" in got[1][1]
