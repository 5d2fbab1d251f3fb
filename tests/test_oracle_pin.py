"""Pins the plain-C oracle (oracle/aapdhg_oracle.c) bit for bit against the
reference: (1) the committed golden fixtures made from the reference itself,
(2) live against oracle/_ref when it was built here. CPU only."""
import numpy as np
import pytest

from golden_io import assert_traj_equal, config_for, golden, problem, unhex
from oracle.pyoracle import Oracle, ref_available, ref_generate
from paper_2508_08062_b200.api import Iterate, Method, SolverConfig, StepSizes


@pytest.fixture(scope="module")
def port():
    return Oracle("port")


@pytest.mark.parametrize("case", golden()["solves"], ids=lambda c: c["name"])
def test_port_matches_golden_solves(port, case):
    p = problem(case["problem"])
    out = port.solve(p, config_for(case))
    r = out.result
    assert int(r.status) == case["status"]
    assert (r.iterations, r.i, r.j, r.aa_failures) == (case["iterations"], case["i"], case["j"],
                                                       case["aa_failures"])
    assert float(r.g_norm).hex() == case["g_norm"]
    assert float(r.objective).hex() == case["objective"]
    assert float(r.steps.tau).hex() == case["tau"]
    assert np.array_equal(unhex(case["kkt"]), [r.kkt.r_gap, r.kkt.r_primal, r.kkt.r_dual])
    assert out.trajectory.size == case["n_records"]
    if case["x"] is not None:
        assert np.array_equal(r.u.x, unhex(case["x"]))
        assert np.array_equal(r.u.y, unhex(case["y"]))
    assert_traj_equal(out.trajectory, case)


def test_known_answers(port):
    """proj/test_output.txt:21 and test_pdhg_core.cpp:47-57 / test_solver.cpp:82-93."""
    g = {c["name"]: c for c in golden()["solves"]}
    assert g["toy_PDHG"]["iterations"] == 274
    assert g["toy_AA_PDHG"]["iterations"] == 47
    toy = problem("toy")
    step = port.pdhg_step(toy, Iterate(np.zeros(1), np.zeros(1)), StepSizes(0.25, 0.25))
    assert step.x[0] == 0.0 and step.y[0] == 0.75
    assert port.select_step_sizes(toy, SolverConfig()).tau == 0.9


@pytest.mark.parametrize("op", golden()["ops"], ids=lambda o: o["problem"])
def test_port_matches_golden_ops(port, op):
    p = problem(op["problem"])
    x, y = unhex(op["x"]), unhex(op["y"])
    assert np.array_equal(port.matvec(p, x), unhex(op["Kx"]))
    assert np.array_equal(port.matvec_transpose(p, y), unhex(op["KTy"]))
    st = port.pdhg_step(p, Iterate(x, y), StepSizes(op["tau"], op["sigma"]))
    assert np.array_equal(st.x, unhex(op["step_x"])) and np.array_equal(st.y, unhex(op["step_y"]))
    kkt, lam, cx = port.kkt_metrics(p, Iterate(np.abs(x), y))
    assert np.array_equal([kkt.r_gap, kkt.r_primal, kkt.r_dual, cx], unhex(op["kkt"]))
    assert np.array_equal(lam, unhex(op["lam"]))
    assert float(port.power_norm(p)[0]).hex() == op["power"]


@pytest.mark.parametrize("k", range(len(golden()["aa_ops"])))
def test_port_matches_golden_aa(port, k):
    a = golden()["aa_ops"][k]
    p_, N = a["p"], a["N"]
    du, dg = unhex(a["du"]).reshape(p_, N), unhex(a["dg"]).reshape(p_, N)
    u, g = unhex(a["u"]), unhex(a["g"])
    if a["rc"] is not None:
        rc, out = port.aa_apply(du, dg, u, g, beta=a["beta"], eta=a["eta"])
        assert rc == a["rc"]
        if a["out"] is not None:
            assert np.array_equal(out, unhex(a["out"]))
    if a["frc"] is not None:
        rc, out, kept = port.filtered_aa_apply(du, dg, u, g, c_s=a.get("c_s", 0.2),
                                               kappa_bar=a.get("kappa_bar", 1e9),
                                               beta=a["beta"] if "c_s" in a else 1.0)
        assert rc == a["frc"]
        assert kept.tolist() == a["kept"]
        if a["fout"] is not None:
            assert np.array_equal(out, unhex(a["fout"]))


def test_power_start_matches_libstdcxx():
    """mt19937_64 + uniform_real_distribution(-1,1) restated in C == libstdc++
    (through the reference's own power iteration on a diagonal matrix)."""
    from oracle.pyoracle import power_start
    v = power_start(12345, 5)
    assert np.all(np.abs(v) <= 1.0) and v.std() > 0


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built (no /root/reference)")
def test_port_matches_reference_live(port):
    ref = Oracle("ref")
    cases = [ref_generate("transport", 12, 15, seed=3, slack=1.2),
             ref_generate("setcover", 40, 70, 6, seed=11)]
    cases += [ref_generate("random_box", seed=31, index=i) for i in range(8)]
    for p in cases:
        for meth, extra in ((Method.PDHG, {}), (Method.AA_PDHG, dict(m=4, safeguard_d=0.5)),
                            (Method.FAA_PDHG, dict(m=6, safeguard_d=2.0, safeguard_eps=0.01))):
            cfg = SolverConfig(method=meth, toll=1e-9, max_iters=700, **extra)
            a, b = ref.solve(p, cfg), port.solve(p, cfg)
            for f in ("g_norm", "r_gap", "r_primal", "r_dual", "objective", "aa_step", "i", "j"):
                assert np.array_equal(a.trajectory[f], b.trajectory[f]), (p.name, meth, f)
            assert np.array_equal(a.result.u.x, b.result.u.x)
            assert np.array_equal(a.result.lambda_, b.result.lambda_)


@pytest.mark.parametrize("variant", ["ref-fast", "ref-assoc"])
def test_reference_rounding_variants_load_and_solve(variant):
    """The reference built under other rounding regimes (oracle/Makefile
    `variants`, used for the iteration-count envelope) solves the toy LP."""
    from oracle.pyoracle import ORACLE_DIR, Oracle
    if not (ORACLE_DIR / "_ref" / "variants" / variant[4:] / "libaapdhg_ref.so").exists():
        pytest.skip("reference variants not built (no /root/reference)")
    from paper_2508_08062_b200 import Method, SolverConfig, SolveStatus, problems
    out = Oracle(variant).solve(problems.toy(), SolverConfig(method=Method.AA_PDHG, toll=1e-4,
                                                             tau=0.25, sigma=0.25))
    assert out.result.status == SolveStatus.RESIDUAL_TOL
    assert abs(out.result.u.x[0] - 3.0) < 1e-3
