"""GPU: the sharded (multi-GPU) solve, SURVEY.md §8(e).

Only one GPU is available, so the partitioned path is exercised three ways:
  * LOOPBACK: `world` shards in one process on cuda:0, all-gathers as device
    copies on one stream (the same kernels and exchange schedule as NCCL);
  * LOOPBACK_P2P: the same shards with the peer-memory exchanges (producers
    store into every shard's buffer, flag barriers between the phases);
  * NCCL / P2P with world = 1: the real ncclCommInitRank / ncclAllGather
    calls, IPC handle export and the flag barrier on one rank.
Bar (SURVEY.md §8(e) "Determinism / parity across G"): the SpMV row sums are
the unsplit CSR rows, only the scalar sums meet across shards, so 1-vs-G
agreement of the first 50 iterates within 1e-10 relative; full solves reach
the same tolerance with the planted objective within 1e-6 relative."""
import numpy as np
import pytest

from paper_2508_08062_b200 import (DistConfig, InputError, Iterate, Method, Solver,
                                   SolverConfig, SolveStatus, UnsupportedError, nccl_unique_id,
                                   problems)

pytestmark = pytest.mark.gpu


def loopback(world):
    return DistConfig(world=world, transport="loopback")


def traj_close(a, b, k, rtol):
    np.testing.assert_allclose(a.trajectory["g_norm"][:k], b.trajectory["g_norm"][:k], rtol=rtol)
    assert np.array_equal(a.trajectory["aa_step"][:k], b.trajectory["aa_step"][:k])


@pytest.fixture(scope="module")
def cfg1():
    p = problems.make_config(1, scale=0.05)
    with Solver(p) as s:
        tau = s.select_step_sizes(SolverConfig(reduction="tree")).tau
        ref = s.solve(SolverConfig(method=Method.AA_PDHG, m=10, toll=1e-9, max_iters=60,
                                   tau=tau, sigma=tau, reduction="tree"))
    return p, tau, ref


@pytest.mark.parametrize("transport", ["loopback", "loopback_p2p"])
@pytest.mark.parametrize("world", [1, 2, 3, 5])
def test_loopback_first_iterates_match_one_gpu(cfg1, world, transport):
    p, tau, ref = cfg1
    with Solver(p, dist=DistConfig(world=world, transport=transport)) as s:
        got = s.solve(SolverConfig(method=Method.AA_PDHG, m=10, toll=1e-9, max_iters=60,
                                   tau=tau, sigma=tau, reduction="tree"))
    assert got.result.iterations == ref.result.iterations
    traj_close(got, ref, 50, 1e-10)
    x, xr = got.result.u.x, ref.result.u.x
    assert np.linalg.norm(x - xr) <= 1e-10 * np.linalg.norm(xr)
    y, yr = got.result.u.y, ref.result.u.y
    assert np.linalg.norm(y - yr) <= 1e-10 * np.linalg.norm(yr)
    # the records are identical on every shard and complete
    assert np.array_equal(got.trajectory["k"], np.arange(got.trajectory.size))


def test_loopback_step_sizes(cfg1):
    p, tau, _ = cfg1
    with Solver(p, dist=loopback(4)) as s:
        t4 = s.select_step_sizes(SolverConfig()).tau
    assert abs(t4 - tau) <= 1e-10 * tau


def test_loopback_full_solve_config0():
    """Config 0 to toll 1e-6 on 2 shards: converges like one GPU, planted
    objective within 1e-6 relative, KKT of the final iterate small."""
    p = problems.make_config(0)
    cfg = SolverConfig(method=Method.AA_PDHG, m=5, toll=1e-6, max_iters=100000,
                       reduction="tree")
    with Solver(p) as s:
        one = s.solve(cfg)
    with Solver(p, dist=loopback(2)) as s:
        two = s.solve(cfg)
    assert one.result.status == two.result.status == SolveStatus.RESIDUAL_TOL
    # AA-PDHG is chaotic under rounding (the reference moves -18%/+8% itself)
    assert abs(two.result.iterations - one.result.iterations) <= 0.25 * one.result.iterations
    obj = p.planted_objective
    assert abs(two.result.objective - obj) <= 1e-6 * abs(obj)
    assert two.result.kkt.max() <= 1e-4
    assert two.result.g_norm < 1e-6


@pytest.mark.parametrize("transport", ["loopback", "loopback_p2p"])
def test_loopback_faa_long_rows(transport):
    """Config 2 shape (transport: K rows of 300 nnz on the long-row path),
    FAA m=10 with the BASELINE filter parameters, on 3 shards."""
    p = problems.make_config(2, scale=0.15)
    spec = problems.CONFIGS[2]
    filt = type(SolverConfig().filter)(c_s=spec["c_s"], kappa_bar=spec["kappa_bar"])
    with Solver(p) as s:
        tau = s.select_step_sizes(SolverConfig(reduction="tree")).tau
        cfg = SolverConfig(method=Method.FAA_PDHG, m=10, toll=1e-9, max_iters=40, tau=tau,
                           sigma=tau, reduction="tree", filter=filt)
        ref = s.solve(cfg)
    with Solver(p, dist=DistConfig(world=3, transport=transport)) as s:
        got = s.solve(cfg)
    traj_close(got, ref, 40, 1e-10)


@pytest.mark.parametrize("transport", ["loopback", "loopback_p2p"])
def test_loopback_pdhg_start_iterate_and_lambda(transport):
    p = problems.make_config(0, scale=0.3)
    rng = np.random.default_rng(5)
    u0 = Iterate(rng.uniform(0, 1, p.n()), rng.normal(size=p.k.nrows))
    cfg = SolverConfig(method=Method.PDHG, toll=1e-9, max_iters=30, tau=0.05, sigma=0.05,
                       reduction="tree")
    with Solver(p) as s:
        ref = s.solve(cfg, u0)
    with Solver(p, dist=DistConfig(world=2, transport=transport)) as s:
        got = s.solve(cfg, u0)
    traj_close(got, ref, 30, 1e-10)
    np.testing.assert_allclose(got.result.lambda_, ref.result.lambda_, rtol=1e-9, atol=1e-12)
    assert got.result.status == ref.result.status == SolveStatus.MAX_ITERS


def test_nccl_world1_matches_one_gpu(cfg1):
    """The NCCL transport with one rank: the real NCCL calls (the per-shard
    totals are summed in another fixed order than the single-GPU fused
    control, so agreement is to rounding)."""
    p, tau, ref = cfg1
    nid = nccl_unique_id()
    assert len(nid) == 128
    with Solver(p, dist=DistConfig(world=1, rank=0, transport="nccl", nccl_id=nid)) as s:
        got = s.solve(SolverConfig(method=Method.AA_PDHG, m=10, toll=1e-9, max_iters=60,
                                   tau=tau, sigma=tau, reduction="tree"))
    assert got.result.iterations == ref.result.iterations
    traj_close(got, ref, 60, 1e-10)
    x, xr = got.result.u.x, ref.result.u.x
    assert np.linalg.norm(x - xr) <= 1e-10 * np.linalg.norm(xr)


def test_p2p_world1_matches_one_gpu(cfg1):
    """The P2P transport with one rank: NCCL setup, IPC handle export, the
    producers' peer-store path and the system-scope flag barriers."""
    p, tau, ref = cfg1
    nid = nccl_unique_id()
    with Solver(p, dist=DistConfig(world=1, rank=0, transport="p2p", nccl_id=nid)) as s:
        cfg = SolverConfig(method=Method.AA_PDHG, m=10, toll=1e-9, max_iters=60, tau=tau,
                           sigma=tau, reduction="tree")
        got = s.solve(cfg)
        again = s.solve(cfg)  # a second solve: the next barrier epoch
    for out in (got, again):
        assert out.result.iterations == ref.result.iterations
        traj_close(out, ref, 60, 1e-10)
    assert np.array_equal(got.result.u.x, again.result.u.x)


def test_loopback_p2p_repeated_solves_and_aa_branch(cfg1):
    """Peer-memory exchanges across solves (barrier epochs) and through many
    AA steps (the DOTS / candidate-x exchanges): 4 shards, 300 iterations,
    against the copy transport."""
    p, tau, _ = cfg1
    cfg = SolverConfig(method=Method.AA_PDHG, m=10, toll=1e-12, max_iters=300, tau=tau,
                       sigma=tau, reduction="tree")
    with Solver(p, dist=DistConfig(world=4, transport="loopback")) as s:
        ref = s.solve(cfg)
    with Solver(p, dist=DistConfig(world=4, transport="loopback_p2p")) as s:
        a = s.solve(cfg)
        b = s.solve(cfg)
    assert ref.result.i > 5  # AA steps taken
    for out in (a, b):
        assert np.array_equal(out.trajectory["g_norm"], ref.trajectory["g_norm"])
        assert np.array_equal(out.result.u.x, ref.result.u.x)
        assert np.array_equal(out.result.u.y, ref.result.u.y)


def test_dist_errors():
    p = problems.toy()
    with pytest.raises(UnsupportedError):
        Solver(p, dist=loopback(p.k.nrows + 1))
    with pytest.raises(InputError):
        Solver(p, dist=DistConfig(world=2, rank=0, transport="nccl"))  # no id
    with pytest.raises(InputError):
        Solver(p, dist=DistConfig(world=1, transport="smoke-signals"))
    with pytest.raises(InputError):
        Solver(p, dist=DistConfig(world=1, rank=0, transport="p2p"))  # no id
    big = problems.make_config(0, scale=0.2)
    with pytest.raises(UnsupportedError):
        Solver(big, dist=DistConfig(world=9, transport="loopback_p2p"))
    q = problems.make_config(0, scale=0.2)
    with Solver(q, dist=loopback(2)) as s:
        with pytest.raises(UnsupportedError):
            s.pdhg_step(Iterate(np.zeros(q.n()), np.zeros(q.k.nrows)),
                        type(s.select_step_sizes(SolverConfig()))(0.1, 0.1))
        with pytest.raises(InputError):
            s.solve(SolverConfig(m=0, method=Method.AA_PDHG))


def test_loopback_with_l2_column_blocking(cfg1, monkeypatch):
    """Shards also split their K / K' blocks into L2 column passes when the
    gathered vector is large (forced here): same first iterates."""
    p, tau, ref = cfg1
    monkeypatch.setenv("AAPDHG_L2_BLOCK_MIN_KB", "0")
    monkeypatch.setenv("AAPDHG_L2_BLOCK_KB", "16")
    with Solver(p, dist=loopback(3)) as s:
        got = s.solve(SolverConfig(method=Method.AA_PDHG, m=10, toll=1e-9, max_iters=60,
                                   tau=tau, sigma=tau, reduction="tree"))
    traj_close(got, ref, 50, 1e-10)


def test_loopback_inequality_rows_and_general_bounds():
    """Inequality rows (m1 > 0) split across shards (each shard projects its
    own leading block of them) and general bounds: free, negative lower and
    finite upper — the lambda set and bound terms of kkt_metrics."""
    from paper_2508_08062_b200 import ProblemData
    base = problems.make_config(0, scale=0.3)
    rng = np.random.default_rng(3)
    n = base.n()
    l = np.where(rng.random(n) < 0.3, -np.inf, np.where(rng.random(n) < 0.5, -1.0, 0.0))
    u = np.where(rng.random(n) < 0.4, 2.0, np.inf)
    p = ProblemData(base.k, base.k.nrows // 2 + 7, base.c, base.q, l, u, name="mixed")
    cfg = SolverConfig(method=Method.AA_PDHG, m=5, toll=1e-9, max_iters=60, tau=0.05, sigma=0.05,
                       reduction="tree")
    with Solver(p) as s:
        ref = s.solve(cfg)
    for world in (2, 3):
        with Solver(p, dist=loopback(world)) as s:
            got = s.solve(cfg)
        traj_close(got, ref, 50, 1e-10)
        for f in ("r_gap", "r_primal", "r_dual"):
            np.testing.assert_allclose(got.trajectory[f][:50], ref.trajectory[f][:50], rtol=1e-9,
                                       atol=1e-14)
        np.testing.assert_allclose(got.result.lambda_, ref.result.lambda_, rtol=1e-8, atol=1e-12)


@pytest.mark.parametrize("transport", ["loopback", "loopback_p2p"])
def test_loopback_setcover_faa(transport):
    """The reference's set-cover generator (all rows inequalities, finite
    upper bounds), FAA with its default filter, on 3 shards."""
    from golden_io import problem
    p = problem("setcover")
    cfg = SolverConfig(method=Method.FAA_PDHG, m=5, toll=1e-9, max_iters=60, tau=0.1, sigma=0.1,
                       reduction="tree")
    with Solver(p) as s:
        ref = s.solve(cfg)
    with Solver(p, dist=DistConfig(world=3, transport=transport)) as s:
        got = s.solve(cfg)
    traj_close(got, ref, 40, 1e-10)
