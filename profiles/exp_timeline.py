"""Experiment (not a benchmark): kernel entry timeline of a configs[1] solve
(EXTRA=-DAAPDHG_TIMELINE build: CTA 0 of each kernel stamps its id and the
globaltimer on entry; k_plain_loop's control CTA stamps its exit). Prints the
20-iteration solve the driver's bench times, then averages over a 3,000
iteration solve: the AA branch kernels and the gaps around them."""
import ctypes as C
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2508_08062_b200 import Method, Solver, SolverConfig, problems  # noqa: E402

NAMES = {1: "k_plain_loop", 2: "  (plain loop control exit)", 10: "k_gram_dots",
         11: "k_gram_dots_dd", 12: "k_aa_solve", 13: "k_mix", 14: "k_spmv", 15: "k_spmv_commit",
         16: "k_dual_side", 17: "k_primal_side", 18: "k_stage_g", 19: "k_tree_dots",
         20: "k_spmv_pass", 21: "k_aa_commit", 22: "k_project_start",
         23: "  (k_aa_solve exit)", 24: "  (k_aa_solve partials reduced)", 25: "  (k_aa_solve Cholesky done)"}
p = problems.make_config(1)
buf = (C.c_double * (2 * 8192))()
with Solver(p) as s:
    tau = 0.0775
    cfg = lambda it: SolverConfig(method=Method.AA_PDHG, m=10, toll=1e-12, max_iters=it,  # noqa
                                  tau=tau, sigma=tau, reduction="tree")
    for _ in range(4):
        s.solve(cfg(300))
    s.lib.aapdhg_cuda_timeline(buf, 8192)
    out = s.solve(cfg(20))
    n = s.lib.aapdhg_cuda_timeline(buf, 8192)
    ev = [(int(buf[2 * i]), buf[2 * i + 1]) for i in range(n)]
    ev.sort(key=lambda e: e[1])
    t0 = ev[0][1]
    print(f"20-iteration solve: {out.result.iterations} iterations, {out.result.i} AA steps, "
          f"{n} kernel entries, first -> last entry {(ev[-1][1] - t0) / 1e3:.1f} us")
    for k, (i, t) in enumerate(ev):
        nxt = ev[k + 1][1] if k + 1 < n else t
        print(f"  {(t - t0) / 1e3:9.2f} us  +{(nxt - t) / 1e3:7.2f}  {NAMES.get(i, i)}")
    out = s.solve(cfg(3000))
    n = s.lib.aapdhg_cuda_timeline(buf, 8192)
    ev = sorted(((int(buf[2 * i]), buf[2 * i + 1]) for i in range(n)), key=lambda e: e[1])
    d = defaultdict(list)
    for k in range(len(ev) - 1):
        d[(ev[k][0], ev[k + 1][0])].append(ev[k + 1][1] - ev[k][1])
    print(f"3000-iteration solve: {out.result.i} AA steps, {n} entries (8192 kept)")
    for (a, b), v in sorted(d.items(), key=lambda kv: -len(kv[1])):
        print(f"  {NAMES.get(a, a):28s} -> {NAMES.get(b, b):28s} n={len(v):5d} "
              f"mean {sum(v) / len(v) / 1e3:8.2f} us")
