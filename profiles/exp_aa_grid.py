"""Experiment (not a benchmark; needs profiles/microbench/aa_grid.patch applied): the AA branch inside k_plain_loop
(AAPDHG_AA_GRID=1, persist.cuh) against the graph's IF branch (=0) on
configs[1]: us/iteration of AA-PDHG and FAA-PDHG (m=10) over 3,000 / 20,000
iterations and the trajectory difference."""
import os
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, str(ROOT))
    import numpy as np

    from paper_2508_08062_b200 import Method, Solver, SolverConfig, problems
    p = problems.make_config(1)
    flag = os.environ.get("AAPDHG_AA_GRID")
    with Solver(p) as s:
        for meth, iters in ((Method.PDHG, 3000), (Method.AA_PDHG, 3000), (Method.AA_PDHG, 20000), (Method.FAA_PDHG, 3000)):
            cfg = SolverConfig(method=meth, m=10, toll=1e-12, max_iters=iters, tau=0.0775,
                               sigma=0.0775, reduction="tree")
            s.solve(cfg)
            t = time.perf_counter()
            o = s.solve(cfg)
            dt = time.perf_counter() - t
            print(f"AA_GRID={flag} {meth.name:8s} {iters:6d} its {1e6 * dt / o.result.iterations:7.2f} "
                  f"us/it  AA steps {o.result.i}  failures {o.result.aa_failures}  "
                  f"|g| {o.result.g_norm:.6e}", flush=True)
            np.save(f"/tmp/aag_{flag}_{meth.name}_{iters}.npy",
                    np.stack([o.trajectory["g_norm"], o.trajectory["aa_step"].astype(float)]))
    sys.exit(0)
for flag in ("0", "1"):
    subprocess.run([sys.executable, __file__, "child"], env=dict(os.environ, AAPDHG_AA_GRID=flag),
                   check=True)
import numpy as np  # noqa: E402

for tag in ("AA_PDHG_3000", "AA_PDHG_20000", "FAA_PDHG_3000"):
    a, b = np.load(f"/tmp/aag_0_{tag}.npy"), np.load(f"/tmp/aag_1_{tag}.npy")
    n = min(a.shape[1], b.shape[1])
    r50 = np.max(np.abs(a[0, :50] - b[0, :50]) / np.abs(a[0, :50]))
    same = int(np.sum(a[1, :n] == b[1, :n]))
    print(f"{tag}: first-50 max rel |g| diff {r50:.3e}; aa_step pattern equal on {same}/{n}")
