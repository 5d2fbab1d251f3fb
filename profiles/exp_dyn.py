"""Experiment (not a benchmark; needs profiles/microbench/dyn_slices.patch applied): k_plain_loop with the dynamic slice
distribution (AAPDHG_DYN=1, per-slice partials) against the static one-slice-
per-warp layout (=0) on configs[1]: us/iteration over 3,000 / 20,000
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
    flag = os.environ.get("AAPDHG_DYN")
    with Solver(p) as s:
        for meth, iters in ((Method.PDHG, 3000), (Method.AA_PDHG, 3000), (Method.AA_PDHG, 20000)):
            cfg = SolverConfig(method=meth, m=10, toll=1e-12, max_iters=iters, tau=0.0775,
                               sigma=0.0775, reduction="tree")
            s.solve(cfg)
            t = time.perf_counter()
            o = s.solve(cfg)
            dt = time.perf_counter() - t
            print(f"DYN={flag} {meth.name:8s} {iters:6d} its {1e6 * dt / o.result.iterations:7.2f} "
                  f"us/it  AA steps {o.result.i}  |g| {o.result.g_norm:.6e}", flush=True)
            np.save(f"/tmp/dyn_{flag}_{meth.name}_{iters}.npy", o.trajectory["g_norm"])
    sys.exit(0)
for flag in ("0", "1"):
    subprocess.run([sys.executable, __file__, "child"], env=dict(os.environ, AAPDHG_DYN=flag),
                   check=True)
import numpy as np  # noqa: E402

for tag in ("PDHG_3000", "AA_PDHG_3000", "AA_PDHG_20000"):
    a, b = np.load(f"/tmp/dyn_0_{tag}.npy"), np.load(f"/tmp/dyn_1_{tag}.npy")
    print(f"{tag}: first-50 max rel |g| diff {np.max(np.abs(a[:50] - b[:50]) / np.abs(a[:50])):.3e}")
