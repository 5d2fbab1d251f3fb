"""configs[1] (100k x 200k, AA-PDHG m=10) to max KKT <= 1e-6: the
reference's own iteration-count envelope (test infrastructure).

The arms are runs of the unmodified reference (oracle/_ref and its rounding
variants) made by profiles/exp_config1_kkt.py, ~45 min each on one core:
  ref, ref-fast, ref-assoc          profiles/r01/config1_kkt.jsonl
  ref@+1, ref@-1, ref@+2, ref@-2    profiles/r02/config1_kkt_envelope_tau_ulps.jsonl
                                    (the strict build at tau shifted by 1-2 ulp)
AA-PDHG is chaotic under rounding: a last-bit change of tau alone moves the
reference's count from 32,566 to 35,588. This script collects those lines
into tests/golden/config1_envelope.json for tests/test_gpu_parity.py."""
import json
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
arms = {}
for f in ("profiles/r01/config1_kkt.jsonl", "profiles/r02/config1_kkt_envelope_tau_ulps.jsonl"):
    for line in (ROOT / f).read_text().splitlines():
        d = json.loads(line)
        if d["arm"].startswith("ref"):
            arms[d["arm"]] = {k: d[k] for k in ("iterations", "aa_steps", "objective", "kkt", "tau")}
its = [a["iterations"] for a in arms.values()]
out = {"arms": arms, "envelope": [min(its), max(its)]}
(Path(__file__).resolve().parent / "config1_envelope.json").write_text(json.dumps(out, indent=1))
print(out["envelope"], {k: v["iterations"] for k, v in arms.items()})
