"""Builds profiles/<round>/traffic.json (the DRAM bytes bench.py reports as
roofline.traffic) from the committed ncu --set full raw pages of
profiles/ncu_<round>.sh: dram__bytes_read.sum + dram__bytes_write.sum per
launch, cold caches (ncu flushes between replays).
  python profiles/make_traffic.py [r02d]     (r02b: the second session's capture order)"""
import csv
import json
import sys
from pathlib import Path

RND = sys.argv[1] if len(sys.argv) > 1 else "r02d"
D = Path(__file__).resolve().parent / RND


def rows(name):
    r = list(csv.reader(open(D / name)))
    hdr, body = r[0], r[2:]
    units = r[1]
    out = []
    for row in body:
        rec = {}
        for k in ("Kernel Name", "Grid Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
                  "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct"):
            i = hdr.index(k)
            v = row[i]
            if k.startswith(("gpu__", "dram__", "lts__")):
                scale = {"ms": 1e-3, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9,
                         "ns": 1e-9, "Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0,
                         "%": 1.0}.get(units[i], 1.0)
                v = float(v.replace(",", "")) * scale
            rec[k] = v
        out.append(rec)
    return out


if RND != "r02b":
    # fourth session (profiles/ncu_r02d.sh): 2 eager AA-PDHG iterations of configs[4], every
    # k_spmv_pass / k_dual_epi / k_primal_epi launch in order. The start iterate's K x is a memset
    # (zero start), so iteration 2 = the launches after the first k_primal_epi up to and including
    # the second one: K' passes x2, then k_dual_epi per K column block with K's passes beside them,
    # then k_primal_epi.
    plain = rows(f"plain_{RND}_raw.csv")[0]
    cfg4 = rows(f"cfg4_{RND}_raw.csv")
    ends = [i for i, r in enumerate(cfg4) if "k_primal_epi" in r["Kernel Name"]]
    # (eager launches of the AA recache's passes are device-predicated no-ops outside an AA
    # step — 0 DRAM bytes, ~44 us of empty CTAs each; the graph keeps them inside the IF node)
    it = [r for r in cfg4[ends[0] + 1:ends[1] + 1]
          if r["dram__bytes_read.sum"] + r["dram__bytes_write.sum"] > 1e6]
    out = {
        "source": f"ncu --set full --clock-control none (profiles/ncu_{RND}.sh; profiles/{RND}/*_raw.csv)",
        "k_plain_loop": {
            "dram_read_bytes": plain["dram__bytes_read.sum"],
            "dram_write_bytes": plain["dram__bytes_write.sum"], "iterations": 8,
            "duration_us": plain["gpu__time_duration.sum"] * 1e6,
            "source": "profiles/profile_plain.py 24 3 (--launch-skip 360: the first launch of the solve after three calibration solves): 8 plain iterations plus the dropped speculative K1"},
        "config4_iteration": {
            "kernels": [{"kernel": r["Kernel Name"].split("(")[0], "grid": r["Grid Size"],
                         "duration_us": r["gpu__time_duration.sum"] * 1e6,
                         "dram_read_bytes": r["dram__bytes_read.sum"],
                         "dram_write_bytes": r["dram__bytes_write.sum"],
                         "lts_hit_pct": r["lts__t_sector_hit_rate.pct"]} for r in it],
            "note": "profiles/profile_cfg.py 4 1.0 2 (eager): the second iteration's launches"},
    }
    k = out["config4_iteration"]["kernels"]
    out["config4_iteration"]["dram_bytes"] = sum(x["dram_read_bytes"] + x["dram_write_bytes"] for x in k)
    out["config4_iteration"]["duration_us"] = sum(x["duration_us"] for x in k)
    json.dump(out, open(D / "traffic.json", "w"), indent=1)
    print(json.dumps(out["config4_iteration"], indent=1))
else:
    plain = rows("plain_r02b_raw.csv")[0]
    cfg4 = rows("cfg4_r02b_raw.csv")
    # launch order of the capture: the start iterate's K x (K passes b0, b1, b2),
    # then iteration 1: K' passes b0, b1, k_dual_epi, K passes b0, b1 (-c 8). One
    # plain iteration = K' b0 + b1 + k_dual_epi + K b0 + b1 + b2 + b3 + k_primal_epi:
    # K b2 / b3 are the start's b1 / b2 (the same block shapes, partials read and
    # written), k_primal_epi comes from the metrics pass cfg4_split_ncu.csv.
    it = [cfg4[3], cfg4[4], cfg4[5], cfg4[6], cfg4[7], cfg4[1], cfg4[2]]
    mcsv = list(csv.reader(l for l in open(D / "cfg4_split_ncu.csv") if not l.startswith("==")))
    mh = mcsv[0]
    pe = {}
    for r in mcsv[1:]:
        if "k_primal_epi" in r[mh.index("Kernel Name")] and r[mh.index("ID")] == "10":
            pe[r[mh.index("Metric Name")]] = float(r[mh.index("Metric Value")].replace(",", ""))
    it.append({"Kernel Name": "k_primal_epi", "Grid Size": "(888, 1, 1)",
               "gpu__time_duration.sum": pe["gpu__time_duration.sum"] * 1e-9,
               "dram__bytes_read.sum": pe["dram__bytes_read.sum"],
               "dram__bytes_write.sum": pe["dram__bytes_write.sum"],
               "lts__t_sector_hit_rate.pct": pe["lts__t_sector_hit_rate.pct"]})
    out = {
        "source": "ncu --set full --clock-control none (profiles/ncu_r02b.sh; profiles/r02b/*_raw.csv)",
        "k_plain_loop": {
            "dram_read_bytes": plain["dram__bytes_read.sum"],
            "dram_write_bytes": plain["dram__bytes_write.sum"], "iterations": 8,
            "duration_us": plain["gpu__time_duration.sum"] * 1e6,
            "source": "profiles/profile_plain.py 24 3 (--launch-skip 360: the first launch of the solve after three calibration solves): 8 plain iterations plus the dropped speculative K1"},
        "config4_iteration": {
            "kernels": [{"kernel": r["Kernel Name"].split("(")[0], "grid": r["Grid Size"],
                         "duration_us": r["gpu__time_duration.sum"] * 1e6,
                         "dram_read_bytes": r["dram__bytes_read.sum"],
                         "dram_write_bytes": r["dram__bytes_write.sum"],
                         "lts_hit_pct": r["lts__t_sector_hit_rate.pct"]} for r in it],
            "note": "profiles/profile_cfg.py 4 1.0 2 (eager); see the launch-order comment in "
                    "profiles/make_traffic.py"},
    }
    k = out["config4_iteration"]["kernels"]
    out["config4_iteration"]["dram_bytes"] = sum(x["dram_read_bytes"] + x["dram_write_bytes"] for x in k)
    out["config4_iteration"]["duration_us"] = sum(x["duration_us"] for x in k)
    json.dump(out, open(D / "traffic.json", "w"), indent=1)
    print(json.dumps(out["config4_iteration"], indent=1))
