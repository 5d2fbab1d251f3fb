"""Builds profiles/r02b/traffic.json (the DRAM bytes bench.py reports as
roofline.traffic) from the committed ncu --set full raw pages of
profiles/ncu_r02b.sh: dram__bytes_read.sum + dram__bytes_write.sum per launch,
cold caches (ncu flushes between replays).
  python profiles/make_traffic.py"""
import csv
import json
from pathlib import Path

D = Path(__file__).resolve().parent / "r02b"


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
