"""DRAM traffic over algorithmic bytes per multigrid launch class, from an
ncu launch list (--metrics dram__bytes_read.sum,dram__bytes_write.sum,
gpu__time_duration.sum -k regex:mg2d_reg --csv) of one PCG solve.

    python scripts/traffic_summary.py gpurun_out/traffic_cfg4.csv 10 > profiles/ncu_traffic_cfg4.json

Algorithmic bytes per launch (8-byte words per temporal row, n = 2^l - 1,
m = 2^(l-1) - 1): DOWN zero start 2n^2 + m^2, DOWN 3n^2 + m^2, UP 3n^2 + m^2,
plus n^2 on the finest UP pass that fuses r.z (one of the four finest
1,025-row UP launches of every K_X application).  Classes as bench.py's
profile classes (hwg_profile_*)."""
import collections
import csv
import json
import re
import sys

path, K = sys.argv[1], int(sys.argv[2])
rows = [r for r in csv.reader(open(path)) if len(r) > 14 and r[0].isdigit()]
launch = collections.OrderedDict()
for r in rows:
    lid = int(r[0])
    rec = launch.setdefault(lid, {"name": r[4], "grid": r[8]})
    rec[r[12]] = float(r[14])
pat = re.compile(r"mg2d_reg<(\d+), (\d+), (\d), (\d), (\d), (\d), (\d)>")
classes = collections.defaultdict(lambda: {"launches": 0, "dram_bytes": 0.0, "alg_bytes": 0.0,
                                           "ms": 0.0})
n_up_fin_1025 = 0
for lid, rec in launch.items():
    m_ = pat.search(rec["name"])
    if not m_:
        continue
    P, NT, down, zs = (int(m_.group(i)) for i in (1, 2, 3, 4))
    n = P * NT - 1
    l = n.bit_length()
    m = (n - 1) // 2
    nrows = int(rec["grid"].strip("()").split(",")[0])
    finest = l == K
    if down:
        words = (2 if zs else 3) * n * n + m * m
        cls = "mg2d_down_finest" if finest else "mg2d_down_coarser"
    else:
        words = 3 * n * n + m * m
        cls = "mg2d_up_finest" if finest else "mg2d_up_coarser"
        if finest and nrows == 2 ** (K) + 1:
            n_up_fin_1025 += 1
            if n_up_fin_1025 % 4 == 0:           # the r.z-fused pass of each K_X
                words += n * n
    c = classes[cls]
    c["launches"] += 1
    c["dram_bytes"] += rec.get("dram__bytes_read.sum", 0) + rec.get("dram__bytes_write.sum", 0)
    c["alg_bytes"] += 8.0 * nrows * words
    c["ms"] += rec.get("gpu__time_duration.sum", 0) / 1e6
out = {}
for k, c in classes.items():
    out[k] = {"launches": c["launches"], "dram_bytes": c["dram_bytes"], "algorithmic_bytes": c["alg_bytes"],
              "traffic_over_algorithmic": c["dram_bytes"] / c["alg_bytes"],
              "dram_bytes_per_launch": c["dram_bytes"] / c["launches"],
              "ncu_ms": c["ms"], "ncu_GBs": c["dram_bytes"] / (c["ms"] / 1e3) / 1e9}
out["source"] = (f"{path}: ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                 "-k regex:mg2d_reg over one cfg PCG solve of the benched build (scripts/profile_solve.py); "
                 "cold-cache serialised replay")
print(json.dumps(out, indent=1))
