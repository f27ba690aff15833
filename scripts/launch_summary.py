"""Per-kernel summary of an ncu launch list (--metrics gpu__time_duration.sum
[,dram__bytes_read.sum,dram__bytes_write.sum] --csv): launches, total ms,
share of the GPU time, average us, and DRAM GB/s when the bytes were captured.

    python scripts/launch_summary.py gpurun_out/launches.csv > profiles/rNN/summary.csv
"""
import csv
import re
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
col = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Grid Size", "Metric Name", "Metric Value")}
per = defaultdict(dict)
meta = {}
for r in rows[start + 1:]:
    if len(r) < len(hdr):
        continue
    i = r[col["ID"]]
    name = re.sub(r"\(.*$", "", r[col["Kernel Name"]]).replace("void ", "").replace("unnamed>::", "")
    name = re.sub(r"^\(anonymous namespace\)::|hw::|^<", "", name).strip()
    meta[i] = (name, r[col["Grid Size"]])
    per[i][r[col["Metric Name"]]] = float(r[col["Metric Value"]].replace(",", ""))
agg = defaultdict(lambda: [0, 0.0, 0.0])
for i, m in per.items():
    t = m.get("gpu__time_duration.sum", 0.0)
    scale = 1e-6 if t > 1e4 else 1e-3       # ns or us
    a = agg[meta[i]]
    a[0] += 1
    a[1] += t * scale
    a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
total = sum(v[1] for v in agg.values())
w = csv.writer(sys.stdout)
w.writerow(["kernel", "grid", "launches", "total_ms", "share_pct", "avg_us", "dram_GBs"])
for (name, grid), (n, ms, by) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    w.writerow([name, grid, n, f"{ms:.2f}", f"{100 * ms / total:.2f}", f"{1e3 * ms / n:.1f}",
                f"{by / (ms / 1e3) / 1e9:.0f}" if by else ""])
