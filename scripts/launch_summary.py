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
col = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Grid Size", "Metric Name", "Metric Unit",
                                  "Metric Value")}
UNIT = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
        "second": 1e3, "s": 1e3,
        "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
per = defaultdict(dict)
meta = {}
for r in rows[start + 1:]:
    if len(r) < len(hdr):
        continue
    i = r[col["ID"]]
    name = re.sub(r"\(.*$", "", r[col["Kernel Name"]]).replace("void ", "").replace("unnamed>::", "")
    name = re.sub(r"^\(anonymous namespace\)::|hw::|^<", "", name).strip()
    meta[i] = (name, r[col["Grid Size"]])
    per[i][r[col["Metric Name"]]] = (float(r[col["Metric Value"]].replace(",", ""))
                                     * UNIT.get(r[col["Metric Unit"]], 1.0))
agg = defaultdict(lambda: [0, 0.0, 0.0])
for i, m in per.items():
    a = agg[meta[i]]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0.0)          # ms
    a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
total = sum(v[1] for v in agg.values())
w = csv.writer(sys.stdout)
w.writerow(["kernel", "grid", "launches", "total_ms", "share_pct", "avg_us", "dram_GBs"])
for (name, grid), (n, ms, by) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    w.writerow([name, grid, n, f"{ms:.2f}", f"{100 * ms / total:.2f}", f"{1e3 * ms / n:.1f}",
                f"{by / (ms / 1e3) / 1e9:.0f}" if by else ""])
