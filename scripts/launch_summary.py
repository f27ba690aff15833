"""Per-kernel summary of an ncu launch list (--metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum --csv): launches, total ms,
share, average us, DRAM GB/s, grouped by kernel name and grid.

    python scripts/launch_summary.py launches.csv > summary.csv
"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14 and r[0].isdigit()]
launch = collections.OrderedDict()
for r in rows:
    rec = launch.setdefault(int(r[0]), {"name": r[4], "grid": r[8]})
    rec[r[12]] = float(r[14])
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for rec in launch.values():
    name = rec["name"].replace("void ", "").replace("(anonymous namespace)::", "").replace("<unnamed>::", "").replace("unnamed>::", "")
    name = name.split("(")[0] if "<" not in name else name[: name.index(">") + 1]
    k = (name.replace("hw::", "").replace("unnamed>::", ""), rec["grid"])
    a = agg[k]
    a[0] += 1
    a[1] += rec.get("gpu__time_duration.sum", 0) / 1e6
    a[2] += rec.get("dram__bytes_read.sum", 0) + rec.get("dram__bytes_write.sum", 0)
tot = sum(v[1] for v in agg.values())
w = csv.writer(sys.stdout)
w.writerow(["kernel", "grid", "launches", "total_ms", "share_pct", "avg_us", "dram_GBs"])
for (k, g), (n, ms, by) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    w.writerow([k, g, n, f"{ms:.2f}", f"{100 * ms / tot:.2f}", f"{1e3 * ms / n:.1f}",
                f"{by / (ms / 1e3) / 1e9:.0f}" if ms else "0"])
print(f"# total {tot:.1f} ms over {len(launch)} launches", file=sys.stderr)
