"""Per-kernel averages from an `ncu --metrics ... --csv --log-file` launch list."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
agg = defaultdict(lambda: defaultdict(list))
for r in rows[hi + 1:]:
    if len(r) > vi:
        agg[r[ki].split("(")[0][:34]][r[mi]].append(float(r[vi].replace(",", "")))
tot = sum(sum(v["gpu__time_duration.sum"]) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]["gpu__time_duration.sum"])):
    t = v["gpu__time_duration.sum"]
    n = len(t)
    line = f"{k:34s} n={n:3d} us={sum(t) / n / 1e3:8.1f} share={sum(t) / tot * 100:5.1f}%"
    for m, lab, sc in (("dram__bytes_read.sum", "rdMB", 1e6), ("dram__bytes_write.sum", "wrMB", 1e6),
                       ("sm__inst_issued.avg.pct_of_peak_sustained_active", "issue%", 1),
                       ("smsp__inst_executed.sum", "Minst", 1e6)):
        if v.get(m):
            line += f" {lab}={sum(v[m]) / n / sc:8.1f}"
    print(line)
