"""Per-function totals (instructions, stall samples, active lanes) from
`ncu --page source --csv --print-source cuda,sass` of one kernel, mapping
each CUDA source line to the enclosing function of the given source file.

    python tools/ncu_funcs.py src.csv path/to/kernel.cu
"""
import csv
import re
import sys
from collections import defaultdict


def main(csv_path, src_path):
    src = open(src_path).read().splitlines()
    starts = []
    for i, line in enumerate(src, 1):
        m = re.match(r"^(?:__device__|__global__|static|extern)[^;]*?\b(\w+)\s*\(", line)
        if m and not line.strip().endswith(";"):
            starts.append((i, m.group(1)))

    def owner(ln):
        name = "?"
        for s, n in starts:
            if s <= ln:
                name = n
        return name

    rows = list(csv.reader(open(csv_path)))
    hdr = next(i for i, r in enumerate(rows) if r[:2] == ["Line No", "Source"])
    h = rows[hdr]
    ei, ti = h.index("Instructions Executed"), h.index("Thread Instructions Executed")
    wi = h.index("Warp Stall Sampling (All Samples)")
    agg = defaultdict(lambda: [0, 0, 0])
    cur = None
    for r in rows[hdr + 1:]:
        if r[:2] == ["Line No", "Source"]:
            break
        if r and r[0].strip().isdigit():
            cur = int(r[0])
            continue
        if cur and len(r) > ei and r[ei].strip().isdigit():
            a = agg[owner(cur)]
            a[0] += int(r[ei])
            a[1] += int(r[ti]) if r[ti].strip().isdigit() else 0
            a[2] += int(r[wi]) if r[wi].strip().isdigit() else 0
    tot = sum(v[0] for v in agg.values())
    tw = sum(v[2] for v in agg.values())
    print(f"warp instructions {tot}, stall samples {tw}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"{k:28s} inst {v[0] / tot * 100:5.1f}%  stall {v[2] / max(tw, 1) * 100:5.1f}%  "
              f"lanes {v[1] / max(v[0], 1):4.1f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
