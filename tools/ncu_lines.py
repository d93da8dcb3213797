"""Per-CUDA-source-line totals from `ncu --page source --csv --print-source cuda,sass`.

    python tools/ncu_lines.py src_mix.csv [N]
"""
import csv
import sys
from collections import defaultdict


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if r[:2] == ["Line No", "Source"])
    h = rows[hdr_i]
    ei = h.index("Instructions Executed")
    ti = h.index("Thread Instructions Executed")
    wi = h.index("Warp Stall Sampling (All Samples)")
    cur = None
    text = {}
    agg = defaultdict(lambda: [0, 0, 0])
    for r in rows[hdr_i + 1:]:
        if len(r) < 4:
            continue
        if r[0] == "Line No":
            break  # next function's table
        if r[0].strip().isdigit():
            cur = int(r[0])
            text[cur] = r[1].strip()
        if cur is None or not r[ei].strip().isdigit():
            continue
        agg[cur][0] += int(r[ei])
        agg[cur][1] += int(r[ti]) if r[ti].strip().isdigit() else 0
        agg[cur][2] += int(r[wi]) if r[wi].strip().isdigit() else 0
    tot = sum(v[0] for v in agg.values())
    tots = sum(v[2] for v in agg.values())
    print(f"warp instructions {tot}, stall samples {tots}")
    for ln, (e, t, w) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{ln:5d} inst {e / tot * 100:5.1f}%  stall {w / max(tots, 1) * 100:5.1f}%  lanes {t / max(e, 1):4.1f}  {text.get(ln, '')[:70]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
