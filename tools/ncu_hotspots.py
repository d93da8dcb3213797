"""Summarise an `ncu --page source --csv --print-source sass` export: stall
samples per opcode and the hottest SASS lines of the first kernel instance.

    ncu -i rep.ncu-rep --page source --csv --print-source sass -k regex:NAME > src.csv
    python tools/ncu_hotspots.py src.csv [N]
"""
import csv
import sys
from collections import Counter


def main(path: str, top: int = 30) -> None:
    rows = list(csv.reader(open(path)))
    hdr = [i for i, r in enumerate(rows) if r[:2] == ["Address", "Source"]]
    start = hdr[0]
    end = hdr[1] - 1 if len(hdr) > 1 else len(rows)
    h = rows[start]
    si, wi, ei = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    stall_cols = [(i, c) for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    by_op, ex_op, reasons = Counter(), Counter(), Counter()
    lines = []
    tot = 0
    for r in rows[start + 1:end]:
        if len(r) <= ei or not r[wi].isdigit():
            continue
        s = r[si].strip()
        w, e = int(r[wi] or 0), int(r[ei] or 0)
        t = s.split()
        op = (t[1] if t and t[0].startswith("@") and len(t) > 1 else (t[0] if t else "")).split(".")[0]
        by_op[op] += w
        ex_op[op] += e
        tot += w
        for i, c in stall_cols:
            if r[i].isdigit():
                reasons[c] += int(r[i])
        lines.append((w, e, s))
    print(f"samples {tot}  instructions {sum(ex_op.values())}")
    print("stall reasons:", ", ".join(f"{k[6:]} {v / max(tot, 1) * 100:.1f}%" for k, v in reasons.most_common(8)))
    for op, c in by_op.most_common(20):
        print(f"  {op:10s} stall {c / max(tot, 1) * 100:5.1f}%  executed {ex_op[op]}")
    for w, e, s in sorted(lines, reverse=True)[:top]:
        print(f"  {w:6d} {e:10d}  {s[:100]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
