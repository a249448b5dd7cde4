"""Aggregate an ncu source page (--print-source cuda,sass csv) per source line:
stall samples and executed instructions, top N."""
import csv
import sys
from collections import defaultdict


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    cur = None
    hdr = None
    agg = defaultdict(lambda: [0, 0])
    text = {}
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 8 or not r[0]:
            continue
        try:
            ln = int(r[0])
        except ValueError:
            continue
        key = (cur, ln)
        text[key] = r[1]
        try:
            agg[key][0] += int(r[4] or 0)
            agg[key][1] += int(r[7] or 0)
        except ValueError:
            pass
    tot = sum(v[0] for v in agg.values()) or 1
    itot = sum(v[1] for v in agg.values()) or 1
    print(f"samples {tot}  warp-instructions {itot}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{k[0]}:{k[1]:4d} {100 * v[0] / tot:5.1f}% inst {100 * v[1] / itot:5.1f}%  {text[k].strip()[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
