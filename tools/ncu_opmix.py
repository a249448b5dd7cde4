"""Dynamic opcode mix of one kernel from an ncu source page
(`ncu -i rep --page source --csv --print-source cuda,sass`), per unit of
work.  SASS rows are de-duplicated by address: an inlined instruction is
listed once under every source file it maps to.
  python tools/ncu_opmix.py src.csv UNITS [top]
"""
import csv
import sys
from collections import Counter


def main(path, units, top=30):
    rows = list(csv.reader(open(path)))
    hdr = None
    seen = set()
    ops = Counter()
    for r in rows:
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr and len(r) > 8 and r[0] == "" and r[2].startswith("0x"):
            if r[2] in seen:
                continue
            seen.add(r[2])
            op = r[3].strip().split()
            o = op[1] if op[0].startswith("@") else op[0]
            ops[o.split(".")[0]] += int(r[7] or 0)
    tot = sum(ops.values())
    print(f"warp-instructions {tot}  per unit x32: {tot * 32 / units:.1f}")
    for k, v in ops.most_common(top):
        print(f"  {k:10s} {v * 32 / units:8.2f}")


if __name__ == "__main__":
    main(sys.argv[1], float(eval(sys.argv[2])), int(sys.argv[3]) if len(sys.argv) > 3 else 30)
