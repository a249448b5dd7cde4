"""Static SASS opcode counts per source line of one kernel (nvdisasm -g on
the in-tree library's cubin), e.g. to spot register moves around a branch:
  python tools/sass_lines.py fused _ZN4diaq16tile_pass_kernelILi4ELi1EEEvNS_10TileParamsE 226 388
"""
import os
import re
import subprocess
import sys
import tempfile
from collections import Counter, defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(unit, kernel, lines):
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(ROOT, "paper_2405_01250_b200", "libdiaq_b200.so")],
                       cwd=d, check=True, capture_output=True)
        txt = subprocess.run(["nvdisasm", "-g", os.path.join(d, f"{unit}.sm_100a.cubin")], check=True,
                             capture_output=True, text=True).stdout.split("\n")
    start = end = None
    for i, l in enumerate(txt):
        if l.startswith(f".text.{kernel}:"):
            start = i
        elif start is not None and l.startswith("//---------------------") and i > start + 5:
            end = i
            break
    ops = defaultdict(Counter)
    tot = Counter()
    cur = None
    for l in txt[start:end]:
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", l)
        if m:
            op = m.group(2).split(".")[0]
            tot[op] += 1
            if cur:
                ops[cur][op] += 1
    print("kernel total", sum(tot.values()), tot.most_common(10))
    for ln in lines:
        for key in ops:
            if key[1] == ln:
                print(key, sum(ops[key].values()), ops[key].most_common(8))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], [int(a) for a in sys.argv[3:]])
