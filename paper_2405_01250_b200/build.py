"""Build the in-tree CUDA library libdiaq_b200.so for sm_100a with nvcc.

`python -m paper_2405_01250_b200.build` (or __graft_entry__.build()).  The
.so is written next to this file so it travels with the repo snapshot.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libdiaq_b200.so")
ROOT = os.path.dirname(HERE)

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "--compiler-options", "-fPIC,-O2",
    "-Xptxas", "-v",
    "-fmad=false",
]


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "diaq_b200.h")]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    cmd = [nvcc, *NVCC_FLAGS, "-shared", "-o", LIB + ".tmp", *sources(),
           "-I", os.path.join(ROOT, "include"), "-lcudart_static", "-lrt", "-ldl", "-lpthread"]
    env = dict(os.environ)
    env.setdefault("CC", "/usr/bin/gcc")
    proc = subprocess.run(cmd, capture_output=True, text=True, env=env,
                          **({"cwd": ROOT}))
    if proc.returncode != 0:
        sys.stderr.write(proc.stdout + proc.stderr)
        raise RuntimeError("nvcc build of libdiaq_b200.so failed")
    if verbose:
        sys.stderr.write(proc.stderr)
    os.replace(LIB + ".tmp", LIB)
    with open(os.path.join(HERE, "ptxas.log"), "w") as f:
        f.write(proc.stderr)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
