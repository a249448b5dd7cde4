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
    env = dict(os.environ)
    env.setdefault("CC", "/usr/bin/gcc")
    objdir = os.path.join(ROOT, "build", "obj")
    os.makedirs(objdir, exist_ok=True)

    def compile_one(src: str):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [nvcc, *NVCC_FLAGS, "-c", "-o", obj, src, "-I", os.path.join(ROOT, "include")]
        return obj, subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=ROOT)

    # one nvcc per translation unit, in parallel (fused.cu dominates)
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=max(1, min(len(sources()), os.cpu_count() or 1))) as ex:
        results = list(ex.map(compile_one, sources()))
    log = "".join(p.stdout + p.stderr for _, p in results)
    if any(p.returncode != 0 for _, p in results):
        sys.stderr.write(log)
        raise RuntimeError("nvcc build of libdiaq_b200.so failed")
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB + ".tmp",
           *[o for o, _ in results], "-lcudart_static", "-lrt", "-ldl", "-lpthread"]
    proc = subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=ROOT)
    if proc.returncode != 0:
        sys.stderr.write(proc.stdout + proc.stderr)
        raise RuntimeError("nvcc link of libdiaq_b200.so failed")
    if verbose:
        sys.stderr.write(log)
    os.replace(LIB + ".tmp", LIB)
    with open(os.path.join(HERE, "ptxas.log"), "w") as f:
        f.write(log)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
