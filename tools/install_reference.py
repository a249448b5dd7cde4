#!/usr/bin/env python3
"""Install the UNMODIFIED reference package into baseline/_ref (git-ignored;
it travels to the GPU box with the snapshot) together with a copy of its
own unit-test suite and fixtures, for
  * bench.py's numpy-reference secondary (the real reference timed on the
    box's host cores), and
  * tests/test_gpu_reference_suite.py (the reference's tests run against
    paper_2405_01250_b200 aliased as `diaqsim`).
Run here (the reference tree only exists in this container):
  python tools/install_reference.py
The build runs from a /tmp copy (the reference tree is read-only)."""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/pkg"
DEST = os.path.join(ROOT, "baseline", "_ref")


def main() -> int:
    if not os.path.isdir(REF):
        print(f"{REF} not present: nothing to install", file=sys.stderr)
        return 1
    with tempfile.TemporaryDirectory() as tmp:
        src = os.path.join(tmp, "pkg")
        shutil.copytree(REF, src, ignore=shutil.ignore_patterns("frontend", "demos", "__pycache__"))
        shutil.rmtree(DEST, ignore_errors=True)
        cmd = [sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation", "--no-deps",
               "--find-links", "/opt/wheelhouse", "--target", DEST, src]
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            print(p.stdout[-2000:] + p.stderr[-2000:], file=sys.stderr)
            return p.returncode
    shutil.copytree(os.path.join(REF, "tests"), os.path.join(DEST, "tests"),
                    ignore=shutil.ignore_patterns("__pycache__"))
    print(f"installed diaqsim + its tests into {DEST}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
