"""GPU: the reference's OWN unit tests run against the drop-in.

`baseline/_ref/tests` is the reference's test directory, installed next to
the unmodified reference package by tools/install_reference.py (git-ignored;
it travels to the GPU box).  The plugin tests/_diaqsim_alias.py maps
`diaqsim` -> paper_2405_01250_b200, so every assertion of test_matrix.py,
test_gates.py, test_sim.py, test_acceptance.py, test_analysis.py and
test_memory.py runs on our device path.

Deselected, with the reason:
  * test_qasm.py, test_cli.py: the QASM front end and the run/bench/analyze/
    gen CLI are out of scope; our cli.py implements the
    `kernel` JSON protocol only (checked in tests/test_cli_protocol.py);
  * test_perf.py and tests marked `perf`: indicative CPU timings (the
    reference's own default run excludes them, pyproject addopts);
  * the one known-red reference test (194 pass, 1
    known-red on the reference itself) -- see KNOWN_RED.
"""
from __future__ import annotations

import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

REF_TESTS = os.path.join(ROOT, "baseline", "_ref", "tests")
SUITES = ["test_matrix.py", "test_gates.py", "test_sim.py", "test_acceptance.py", "test_analysis.py",
          "test_memory.py"]
# fails identically on the unmodified reference ("1
# known-red"): its GHZ memory-ordering claim (diaq < csr bytes) is false for
# the reference's own byte model -- same numbers here (diaq=952 csr=904 at
# q=4 t=2)
KNOWN_RED: list[str] = ["tests/test_acceptance.py::test_memory_format_ordering"]


@pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="baseline/_ref not installed (tools/install_reference.py)")
def test_reference_unit_suite_on_device():
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(ROOT, "tests"), ROOT, env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "_diaqsim_alias", "-p", "no:cacheprovider", "-m", "not perf",
           "-o", "addopts=", "--rootdir", os.path.dirname(REF_TESTS)]
    cmd += [os.path.join("tests", s) for s in SUITES]
    for nodeid in KNOWN_RED:
        cmd += ["--deselect", nodeid]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=1800, cwd=os.path.dirname(REF_TESTS), env=env)
    tail = p.stdout[-6000:] + p.stderr[-3000:]
    print(tail)
    assert p.returncode == 0, tail
