"""pytest plugin (-p _diaqsim_alias): makes `import diaqsim` resolve to
paper_2405_01250_b200, so the reference's own unit tests
(baseline/_ref/tests, copied there by tools/install_reference.py) exercise
the drop-in.  Every module the hot path owns maps to ours; the reference's
host-only front end that is out of scope here (the QASM
parser and the circuit generators) is loaded from the unmodified reference
source under the alias package, so it builds our Circuit/GateOp objects."""
import importlib
import importlib.util
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref", "diaqsim")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import paper_2405_01250_b200 as _pkg  # noqa: E402

OURS = ["alloc", "errors", "matrix", "gates", "sim", "memory", "analysis", "cli"]
REFERENCE_HOST_ONLY = ["qasm", "circuits"]

sys.modules["diaqsim"] = _pkg
for _name in OURS:
    sys.modules[f"diaqsim.{_name}"] = importlib.import_module(f"paper_2405_01250_b200.{_name}")
for _name in REFERENCE_HOST_ONLY:
    _spec = importlib.util.spec_from_file_location(f"diaqsim.{_name}", os.path.join(REF, f"{_name}.py"))
    _mod = importlib.util.module_from_spec(_spec)
    _mod.__package__ = "diaqsim"
    sys.modules[f"diaqsim.{_name}"] = _mod
    _spec.loader.exec_module(_mod)
    setattr(_pkg, _name, _mod)
for _sym in ("lower", "parse", "parse_circuit", "unparse"):
    if not hasattr(_pkg, _sym):
        setattr(_pkg, _sym, getattr(sys.modules["diaqsim.qasm"], _sym))
for _sym in ("ghz_qasm", "qft_qasm", "tfim_qasm"):
    if not hasattr(_pkg, _sym):
        setattr(_pkg, _sym, getattr(sys.modules["diaqsim.circuits"], _sym))
