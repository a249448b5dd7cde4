"""CPU checks of the runtime-specialised fused passes (fused_jit.cu): the
pass structures the scheduler emits compile through NVRTC for sm_100a (no
device needed), over the benchmark layer and the seeded scheduler fuzz
circuits (generic shared-memory phases, tile permutations, global tails,
dense two-qubit gates).  Their results are checked bitwise on the GPU
(test_gpu_parity.py::test_fused_jit_matches_interpreter)."""
import ctypes

import pytest

from _circuits import fuzz_circuit
import paper_2405_01250_b200 as D
from paper_2405_01250_b200 import _lib as L
from paper_2405_01250_b200 import workloads as W
from paper_2405_01250_b200.sim import _GateProgram


def _compile(n, pls, tile_bits, cmul_mode=1):
    prog = _GateProgram([p.compact() for p in pls])
    secs, k = ctypes.c_double(), ctypes.c_int()
    rc = L.load().diaq_fused_jit_compile(n, n, prog.n, prog.arr, tile_bits, cmul_mode, ctypes.byref(secs),
                                         ctypes.byref(k))
    L.check(rc, "diaq_fused_jit_compile")
    return k.value, secs.value


def test_jit_exports():
    lib = L.load()
    for name in ("diaq_jit_wait", "diaq_jit_stats", "diaq_jit_last_error", "diaq_fused_jit_compile"):
        assert hasattr(lib, name)
    st = (ctypes.c_int64 * 6)()
    L.call("diaq_jit_stats", ctypes.addressof(st))
    L.call("diaq_jit_wait", 0.0)  # nothing queued: returns at once
    with pytest.raises(ValueError):
        L.call("diaq_jit_stats", None)


@pytest.mark.parametrize("cmul_mode", [L.CMUL_FMA, L.CMUL_CONTRACT])
def test_jit_compiles_benchmark_layer(cmul_mode):
    n = 28
    ops = W.random_layered_ops(n, 1, seed=0)
    pls = D.compile_circuit(D.Circuit(n, [D.GateOp(*o) for o in ops]), span_limit=n)
    for tb in (11, 12):
        kernels, secs = _compile(n, pls, tb, cmul_mode=cmul_mode)
        assert kernels == 2, (tb, kernels)


def test_jit_rejects_unknown_cmul_mode():
    n = 12
    ops = W.random_layered_ops(n, 1, seed=0)
    pls = D.compile_circuit(D.Circuit(n, [D.GateOp(*o) for o in ops]), span_limit=n)
    with pytest.raises(ValueError):
        _compile(n, pls, 11, cmul_mode=3)


@pytest.mark.parametrize("seed", [0, 3])
def test_jit_compiles_fuzz_programs(seed):
    n, pls, _ = fuzz_circuit(seed)
    kernels, _ = _compile(n, pls, 11, cmul_mode=seed % 2)
    assert kernels >= 1
