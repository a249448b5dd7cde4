"""CPU-side checks of the C-ABI library and the host logic (no GPU needed).

* the in-tree libdiaq_b200.so loads and exports every symbol declared in
  include/diaq_b200.h;
* the host-only ABI functions (layout, span plan, spgemm plan) agree with
  the oracle / reference rules;
* compile_circuit's compact placements agree with the reference's
  dims and embedding;
* compute entry points fail loudly without a device (no CPU fallback).
"""
from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, dense_from_pairs
from oracle import oracle as O
from paper_2405_01250_b200 import _lib as L
from paper_2405_01250_b200 import build as B
from paper_2405_01250_b200 import workloads as W


@pytest.fixture(scope="module")
def lib():
    B.build()
    return L.load()


def header_functions() -> list[str]:
    with open(os.path.join(ROOT, "include", "diaq_b200.h")) as f:
        text = f.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|uint64_t|void|const char \*)\s*\**\s*(diaq_\w+)\s*\(",
                                 text, flags=re.M)))


def test_exports_every_header_symbol(lib):
    names = header_functions()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(L.EXPORTED)


def test_version_and_counters(lib):
    assert lib.diaq_version() == 1
    lib.diaq_reset_launch_count()
    assert lib.diaq_launch_count() == 0


@pytest.mark.parametrize("n,offs", [(16, [-15, -3, 0, 1, 7, 15]), (2**20, [-(2**19) - 3, -1, 0, 5, 2**19]),
                                    (9, [0]), (1, [0])])
def test_layout_row_aligned(lib, n, offs):
    offs = np.array(offs, dtype=np.int64)
    starts, total = L.layout(n, offs)
    prev_end = 0
    for d, s in zip(offs.tolist(), starts.tolist()):
        assert s >= prev_end
        assert (s + min(d, 0)) % 8 == 0          # row r%8==0 sits 128-byte aligned
        prev_end = s + n - abs(d)
    assert total >= prev_end and total % 8 == 0


def test_layout_rejects_bad_offsets(lib):
    with pytest.raises(ValueError):
        L.layout(4, np.array([4]))
    with pytest.raises(ValueError):
        L.layout(4, np.array([1, 0]))


def test_span_plan_matches_oracle(lib, kats):
    for case in kats["kats"]["span"]:
        g = np.ascontiguousarray(dense_from_pairs(case["g"]))
        k = int(np.log2(g.shape[0]))
        pos = np.ascontiguousarray(case["positions"], dtype=np.int32)
        offs = np.zeros(4**k, dtype=np.int64)
        nd = ctypes.c_int64(0)
        L.call("diaq_span_plan", k, g.ctypes.data, pos.ctypes.data, case["span"], offs.ctypes.data,
               ctypes.addressof(nd))
        assert offs[: nd.value].tolist() == case["offsets"]


def test_spgemm_plan_matches_oracle(lib, random_cases):
    for i in range(48):
        a = O.from_dense(random_cases[f"mm{i}_a"])
        b = O.from_dense(random_cases[f"mm{i}_b"])
        cap = max(1, len(a.offs) * len(b.offs))
        want = np.zeros(cap, dtype=np.int64)
        nw = O.lib().oracle_matmul_plan(a.n, len(a.offs), O._p(a.offs), len(b.offs), O._p(b.offs),
                                        O._p(want))
        got = np.zeros(cap, dtype=np.int64)
        nc = ctypes.c_int64(0)
        L.call("diaq_spgemm_plan", a.n, len(a.offs), a.offs.ctypes.data, len(b.offs), b.offs.ctypes.data,
               got.ctypes.data, ctypes.addressof(nc))
        assert got[: nc.value].tolist() == want[:nw].tolist()


def test_compile_compact_placements_match_reference_dims():
    from paper_2405_01250_b200 import Circuit, GateOp, ResourceError, compile_circuit
    ops = W.random_layered_ops(12, 3, seed=1)
    c = Circuit(12, [GateOp(*o) for o in ops])
    pls = compile_circuit(c, span_limit=12)
    for p, (name, qubits, params) in zip(pls, ops):
        lo, hi = min(qubits), max(qubits)
        assert (p.dim_a, p.dim_b, p.span_lo, p.span_hi, p.name) == (2**lo, 2 ** (11 - hi), lo, hi, name)
        assert p.n_dim == 2**12
        g, shifts = p.compact()
        # operand i sits on state bit n-1-q_i (qubit 0 = most significant)
        assert shifts == [11 - q for q in qubits]
        assert np.array_equal(g, O.GATES[name](*params))
    with pytest.raises(ResourceError, match="cx"):
        compile_circuit(Circuit(8, [GateOp("cx", (0, 7))]), span_limit=4)


def test_gateop_validation_errors():
    from paper_2405_01250_b200 import Circuit, GateOp, ShapeError, UnsupportedGateError
    with pytest.raises(UnsupportedGateError):
        GateOp("frobnicate", (0,))
    with pytest.raises(ShapeError):
        GateOp("cx", (1, 1))
    with pytest.raises(ShapeError):
        GateOp("h", (0,), (0.5,))
    with pytest.raises(ShapeError):
        Circuit(2, [GateOp("h", (5,))])


def test_diag_len_and_shape_errors():
    from paper_2405_01250_b200 import DiaqMatrix, ShapeError, diag_len
    assert diag_len(0, 4) == 4 and diag_len(-3, 4) == 1
    with pytest.raises(ValueError):
        diag_len(4, 4)
    with pytest.raises(ShapeError):
        DiaqMatrix(0)
    a = DiaqMatrix(4)
    with pytest.raises(ShapeError):
        a.set_diag(1, [1.0, 2.0])


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="checks the no-device path")
def test_compute_fails_loudly_without_device():
    from paper_2405_01250_b200 import from_dense, init_state
    with pytest.raises(L.DeviceError):
        init_state(3)
    with pytest.raises(L.DeviceError):
        from_dense(np.eye(2))


def test_analysis_guard_without_device():
    from paper_2405_01250_b200 import Circuit, GateOp, ResourceError, chain_product_analysis
    with pytest.raises(ResourceError):
        chain_product_analysis(Circuit(15, [GateOp("h", (0,))]))
    with pytest.raises(ValueError):
        chain_product_analysis(Circuit(2, [GateOp("h", (0,))]), order="middle")


def _plan(lib, n, ops, tile_bits=12, local_bits=None):
    import paper_2405_01250_b200 as D
    from paper_2405_01250_b200.sim import _GateProgram
    pls = D.compile_circuit(D.Circuit(n, [D.GateOp(*o) for o in ops]), span_limit=n)
    prog = _GateProgram([p.compact() for p in pls])
    st = (ctypes.c_int * 5)()
    L.check(lib.diaq_fused_plan(n, n if local_bits is None else local_bits, prog.n, prog.arr, tile_bits, st),
            "diaq_fused_plan")
    return dict(zip(["passes", "single", "phases", "folded", "smem_phases"], list(st)))


def test_fused_schedule_lookahead_host_only(lib):
    """Contracted arithmetic: the lookahead schedule of config 5 (n=30, 20
    layers) needs about half the passes of first fit, the program-order
    schedule of the bitwise modes is untouched by the knob, and a one-layer
    program (the benchmark's step) keeps its two passes."""
    import paper_2405_01250_b200 as D
    from paper_2405_01250_b200.sim import _GateProgram

    phases = {}

    def passes(n, ops, mode):
        pls = D.compile_circuit(D.Circuit(n, [D.GateOp(*o) for o in ops]), span_limit=n)
        prog = _GateProgram([p.compact() for p in pls])
        st = (ctypes.c_int * 5)()
        L.check(lib.diaq_fused_plan_mode(n, n, prog.n, prog.arr, 0, mode, st), "diaq_fused_plan_mode")
        assert st[3] == sum(1 for o in ops if o[0] == "cx")  # every CX folded or a register exchange, none executed
        assert st[1] == 0 and st[4] == 0
        phases[(n, mode)] = st[2]
        return st[0]

    ops = W.random_layered_ops(30, 20, seed=0)
    inorder = passes(30, ops, L.CMUL_FMA)
    look = passes(30, ops, L.CMUL_CONTRACT)
    ph_slots = phases[(30, L.CMUL_CONTRACT)]
    L.tune("fused_lookahead", 0)
    try:
        first_fit = passes(30, ops, L.CMUL_CONTRACT)
        assert passes(30, ops, L.CMUL_FMA) == inorder
    finally:
        L.tune("fused_lookahead", 1)
    assert look < first_fit < inorder
    assert look <= 0.6 * inorder
    # phase slots: several layers' gates per phase -- fewer shared-memory round
    # trips at about the same pass count, and never more than the cap per pass
    assert ph_slots <= 5 * look
    L.tune("fused_slots", 0)
    try:
        flat = passes(30, ops, L.CMUL_CONTRACT)
        assert ph_slots < phases[(30, L.CMUL_CONTRACT)] and look <= flat + 2
    finally:
        L.tune("fused_slots", 1)
    one = W.random_layered_ops(28, 1, seed=0)
    assert passes(28, one, L.CMUL_CONTRACT) == passes(28, one, L.CMUL_FMA) == 2


def test_fused_schedule_host_only(lib):
    """The fused-pass scheduler (host code behind diaq_run_gates_fused) on
    the benchmark layer and on permutation-heavy circuits: CX/X/SWAP runs
    are folded into the pass addressing, never executed."""
    n = 28
    ops = W.random_layered_ops(n, 1, seed=0)
    st = _plan(lib, n, ops)
    assert st["folded"] == n // 2 and st["single"] == 0 and st["smem_phases"] == 0
    # 28 mixing bits through 12-bit tiles (3 low bits shared): two compute
    # passes; the CX run whose targets leave the tile rides the second pass's store
    assert st["passes"] == 2
    L.tune("fused_gperm", 0)
    try:
        assert _plan(lib, n, ops)["passes"] == 4  # tile-only folding: two relabelling copy passes
        many = [("cx", (27 - i, 0), ()) for i in range(12)]
        st = _plan(lib, 28, many)   # more than 8 distinct controls outside the tile start a new pass
        assert st["folded"] + st["single"] == 12 and st["passes"] == 2
    finally:
        L.tune("fused_gperm", 1)
    many = [("h", (27,), ())] + [("cx", (27 - i, 0), ()) for i in range(12)]
    st = _plan(lib, 28, many)     # ... or join the global tail of the pass
    assert st["folded"] == 12 and st["passes"] == 1
    # a pure permutation circuit: everything folded, every pass a relabelling copy
    cx = [("cx", (i, (i + 5) % 20), ()) for i in range(20)] + [("x", (3,), ()), ("swap", (0, 19), ())]
    st = _plan(lib, 20, cx)
    assert st["folded"] == len(cx) and st["phases"] == 0
    # CCX is a permutation but not affine: shared-memory path, not folded
    st = _plan(lib, 16, [("ccx", (0, 1, 2), ()), ("cx", (3, 4), ())])
    assert st["folded"] == 1
    # states smaller than a tile: gate by gate
    st = _plan(lib, 8, [("h", (0,), ()), ("cx", (0, 1), ())])
    assert st["passes"] == st["single"] == 2
    # shard view: a gate mixing a global bit is refused (it needs the partner shard)
    with pytest.raises(ValueError):
        _plan(lib, 24, [("h", (0,), ())], local_bits=22)


def test_sharded_and_peer_entry_points_validate_first(lib):
    """Argument errors of the sharded/peer ABI are reported before any device
    work (so they behave the same with or without a GPU)."""
    P = ctypes.c_void_p
    offs = np.array([-4, 0, 4], dtype=np.int64)
    rows = (P * 3)(1, 2, 3)
    parts = (P * 2)(16, 32)
    y = P(64)
    # parts do not tile n
    assert lib.diaq_spmv_sharded(100, 3, offs.ctypes.data, rows, 0, 50, parts, 5, 2, y, None) == L.DIAQ_ERR_SHAPE
    # rows outside n
    assert lib.diaq_spmv_sharded(64, 3, offs.ctypes.data, rows, 40, 32, parts, 5, 2, y, None) == L.DIAQ_ERR_SHAPE
    # offsets not ascending / out of range
    bad = np.array([0, -4, 4], dtype=np.int64)
    assert lib.diaq_spmv_sharded(64, 3, bad.ctypes.data, rows, 0, 32, parts, 5, 2, y, None) == L.DIAQ_ERR_VALUE
    far = np.array([-64, 0, 4], dtype=np.int64)
    assert lib.diaq_spmv_sharded(64, 3, far.ctypes.data, rows, 0, 32, parts, 5, 2, y, None) == L.DIAQ_ERR_VALUE
    # a missing x part
    holes = (P * 2)(16, None)
    assert lib.diaq_spmv_sharded(64, 3, offs.ctypes.data, rows, 0, 32, holes, 5, 2, y, None) == L.DIAQ_ERR_VALUE
    assert "x part 1 missing" in L.last_error()
    # peer-memory helpers
    assert lib.diaq_alloc(0, ctypes.byref(P())) == L.DIAQ_ERR_VALUE
    assert lib.diaq_ipc_handle(None, ctypes.create_string_buffer(64)) == L.DIAQ_ERR_VALUE
    assert lib.diaq_ipc_open(None, ctypes.byref(P())) == L.DIAQ_ERR_VALUE
    assert lib.diaq_free(None) == L.DIAQ_OK and lib.diaq_ipc_close(None) == L.DIAQ_OK
