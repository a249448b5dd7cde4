"""GPU parity of the contracted gate arithmetic (DIAQ_CMUL_CONTRACT,
sim.set_numerics("contracted")): fused multiply-add chains and folded runs
of diagonal factors inside the fused passes.  Not bitwise the reference by
design; the bar is the north-star tolerance, 1e-12 relative L2, against the
pinned CPU oracle (config 3) or the bitwise gate-by-gate path (which the
parity suite pins to the oracle).  The contracted passes must still be
deterministic: the AOT interpreter and the NVRTC-specialised kernels give
bitwise the same state, run after run.
"""
from __future__ import annotations

import numpy as np
import pytest

from _circuits import fuzz_circuit
import paper_2405_01250_b200 as D
from conftest import rel_l2
from oracle import oracle as O
from paper_2405_01250_b200 import _lib as L
from paper_2405_01250_b200 import workloads as W

pytestmark = pytest.mark.gpu

TOL = 1e-12  # north_star: amplitudes within 1e-12 relative L2 (complex128)
C = L.CMUL_CONTRACT


@pytest.fixture(scope="module")
def ref_mode(configs):
    return L.CMUL_FMA if configs["meta"]["numpy_cmul"] == "fma" else L.CMUL_PLAIN


@pytest.fixture(autouse=True, scope="module")
def _built():
    from paper_2405_01250_b200 import build
    build.build()
    L.load()
    yield
    D.sim.set_numerics("reference")


def test_set_numerics_switch():
    D.sim.set_numerics("contracted")
    assert D.sim.CMUL_MODE == L.CMUL_CONTRACT
    D.sim.set_numerics("reference")
    assert D.sim.CMUL_MODE in (L.CMUL_PLAIN, L.CMUL_FMA)
    with pytest.raises(ValueError):
        D.sim.set_numerics("fast")


def test_contracted_config3_vs_oracle(ref_mode):
    """Config 3 (n=20, 40 layers, 1200 gates) through run(): within 1e-12
    of the oracle's reference-rounded state."""
    n = 20
    ops = W.random_layered_ops(n, 40, seed=0)
    want = O.run_circuit(n, ops, cmul_mode=ref_mode)
    D.sim.set_numerics("contracted")
    try:
        res = D.run(D.Circuit(n, [D.GateOp(*o) for o in ops]), shots=0, span_limit=n, emit_state=True)
    finally:
        D.sim.set_numerics("reference")
    err = rel_l2(res.state, want)
    assert err < TOL, err
    assert abs(np.linalg.norm(res.state) - 1.0) < 1e-12
    # the same program with every specialised kernel compiled before it runs
    # (the default compiles in the background and interprets meanwhile), in
    # both numerics: 1e-12 contracted, bitwise with the reference rounding
    pls = D.compile_circuit(D.Circuit(n, [D.GateOp(*o) for o in ops]), span_limit=n)
    try:
        L.tune("fused_jit", 2)
        got = D.run_gates(D.init_state(n), pls, cmul_mode=C).amps
        assert rel_l2(got, want) < TOL
        assert np.array_equal(D.run_gates(D.init_state(n), pls, cmul_mode=ref_mode).amps, want)
    finally:
        L.tune("fused_jit", 1)


@pytest.mark.parametrize("seed", range(6))
def test_contracted_fuzz_every_tile(ref_mode, seed):
    """Every gate kind the scheduler routes differently, every tile size and
    scheduling switch: within 1e-12 of the bitwise gate-by-gate state."""
    n, pls, rng = fuzz_circuit(seed)
    x0 = D.StateVector(n, W.random_state(rng, 2**n))
    want = D.run_gates(x0, pls, cmul_mode=ref_mode, tile_bits=0).amps
    switches = [{}, {"fused_seq": 0}, {"fused_gperm": 0}, {"fused_dense2": 0}, {"fused_lookahead": 0},
                {"fused_unit": 0}, {"fused_reorder": 0}, {"fused_slots": 0}, {"fused_maxph": 3}]
    try:
        for sw in switches:
            for k, v in sw.items():
                L.tune(k, v)
            for tb in (11, 12, -1, 0):
                got = D.run_gates(x0, pls, cmul_mode=C, tile_bits=tb).amps
                err = rel_l2(got, want)
                assert err < TOL, (seed, n, tb, sw, err)
            for k in sw:
                L.tune(k, 5 if k == "fused_maxph" else 1)
    finally:
        for k in ("fused_seq", "fused_gperm", "fused_dense2", "fused_lookahead", "fused_unit", "fused_reorder",
                  "fused_slots"):
            L.tune(k, 1)
        L.tune("fused_maxph", 5)


@pytest.mark.parametrize("seed", range(3))
def test_contracted_jit_matches_interpreter_bitwise(seed):
    """Deterministic: the specialised passes and the AOT interpreter compute
    the contracted state identically (same helpers, same order)."""
    n, pls, rng = fuzz_circuit(seed)
    x0 = D.StateVector(n, W.random_state(rng, 2**n))
    try:
        for tb, pst in ((11, 2), (12, 2), (11, 0)):
            L.tune("fused_pair_store", pst)
            L.tune("fused_jit", 0)
            aot = D.run_gates(x0, pls, cmul_mode=C, tile_bits=tb).amps
            L.tune("fused_jit", 2)
            jit = D.run_gates(x0, pls, cmul_mode=C, tile_bits=tb).amps
            again = D.run_gates(x0, pls, cmul_mode=C, tile_bits=tb).amps
            assert np.array_equal(aot, jit) and np.array_equal(jit, again), (seed, tb, pst)
    finally:
        L.tune("fused_jit", 1)
        L.tune("fused_pair_store", 2)


def test_contracted_haar4_layers(ref_mode):
    """Dense two-qubit gates (the metric's Haar4 kind) through the contracted
    dense2 chains, n=20, two layers on random matchings."""
    n = 20
    rng = np.random.default_rng(3)
    pls = []
    for _ in range(2):
        perm = rng.permutation(n)
        for i in range(n // 2):
            qa, qb = int(perm[2 * i]), int(perm[2 * i + 1])
            lo, hi = min(qa, qb), max(qa, qb)
            pls.append(D.Placement(2**lo, None, 2 ** (n - 1 - hi), lo, hi, "haar",
                                   gate=(W.haar(rng, 4), [qa - lo, qb - lo])))
    x0 = D.StateVector(n, W.random_state(rng, 2**n))
    want = D.run_gates(x0, pls, cmul_mode=ref_mode, tile_bits=0).amps
    for tb in (11, 12, -1):
        err = rel_l2(D.run_gates(x0, pls, cmul_mode=C, tile_bits=tb).amps, want)
        assert err < TOL, (tb, err)


def test_contracted_layer_n24_norm_and_parity(ref_mode):
    """The benchmark's layer kind at n=24, 6 layers from |0..0>: parity with
    the bitwise path and norm preservation."""
    n = 24
    ops = W.random_layered_ops(n, 6, seed=11)
    pls = D.compile_circuit(D.Circuit(n, [D.GateOp(*o) for o in ops]), span_limit=n)
    want = D.run_gates(D.init_state(n), pls, cmul_mode=ref_mode).amps
    got = D.run_gates(D.init_state(n), pls, cmul_mode=C)
    assert rel_l2(got.amps, want) < TOL
    assert abs(got.norm() - 1.0) < 1e-12


def test_contracted_sharded_emulated(ref_mode):
    """The sharded code path (2 and 4 emulated shards) under the contracted
    arithmetic against the unsharded bitwise state."""
    from paper_2405_01250_b200.shard import run_emulated
    n = 20
    ops = W.random_layered_ops(n, 4, seed=2)
    pls = D.compile_circuit(D.Circuit(n, [D.GateOp(*o) for o in ops]), span_limit=n)
    want = D.run_gates(D.init_state(n), pls, cmul_mode=ref_mode).amps
    for p in (2, 4):
        shards, _ = run_emulated(n, p, pls, cmul_mode=C)
        got = np.concatenate([s.cpu().numpy() for s in shards])
        assert rel_l2(got, want) < TOL, p


@pytest.mark.parametrize("n,layers,seed", [(16, 12, 5), (22, 10, 6), (24, 8, 7)])
def test_contracted_lookahead_deep_passes(ref_mode, n, layers, seed):
    """Layered circuits deep enough that the lookahead schedule packs several
    layers into a pass (tile bits chosen by trial sweeps, gates joining the
    body ahead of a global permutation tail, rotations in unit-diagonal
    form): within 1e-12 of the bitwise program-order state, with fewer
    passes than first fit, and the same state from the interpreter."""
    import ctypes
    from paper_2405_01250_b200.sim import _GateProgram
    ops = W.random_layered_ops(n, layers, seed=seed)
    pls = D.compile_circuit(D.Circuit(n, [D.GateOp(*o) for o in ops]), span_limit=n)
    rng = np.random.default_rng(seed)
    x0 = D.StateVector(n, W.random_state(rng, 2**n))
    want = D.run_gates(x0, pls, cmul_mode=ref_mode).amps
    prog = _GateProgram([p.compact() for p in pls])

    def passes():
        st = (ctypes.c_int * 5)()
        L.check(L.load().diaq_fused_plan_mode(n, n, prog.n, prog.arr, 0, C, st), "diaq_fused_plan_mode")
        return st[0]

    try:
        L.tune("fused_lookahead", 0)
        first_fit = passes()
        L.tune("fused_lookahead", 1)
        assert passes() < first_fit
        L.tune("fused_jit", 2)
        got = D.run_gates(x0, pls, cmul_mode=C).amps
        assert rel_l2(got, want) < TOL
        L.tune("fused_jit", 0)
        assert np.array_equal(D.run_gates(x0, pls, cmul_mode=C).amps, got)
        L.tune("fused_unit", 0)  # the same schedule without the unit forms
        assert rel_l2(D.run_gates(x0, pls, cmul_mode=C).amps, want) < TOL
    finally:
        L.tune("fused_jit", 1)
        L.tune("fused_lookahead", 1)
        L.tune("fused_unit", 1)
