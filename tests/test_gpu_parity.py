"""GPU parity: the CUDA path (through the public API / C-ABI) against the
reference's golden vectors and the pinned CPU oracle.

Bar: bitwise (values equal, signed zeros folded) for spmv, spgemm,
kron_identity, build_span_unitary, from_dense and -- with the reference
host's complex-multiply rounding -- gate application.  Where a test states a
tolerance it is the north-star 1e-12 relative L2.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

from _circuits import fuzz_circuit
import paper_2405_01250_b200 as D
from conftest import GOLDEN, dense_from_pairs, digest, pairs_to_complex, rel_l2
from oracle import oracle as O
from paper_2405_01250_b200 import _lib as L
from paper_2405_01250_b200 import workloads as W

pytestmark = pytest.mark.gpu

CORNER = np.array([[1, 0, 0, 2], [0, 3, 0, 0], [0, 0, 4, 0], [5, 0, 0, 6]], dtype=complex)
CX = np.array([[1, 0, 0, 0], [0, 1, 0, 0], [0, 0, 0, 1], [0, 0, 1, 0]], dtype=complex)


@pytest.fixture(scope="module")
def cmul(configs):
    return L.CMUL_FMA if configs["meta"]["numpy_cmul"] == "fma" else L.CMUL_PLAIN


@pytest.fixture(autouse=True, scope="module")
def _built(cmul):
    """Build/load the library and use the golden host's complex-multiply rounding."""
    from paper_2405_01250_b200 import build
    build.build()
    L.load()
    old = D.sim.CMUL_MODE
    D.sim.CMUL_MODE = cmul
    yield
    D.sim.CMUL_MODE = old


def values(m) -> np.ndarray:
    parts = [dg.re + 1j * dg.im for dg in m.diagonals()]
    return np.concatenate(parts) if parts else np.zeros(0, np.complex128)


def omat(m) -> O.OMat:
    return O.omat_from_diags(m.n_dim, {dg.index: (dg.re, dg.im) for dg in m.diagonals()})


# ---- KATs -------------------------------------------------------------------

def test_corner_layout_and_spmv(kats):
    a = D.from_dense(CORNER, 0.0)
    assert a.diag_indices() == [-3, 0, 3]
    assert a.get(-3).re.tolist() == [5.0]
    assert a.get(0).re.tolist() == [1.0, 3.0, 4.0, 6.0]
    assert a.get(3).re.tolist() == [2.0]
    assert not any(a.get(d).im.any() for d in (-3, 0, 3))
    y = D.spmv(a, np.ones(4, dtype=complex))
    assert np.array_equal(y, pairs_to_complex(kats["kats"]["corner_spmv_ones"]))
    assert np.array_equal(D.to_dense(a), CORNER)


def test_cx_layout_and_prune(kats):
    a = D.from_dense(CX, 0.0)
    assert a.diag_indices() == [-1, 0, 1]
    assert a.get(-1).re.tolist() == [0.0, 0.0, 1.0]
    assert a.get(0).re.tolist() == [1.0, 1.0, 0.0, 0.0]
    x = D.from_dense(np.array([[0, 1], [1, 0]], dtype=complex), 0.0)
    assert D.matmul(x, x).diag_indices() == [0]
    z = D.from_dense(np.diag([1.0, -1.0]), 0.0)
    zz = D.matmul(z, z)
    assert zz.diag_indices() == [0] and zz.get(0).re.tolist() == [1.0, 1.0]


def test_from_dense_edge_cases():
    z = D.from_dense(np.zeros((4, 4)), 0.0)
    assert z.diag_count() == 0
    assert np.array_equal(D.to_dense(z), np.zeros((4, 4)))
    assert np.array_equal(D.spmv(z, np.ones(4)), np.zeros(4))
    m = CORNER.copy()
    m[0, 3] = 1e-9
    assert D.from_dense(m, 1e-6).diag_indices() == [-3, 0]
    one = D.from_dense(np.array([[2.5 - 1j]]), 0.0)
    assert one.diag_indices() == [0] and one.get(0).im.tolist() == [-1.0]
    with pytest.raises(D.ShapeError):
        D.from_dense(np.zeros((2, 3)))
    rng = np.random.default_rng(3)
    for n in (1, 2, 3, 5, 16, 64):
        m = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))
        m[np.abs(np.subtract.outer(np.arange(n), np.arange(n))) % 3 == 1] = 0
        a = D.from_dense(m, 0.0)
        assert a.diag_indices() == O.from_dense(m).offs.tolist()
        assert np.array_equal(D.to_dense(a), m)


def test_multiply_diagonals_corner(kats):
    a = D.from_dense(CORNER, 0.0)
    d_c, diag = D.multiply_diagonals(a.get(3), a.get(-3), 4)
    k = kats["kats"]["multiply_diagonals_corner"]
    assert d_c == k["d_c"] == 0
    assert diag.re.tolist() == k["re"] == [10.0, 0.0, 0.0, 0.0]
    b = D.DiaqMatrix(4)
    b.set_diag(3, [1.0])
    assert D.multiply_diagonals(b.get(3), b.get(3), 4) is None


def test_kron_identity_patterns(kats):
    z = D.from_dense(np.diag([1.0, -1.0]), 0.0)
    kz = D.kron_identity(2, z, 1)
    assert kz.diag_indices() == [0] and kz.get(0).re.tolist() == [1.0, -1.0, 1.0, -1.0]
    h = np.array([[1, 1], [1, -1]]) / np.sqrt(2)
    kh = D.kron_identity(2, D.from_dense(h, 0.0), 2)
    assert kh.diag_indices() == kats["kats"]["kron_identity_h"]["offsets"]
    assert np.array_equal(D.to_dense(kh), dense_from_pairs(kats["kats"]["kron_identity_h"]["dense"]))
    a = D.from_dense(CORNER, 0.0)
    assert D.kron_identity(1, a, 1) == a
    rng = np.random.default_rng(5)
    for left, right in ((1, 4), (4, 1), (2, 2), (8, 2), (3, 5)):
        m = rng.normal(size=(4, 4)) + 1j * rng.normal(size=(4, 4))
        m[0, 2] = m[1, 3] = 0
        want = O.kron_identity(left, O.from_dense(m), right)
        got = D.kron_identity(left, D.from_dense(m, 0.0), right)
        assert got.diag_indices() == want.offs.tolist()
        assert np.array_equal(D.to_dense(got), want.to_dense())


def banded(rng, n, k):
    m = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))
    m[np.abs(np.subtract.outer(np.arange(n), np.arange(n))) > k] = 0
    return m


@pytest.mark.parametrize("flat", [1, 0])
def test_kron_identity_store_paths(flat):
    """Arena-linear (default) and per-diagonal kron_identity kernels, odd and
    power-of-two shapes, ragged diagonal lengths, against the oracle."""
    from paper_2405_01250_b200 import _lib as L
    rng = np.random.default_rng(11)
    L.tune("kron_flat", flat)
    try:
        for nm, left, right, band in ((37, 3, 5, 6), (16, 64, 8, 3), (5, 1, 1, 4), (33, 7, 1, 32), (64, 2, 32, 9)):
            m = banded(rng, nm, band)
            m[np.abs(rng.normal(size=m.shape)) > 1.5] = 0   # holes inside kept diagonals
            want = O.kron_identity(left, O.from_dense(m), right)
            got = D.kron_identity(left, D.from_dense(m, 0.0), right)
            assert got.diag_indices() == want.offs.tolist()
            for d in got.diag_indices():
                wre, wim = want.diag(d)
                assert np.array_equal(got.get(d).re, wre) and np.array_equal(got.get(d).im, wim), (nm, d)
    finally:
        L.tune("kron_flat", 1)


def test_span_embeddings(kats):
    for case in kats["kats"]["span"]:
        g = D.from_dense(dense_from_pairs(case["g"]), 0.0)
        u = D.build_span_unitary(g, case["positions"], case["span"])
        assert u.diag_indices() == case["offsets"], case["name"]
        assert np.array_equal(values(u), pairs_to_complex(case["values"])), case["name"]
    gsw = D.gate_matrix(D.GateOp("swap", (0, 1)))
    assert D.build_span_unitary(gsw, [0, 1], 2) == gsw
    with pytest.raises(D.ShapeError):
        D.build_span_unitary(gsw, [0, 0], 2)
    with pytest.raises(D.ShapeError):
        D.build_span_unitary(gsw, [0, 2], 2)


def test_catalog_gates(kats):
    for name, rec in kats["kats"]["catalog"].items():
        nq = D.GATE_DEFS[name][0]
        g = D.gate_matrix(D.GateOp(name, tuple(range(nq)), tuple(rec["params"])))
        assert g.diag_indices() == rec["offsets"], name
        assert np.array_equal(values(g), pairs_to_complex(rec["values"])), name


def test_kernel_protocol_goldens(kats):
    proto = kats["kernel_protocol"]
    corner = proto["corner"]
    a = D.from_dense(dense_from_pairs(corner["dense"]), 0.0)
    assert D.to_json_dict(a) == corner["wire"]
    assert np.array_equal(D.to_dense(D.from_json_dict(corner["wire"])), dense_from_pairs(corner["round_trip"]))
    mc = proto["matmul_case"]
    a = D.from_json_dict(mc["a"])
    b = D.from_json_dict(mc["b"])
    c = D.matmul(a, b)
    assert D.to_json_dict(c) == mc["c"]
    assert np.array_equal(D.to_dense(c), dense_from_pairs(mc["c_dense"]))
    y = D.spmv(a, pairs_to_complex(mc["x"]))
    assert np.array_equal(y, pairs_to_complex(mc["y"]))


# ---- BASELINE configs ------------------------------------------------------

def test_config1_spmv_bitwise():
    g = np.load(os.path.join(GOLDEN, "config1_spmv.npz"))
    c1 = W.config1(0)
    a = D.kron_identity(c1["left"], D.from_dense(c1["u"], 0.0), c1["right"])
    assert a.diag_indices() == g["offsets"].tolist() == [-32, 0, 32]
    assert [len(dg) for dg in a.diagonals()] == [16352, 16384, 16352]
    assert np.array_equal(values(a), g["a_values"])
    y = D.spmv(a, c1["x"])
    assert np.array_equal(y, g["y"])


def _c2(seed):
    p = W.config2(seed)
    span = D.build_span_unitary(D.from_dense(p["u4"], 0.0), p["u4_positions"], p["u4_span"])
    A = D.kron_identity(p["a_left"], span, p["a_right"])
    B1 = D.kron_identity(p["b1_left"], D.from_dense(p["u2"], 0.0), p["b1_right"])
    B0 = D.kron_identity(p["b0_left"], D.from_dense(W.rz(p["theta"]), 0.0), p["b0_right"])
    B = D.matmul(B1, B0)
    return A, B1, B0, B, D.matmul(A, B)


def test_config2_spgemm_bitwise():
    g = np.load(os.path.join(GOLDEN, "config2_spgemm.npz"))
    A, B1, B0, B, C = _c2(0)
    assert A.diag_indices() == g["a_offsets"].tolist()
    assert B.diag_indices() == g["b_offsets"].tolist()
    assert np.array_equal(values(B), g["b_values"])
    assert C.diag_indices() == g["c_offsets"].tolist()
    assert C.diag_count() == 27
    assert np.array_equal(values(C), g["c_values"])
    assert D.matmul(A, B) == C  # bitwise repeatable


def test_config2_sweep_digests(configs):
    for rec in configs["config2_sweep"]:
        _, _, _, B, C = _c2(rec["seed"])
        assert B.diag_indices() == rec["b_offsets"]
        assert digest(values(B)) == rec["b_digest"]
        assert C.diag_indices() == rec["c_offsets"]
        assert digest(values(C)) == rec["c_digest"], rec["seed"]


def test_random_kernel_cases(random_cases, cmul):
    rc = random_cases
    for i in range(48):
        c = D.matmul(D.from_dense(rc[f"mm{i}_a"], 0.0), D.from_dense(rc[f"mm{i}_b"], 0.0))
        assert c.diag_indices() == rc[f"mm{i}_c_offsets"].tolist()
        assert np.array_equal(values(c), rc[f"mm{i}_c_values"])
    for i in range(100):
        y = D.spmv(D.from_dense(rc[f"mv{i}_a"], 0.0), rc[f"mv{i}_x"])
        assert np.array_equal(y, rc[f"mv{i}_y"]), i
    for i in range(100):
        dim_a, dim_b = (int(v) for v in rc[f"ap{i}_dims"])
        m = D.from_dense(rc[f"ap{i}_m"], 0.0)
        n_q = int(np.log2(m.n_dim))
        p = D.Placement(dim_a, m, dim_b, 0, n_q - 1, "rand")
        x = D.StateVector(int(np.log2(len(rc[f"ap{i}_x"]))), rc[f"ap{i}_x"])
        y = D.apply_placed(p, x, cmul_mode=cmul).amps
        assert np.array_equal(y, rc[f"ap{i}_y"]), i


def test_generic_placed_kernel_matches_oracle(cmul):
    """Non-power-of-two placements take the diagonal kernel (apply.cu placed_kernel)."""
    rng = np.random.default_rng(11)
    for dim_a, n_m, dim_b in ((3, 5, 2), (1, 7, 1), (5, 3, 4), (2, 33, 3)):
        m = rng.normal(size=(n_m, n_m)) + 1j * rng.normal(size=(n_m, n_m))
        m[np.abs(np.subtract.outer(np.arange(n_m), np.arange(n_m))) % 2 == 1] = 0
        x = rng.normal(size=dim_a * n_m * dim_b) + 1j * rng.normal(size=dim_a * n_m * dim_b)
        p = D.Placement(dim_a, D.from_dense(m, 0.0), dim_b, 0, 0, "g")
        assert p.compact() is None
        got = D.apply_placed(p, D.StateVector(0, x), cmul_mode=cmul).amps
        want = O.apply_placed(dim_a, O.from_dense(m), dim_b, x, cmul)
        assert np.array_equal(got, want)


@pytest.mark.parametrize("n", [8, 12])
def test_circuit_full_state(configs, cmul, n):
    rec = configs["circuits"][str(n)]
    ops = W.random_layered_ops(n, rec["layers"], rec["seed"])
    c = D.Circuit(n, [D.GateOp(*o) for o in ops])
    res = D.run(c, shots=1024, seed=0, span_limit=n, emit_state=True)
    want = np.load(os.path.join(GOLDEN, f"circuit_n{n}_state.npy"))
    assert np.array_equal(res.state, want)
    assert res.counts == rec["counts"]
    assert len(res.timings_ns["per_gate"]) == len(ops)


def test_circuit_n20_vs_reference_digest_and_oracle(configs, cmul):
    rec = configs["circuits"]["20"]
    ops = W.random_layered_ops(20, rec["layers"], rec["seed"])
    c = D.Circuit(20, [D.GateOp(*o) for o in ops])
    st = D.run_gates(D.init_state(20), D.compile_circuit(c, span_limit=20), cmul_mode=cmul)
    amps = st.amps
    assert digest(amps) == rec["digest"]
    idx = np.array(rec["sample_idx"])
    assert np.array_equal(amps[idx], pairs_to_complex(rec["sample"]))
    assert abs(st.norm() - 1.0) < 1e-10


def test_fusion_case(configs, cmul):
    rec = configs["circuits"]["fusion_case"]
    c = D.Circuit(rec["n"], [D.GateOp(*o) for o in rec["ops"]])
    for fusion in (False, True):
        res = D.run(c, shots=512, seed=3, fusion=fusion, emit_state=True, span_limit=6)
        want = pairs_to_complex(rec["runs"][str(fusion)]["state"])
        assert rel_l2(res.state, want) < 1e-12
        assert np.array_equal(res.state, want), fusion
        assert len(res.timings_ns["per_gate"]) == rec["runs"][str(fusion)]["gates"]
        assert res.counts == rec["runs"][str(fusion)]["counts"]


def test_ghz_kats(kats, cmul):
    for n, rec in kats["kats"]["ghz"].items():
        n = int(n)
        ops = [("h", (0,), ())] + [("cx", (i, i + 1), ()) for i in range(n - 1)]
        res = D.run(D.Circuit(n, [D.GateOp(*o) for o in ops]), shots=1024, seed=0, emit_state=True)
        assert digest(res.state) == rec["digest"]
        assert res.counts == rec["counts"]
    sim = kats["kernel_protocol"]["ghz4_simulate"]
    res = D.run(D.Circuit(4, [D.GateOp(*o) for o in sim["ops"]]), shots=1024, seed=7, emit_state=True)
    assert np.array_equal(res.state, pairs_to_complex(sim["result"]["state"]))
    assert res.counts == sim["result"]["counts"] == {"0000": 534, "1111": 490}


def test_config4_n22_slice(configs):
    rec = configs["config4_n22"]
    c4 = W.config4(22, seed=0)
    assert digest(c4["x"]) == rec["x_digest"]
    span = D.build_span_unitary(D.from_dense(c4["u4"], 0.0), c4["positions"], c4["span"])
    a = D.kron_identity(c4["left"], span, c4["right"])
    assert a.diag_indices() == rec["offsets"]
    assert digest(values(a)) == rec["a_digest"]
    y = D.spmv(a, c4["x"])
    assert digest(y) == rec["y_digest"]


# ---- errors, determinism, edge sizes ----------------------------------------------

def test_error_contract():
    with pytest.raises(D.ShapeError, match="not multiplyable"):
        D.spmv(D.identity(4), np.ones(5))
    with pytest.raises(D.ShapeError, match="not multiplyable"):
        D.matmul(D.identity(4), D.identity(8))
    with pytest.raises(D.ResourceError):
        D.init_state(31)
    with pytest.raises(D.ResourceError):
        D.init_state(0)
    p = D.Placement(2, D.from_dense(np.eye(4), 0.0), 2, 0, 1, "i")
    with pytest.raises(D.ShapeError):
        D.apply_placed(p, D.init_state(3))
    with pytest.raises(ValueError):
        D.run(D.Circuit(1, [D.GateOp("h", (0,))]), backend="gpu")


def test_spmv_many_diagonals_and_extremes():
    """nd beyond the unrolled paths (13..64 dynamic, >64 global table) and |d| = n-1."""
    rng = np.random.default_rng(21)
    for n, nd in ((97, 13), (200, 40), (300, 80), (1000, 130)):
        offs = rng.choice(np.arange(-(n - 1), n), size=nd, replace=False)
        offs[0], offs[1] = n - 1, -(n - 1)
        diags = {}
        for d in sorted(set(int(o) for o in offs)):
            ln = n - abs(d)
            diags[d] = (rng.normal(size=ln), rng.normal(size=ln))
        om = O.omat_from_diags(n, diags)
        a = D.DiaqMatrix(n)
        for d, (r, i) in diags.items():
            a.set_diag(d, r, i)
        x = rng.normal(size=n) + 1j * rng.normal(size=n)
        assert np.array_equal(D.spmv(a, x), O.spmv(om, x))


def test_determinism_and_immutability(cmul):
    rng = np.random.default_rng(2)
    m = rng.normal(size=(48, 48)) + 1j * rng.normal(size=(48, 48))
    m[np.abs(np.subtract.outer(np.arange(48), np.arange(48))) > 5] = 0
    a = D.from_dense(m, 0.0)
    assert D.matmul(a, a) == D.matmul(a, a)
    x = rng.normal(size=48) + 1j * rng.normal(size=48)
    assert np.array_equal(D.spmv(a, x), D.spmv(a, x))
    p = D.compile_circuit(D.Circuit(10, [D.GateOp("cx", (3, 8))]), span_limit=10)[0]
    xs = D.StateVector(10, rng.normal(size=1024) + 1j * rng.normal(size=1024))
    before = xs.amps.copy()
    base = D.apply_placed(p, xs, threads=1).amps
    for workers in (2, 3, 8):
        assert np.array_equal(D.apply_placed(p, xs, threads=workers).amps, base)
    assert np.array_equal(xs.amps, before)
    # lazily built span matrix agrees with the compact apply
    want = O.apply_placed(p.dim_a, omat(p.m), p.dim_b, before, cmul)
    assert np.array_equal(base, want)


def test_fused_passes_match_unfused(cmul):
    """Shared-memory multi-gate passes are bitwise equal to gate-by-gate sweeps."""
    rng = np.random.default_rng(8)
    for n in (3, 8, 11, 14, 20):
        ops = W.random_layered_ops(n, 3, seed=n)
        for _ in range(12):
            q = [int(v) for v in rng.choice(n, size=3, replace=False)]
            ops += [("ccx", tuple(q), ()), ("swap", (q[0], q[1]), ()), ("cz", (q[1], q[2]), ()),
                    ("u3", (q[2],), (0.1, 0.7, 1.3)), ("h", (q[0],), ()), ("t", (q[1],), ())]
        pls = D.compile_circuit(D.Circuit(n, [D.GateOp(*o) for o in ops]), span_limit=n)
        u = W.haar(rng, 4)
        a, b = (int(v) for v in rng.choice(n, size=2, replace=False))
        lo, hi = min(a, b), max(a, b)
        pls.append(D.Placement(2**lo, None, 2 ** (n - 1 - hi), lo, hi, "haar",
                               gate=(u, [a - lo, b - lo])))
        x0 = D.StateVector(n, W.random_state(rng, 2**n))
        want = D.run_gates(x0, pls, cmul_mode=cmul, tile_bits=0).amps
        from paper_2405_01250_b200 import _lib as L
        for seq in (1, 0):  # sequence phases (unrolled register bits) and the generic gate loop
            L.tune("fused_seq", seq)
            try:
                for tb in (6, 8, 11, 12):
                    got = D.run_gates(x0, pls, cmul_mode=cmul, tile_bits=tb).amps
                    assert np.array_equal(got, want), (n, tb, seq)
            finally:
                L.tune("fused_seq", 1)


def _perm_gate(q):
    """0/1 matrix moving old index c to new index q[c]."""
    m = np.zeros((len(q), len(q)), dtype=complex)
    for c, r in enumerate(q):
        m[r, c] = 1.0
    return m


@pytest.mark.parametrize("fold,gperm", [(1, 1), (1, 0), (0, 0)], ids=["folded-global", "folded-tile", "executed"])
def test_fused_permutation_runs(cmul, fold, gperm):
    """X / CX / SWAP runs (and any 2-qubit 0/1 permutation) folded into the
    passes' shared-memory addressing: runs opening a pass, closing a phase,
    after a shared-memory phase, with controls inside and outside the tile
    (more than the fold bound, forcing a new pass), against gate-by-gate."""
    from paper_2405_01250_b200 import _lib as L
    rng = np.random.default_rng(21)
    L.tune("fused_perm", fold)
    L.tune("fused_gperm", gperm)
    try:
        for n in (9, 12, 16, 20):
            ops = [("cx", (int(n - 1 - i), int(i % 3)), ()) for i in range(min(n - 3, 12))]  # high controls
            ops += [("x", (0,), ()), ("swap", (1, n - 1), ())]
            ops += W.random_layered_ops(n, 2, seed=n)
            for _ in range(10):
                q = [int(v) for v in rng.choice(n, size=3, replace=False)]
                ops += [("cz", (q[0], q[1]), ()), ("cx", (q[1], q[2]), ()), ("x", (q[2],), ()),
                        ("ry", (q[0],), (0.3,)), ("cx", (q[2], q[0]), ()), ("swap", (q[0], q[2]), ()),
                        ("ccx", (q[0], q[1], q[2]), ()), ("cx", (q[0], q[1]), ())]
            pls = D.compile_circuit(D.Circuit(n, [D.GateOp(*o) for o in ops]), span_limit=n)
            for cyc in ([1, 3, 0, 2], [2, 0, 3, 1], [3, 2, 1, 0]):
                a, b = (int(v) for v in rng.choice(n, size=2, replace=False))
                lo, hi = min(a, b), max(a, b)
                pls.append(D.Placement(2**lo, None, 2 ** (n - 1 - hi), lo, hi, "perm",
                                       gate=(_perm_gate(cyc), [a - lo, b - lo])))
            x0 = D.StateVector(n, W.random_state(rng, 2**n))
            want = D.run_gates(x0, pls, cmul_mode=cmul, tile_bits=0).amps
            for tb in (8, 11, 12):
                got = D.run_gates(x0, pls, cmul_mode=cmul, tile_bits=tb).amps
                assert np.array_equal(got, want), (n, tb)
        # a pure permutation circuit is a relabelling: exact values, any order of runs
        n = 18
        ops = [("cx", (int(a), int(b)), ()) for a, b in rng.integers(0, n, size=(60, 2)) if a != b]
        ops += [("x", (int(q),), ()) for q in rng.integers(0, n, size=10)]
        pls = D.compile_circuit(D.Circuit(n, [D.GateOp(*o) for o in ops]), span_limit=n)
        x0 = D.StateVector(n, W.random_state(rng, 2**n))
        want = D.run_gates(x0, pls, cmul_mode=cmul, tile_bits=0).amps
        assert np.array_equal(D.run_gates(x0, pls, cmul_mode=cmul, tile_bits=11).amps, want)
        # odd and even numbers of out-of-place passes, the caller's buffer updated in place
        for k in (1, 2, 3):
            ops = []
            for layer in range(k):
                ops += W.random_layered_ops(n, 1, seed=layer)
            pls = D.compile_circuit(D.Circuit(n, [D.GateOp(*o) for o in ops]), span_limit=n)
            st = D.StateVector(n, W.random_state(rng, 2**n))
            want = D.run_gates(st, pls, cmul_mode=cmul, tile_bits=0).amps
            out = D.run_gates(st, pls, cmul_mode=cmul, tile_bits=12, inplace=True)
            assert out.device_amps.data_ptr() == st.device_amps.data_ptr()
            assert np.array_equal(out.amps, want), k
    finally:
        L.tune("fused_perm", 1)
        L.tune("fused_gperm", 1)


def test_spmv_host_pipeline_chunks(monkeypatch):
    """Pipelined host spmv (chunked H2D / kernel / D2H) is bitwise the device spmv."""
    import torch
    c4 = W.config4(22, seed=0, with_x=False)
    span = D.build_span_unitary(D.from_dense(c4["u4"], 0.0), c4["positions"], c4["span"])
    a = D.kron_identity(1, span, c4["right"])
    x = W.random_state(np.random.default_rng(6), 2**22)
    want = D.spmv(a, torch.from_numpy(x).cuda()).cpu().numpy()
    for chunk in (300007, 2**20, 2**23):
        monkeypatch.setattr(D.matrix, "HOST_CHUNK_ROWS", chunk)
        assert np.array_equal(D.spmv(a, x), want), chunk
        xh = torch.from_numpy(x).pin_memory()
        yh = torch.empty(2**22, dtype=torch.complex128).pin_memory()
        assert D.spmv(a, xh, out=yh) is yh
        assert np.array_equal(yh.numpy(), want), chunk


def test_device_sampler_matches_reference_sampler():
    """Device sampler (exact sequential CDF) == the reference numpy sampler, shot for shot."""
    rng = np.random.default_rng(31)
    for n, shots, seed in ((1, 100, 0), (6, 4096, 3), (10, 100000, 7), (14, 50000, 11), (18, 20000, 5),
                           (20, 1024, 0), (22, 4096, 9)):
        x = W.random_state(rng, 2**n)
        if n == 6:
            x[::3] = 0  # zero runs and a sparse CDF
            x /= np.sqrt(np.sum(np.abs(x) ** 2))
        st = D.StateVector(n, x)
        assert D.measure_all_sample(st, shots, seed) == O.measure_all_sample(x, n, shots, seed), n
    uni = D.StateVector(10, np.full(1024, 1 / 32, dtype=complex))
    assert D.measure_all_sample(uni, 8192, 1) == O.measure_all_sample(np.full(1024, 1 / 32, dtype=complex),
                                                                      10, 8192, 1)
    assert D.measure_all_sample(D.init_state(3), 100, 5) == {"000": 100}
    assert D.measure_all_sample(D.init_state(2), 0, 1) == {}
    with pytest.raises(D.NormalizationError):
        D.measure_all_sample(D.StateVector(1, np.array([1.0, 0.5], dtype=complex)), 16, 0)


def test_spgemm_large_plan_and_offsets():
    """Plans beyond the by-value limit (>512 pairs) use the device-table kernel; bitwise."""
    rng = np.random.default_rng(17)
    for n, band in ((48, 24), (64, 40)):
        m1 = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))
        m2 = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))
        mask = np.abs(np.subtract.outer(np.arange(n), np.arange(n))) > band
        m1[mask] = 0
        m2[mask] = 0
        c = D.matmul(D.from_dense(m1, 0.0), D.from_dense(m2, 0.0))
        oc = O.matmul(O.from_dense(m1), O.from_dense(m2))
        assert c.diag_indices() == oc.offs.tolist()
        assert np.array_equal(values(c), np.concatenate([r + 1j * i for r, i in (oc.diag(d) for d in oc.offs)]))


def test_spmv_banded_staging_is_bitwise():
    """The shared-memory banded spmv path equals the direct path bitwise."""
    import torch
    rng = np.random.default_rng(23)
    for n, offs in ((4096, [-40, -32, 0, 8, 24]), (1 << 16, [-(1 << 12) - 8, -(1 << 12), 0, 3, (1 << 12) + 5]),
                    (1000, [-999, 0, 999]), (777, [-5, -4, 0, 1, 2, 60, 61])):
        a = D.DiaqMatrix(n)
        for d in offs:
            ln = n - abs(d)
            a.set_diag(d, rng.normal(size=ln), rng.normal(size=ln))
        x = torch.from_numpy(rng.normal(size=n) + 1j * rng.normal(size=n)).cuda()
        L.tune("spmv_banded", 1)
        y1 = D.spmv(a, x).cpu().numpy()
        L.tune("spmv_async", 0)
        y2 = D.spmv(a, x).cpu().numpy()
        L.tune("spmv_async", 1)
        L.tune("spmv_banded", 0)
        y0 = D.spmv(a, x).cpu().numpy()
        L.tune("spmv_banded", 1)
        assert np.array_equal(y0, y1) and np.array_equal(y0, y2), offs
        om = O.omat_from_diags(n, {dg.index: (dg.re, dg.im) for dg in a.diagonals()})
        assert np.array_equal(y1, O.spmv(om, x.cpu().numpy()))


def test_spmv_tma_pipeline_is_bitwise():
    """Opt-in TMA bulk-copy spmv (cp.async.bulk + mbarrier ring) equals the default path."""
    import torch
    c4 = W.config4(22, seed=0, with_x=False)
    span = D.build_span_unitary(D.from_dense(c4["u4"], 0.0), c4["positions"], c4["span"])
    a = D.kron_identity(1, span, c4["right"])
    x = torch.from_numpy(W.random_state(np.random.default_rng(9), 2**22)).cuda()
    want = D.spmv(a, x).cpu().numpy()
    try:
        L.tune("spmv_tma", 1)
        for stages in (2, 3, 4):
            L.tune("spmv_tma_stages", stages)
            assert np.array_equal(D.spmv(a, x).cpu().numpy(), want), stages
    finally:
        L.tune("spmv_tma", 0)
        L.tune("spmv_tma_stages", 4)


def test_fused_program_cache_keys_on_values(cmul):
    """The per-thread cache of scheduled fused programs is keyed by the exact
    gate data: same structure with other angles, or the same gates on other
    qubits, must not reuse a stale program."""
    n = 14
    runs = []
    for seed in (1, 2, 1, 3, 1):  # interleave so cached entries are hit and evicted
        ops = W.random_layered_ops(n, 2, seed=seed)
        pls = D.compile_circuit(D.Circuit(n, [D.GateOp(*o) for o in ops]), span_limit=n)
        got = D.run_gates(D.init_state(n), pls, cmul_mode=cmul, tile_bits=12).amps
        want = D.run_gates(D.init_state(n), pls, cmul_mode=cmul, tile_bits=0).amps
        assert np.array_equal(got, want), seed
        runs.append(got)
    assert np.array_equal(runs[0], runs[2]) and np.array_equal(runs[0], runs[4])
    assert not np.array_equal(runs[0], runs[1])
    # same angles, operands moved: a different program
    ops = [("rx", (q,), (0.3,)) for q in range(n)]
    ops2 = [("rx", (n - 1 - q,), (0.3,)) for q in range(n)] + [("cx", (0, 5), ())]
    for o in (ops, ops2, ops):
        pls = D.compile_circuit(D.Circuit(n, [D.GateOp(*x) for x in o]), span_limit=n)
        assert np.array_equal(D.run_gates(D.init_state(n), pls, cmul_mode=cmul, tile_bits=12).amps,
                              D.run_gates(D.init_state(n), pls, cmul_mode=cmul, tile_bits=0).amps)


def test_fused_two_qubit_gates(cmul):
    """Dense two-qubit gates (Haar4, and controlled Haar4 with a selector)
    fused into the passes through the shared-memory path: bitwise the
    gate-by-gate kernel, at every tile size."""
    rng = np.random.default_rng(17)
    for n in (12, 16, 20):
        pls = []
        for i in range(24):
            a, b, c = (int(v) for v in rng.choice(n, size=3, replace=False))
            u = W.haar(rng, 4)
            if i % 3 == 2:  # controlled-U: block diag(I4, U) on (c, a, b)
                g = np.eye(8, dtype=complex)
                g[4:, 4:] = u
                qs = [c, a, b]
            else:
                g, qs = u, [a, b]
            lo, hi = min(qs), max(qs)
            pls.append(D.Placement(2**lo, None, 2 ** (n - 1 - hi), lo, hi, "u",
                                   gate=(g, [q - lo for q in qs])))
            if i % 4 == 0:
                pls += D.compile_circuit(D.Circuit(n, [D.GateOp("rx", (a,), (0.3 * i,)),
                                                       D.GateOp("cx", (b, c), ())]), span_limit=n)
        x0 = D.StateVector(n, W.random_state(rng, 2**n))
        want = D.run_gates(x0, pls, cmul_mode=cmul, tile_bits=0).amps
        for tb in (11, 12, -1):
            assert np.array_equal(D.run_gates(x0, pls, cmul_mode=cmul, tile_bits=tb).amps, want), (n, tb)


@pytest.mark.parametrize("seed", range(6))
def test_fused_scheduler_fuzz(cmul, seed):
    """Seeded random circuits over every gate kind the scheduler routes
    differently (dense/sparse 1-qubit, diagonals with and without selectors,
    X/CX/SWAP runs inside and across tiles, affine 2-qubit permutations,
    CCX, dense and controlled two-qubit gates), fused at every tile setting
    and with every scheduling switch, bitwise against gate by gate."""
    from paper_2405_01250_b200 import _lib as L
    n, pls, rng = fuzz_circuit(seed)
    x0 = D.StateVector(n, W.random_state(rng, 2**n))
    want = D.run_gates(x0, pls, cmul_mode=cmul, tile_bits=0).amps
    switches = [{}, {"fused_seq": 0}, {"fused_gperm": 0}, {"fused_dense2": 0}, {"fused_perm": 0},
                {"fused_gperm_rows": 1}]
    try:
        for sw in switches:
            for k, v in sw.items():
                L.tune(k, v)
            for tb in (11, 12, -1):
                got = D.run_gates(x0, pls, cmul_mode=cmul, tile_bits=tb).amps
                assert np.array_equal(got, want), (seed, n, tb, sw)
            for k in sw:
                L.tune(k, {"fused_gperm_rows": 0}.get(k, 1))
    finally:
        for k, v in (("fused_seq", 1), ("fused_gperm", 1), ("fused_dense2", 1), ("fused_perm", 1),
                     ("fused_gperm_rows", 0)):
            L.tune(k, v)


def _jit_stats():
    import ctypes
    st = (ctypes.c_int64 * 6)()
    L.call("diaq_jit_stats", ctypes.addressof(st))
    return dict(zip(["compiled", "failed", "launches", "modules", "pending", "compile_ms"], list(st)))


@pytest.mark.parametrize("seed", range(3))
def test_fused_jit_matches_interpreter(cmul, seed):
    """Runtime-specialised passes (NVRTC, structure constant) against the AOT
    interpreter kernel and gate by gate: bitwise, and the specialised kernels
    are the ones that ran (no compile failures, launches counted)."""
    n, pls, rng = fuzz_circuit(seed)
    x0 = D.StateVector(n, W.random_state(rng, 2**n))
    want = D.run_gates(x0, pls, cmul_mode=cmul, tile_bits=0).amps
    try:
        # pair store: any tile (default), 11-bit tiles only, off
        for tb, pst in ((11, 2), (12, 2), (12, 1), (11, 0)):
            L.tune("fused_pair_store", pst)
            L.tune("fused_jit", 0)
            aot = D.run_gates(x0, pls, cmul_mode=cmul, tile_bits=tb).amps
            L.tune("fused_jit", 2)
            before = _jit_stats()
            got = D.run_gates(x0, pls, cmul_mode=cmul, tile_bits=tb).amps
            after = _jit_stats()
            assert np.array_equal(got, want) and np.array_equal(aot, want), (seed, n, tb, pst)
            assert after["failed"] == 0, L.load().diaq_jit_last_error()
            assert after["launches"] > before["launches"], (before, after, L.load().diaq_jit_last_error())
    finally:
        L.tune("fused_jit", 1)
        L.tune("fused_pair_store", 2)


@pytest.mark.parametrize("seed", [8, 13, 21, 34])
def test_fused_jit_matches_interpreter_more_seeds(cmul, seed):
    """More circuit shapes through the specialised kernels (seed 8: a pass
    opening with a permutation run AND running as a plain pair -- the pair
    fetch once ignored the opening relabelling, r02x)."""
    n, pls, rng = fuzz_circuit(seed)
    x0 = D.StateVector(n, W.random_state(rng, 2**n))
    want = D.run_gates(x0, pls, cmul_mode=cmul, tile_bits=0).amps
    try:
        L.tune("fused_jit", 2)
        for tb in (11, 12):
            assert np.array_equal(D.run_gates(x0, pls, cmul_mode=cmul, tile_bits=tb).amps, want), (seed, n, tb)
        for knob in ("fused_ppipe",):  # the pipelined pair schedules share the fetch
            for v in (1, 2):
                L.tune(knob, v)
                assert np.array_equal(D.run_gates(x0, pls, cmul_mode=cmul, tile_bits=11).amps, want), (seed, knob, v)
            L.tune(knob, 0)
    finally:
        L.tune("fused_jit", 1)
        L.tune("fused_ppipe", 0)


def test_fused_jit_opening_permutation_plain_pair(cmul):
    """The minimal form of that case: CX / SWAP opening a pass whose lowest
    non-tile bit is bit 3 (plain pair), then dense gates, no global tail."""
    n = 13
    ops = [("cx", (2, 6), ()), ("swap", (2, 8), ()), ("swap", (10, 1), ()), ("u3", (5,), (0.1, 0.5, 0.2)),
           ("ry", (7,), (0.9,)), ("rx", (12,), (0.4,)), ("h", (0,), ()), ("rx", (4,), (1.3,))]
    pls = D.compile_circuit(D.Circuit(n, [D.GateOp(*o) for o in ops]), span_limit=n)
    rng = np.random.default_rng(1)
    x0 = D.StateVector(n, W.random_state(rng, 2**n))
    want = D.run_gates(x0, pls, cmul_mode=cmul, tile_bits=0).amps
    try:
        for jit in (0, 2):
            L.tune("fused_jit", jit)
            assert np.array_equal(D.run_gates(x0, pls, cmul_mode=cmul, tile_bits=11).amps, want), jit
    finally:
        L.tune("fused_jit", 1)


def test_fused_jit_layer_n24_async(cmul):
    """The default (asynchronous) mode: the first calls run the AOT kernel
    while the passes compile, later calls the specialised kernels -- the
    state is bitwise the same either way."""
    n = 24
    ops = W.random_layered_ops(n, 2, seed=5)
    pls = D.compile_circuit(D.Circuit(n, [D.GateOp(*o) for o in ops]), span_limit=n)
    x0 = D.init_state(n)
    want = D.run_gates(x0, pls, cmul_mode=cmul, tile_bits=0).amps
    first = D.run_gates(x0, pls, cmul_mode=cmul).amps
    L.call("diaq_jit_wait", -1.0)
    before = _jit_stats()
    second = D.run_gates(x0, pls, cmul_mode=cmul).amps
    assert _jit_stats()["launches"] > before["launches"]
    assert np.array_equal(first, want) and np.array_equal(second, want)


@pytest.mark.parametrize("seed", range(3))
def test_fused_dynamic_unit_order_is_bitwise(cmul, seed):
    """The dynamic unit order (fused_dyn: units handed out by a global
    counter, active when every CTA runs several units) changes only which
    CTA computes which unit: at n=24 the scheduler fuzz circuits -- pair
    store, plain pair and scatter passes, both numerics -- give bitwise the
    same state with it on and off, and (reference rounding) the gate-by-gate
    state."""
    n, pls, rng = fuzz_circuit(seed, n=24)
    x0 = D.StateVector(n, W.random_state(rng, 2**n))
    want = D.run_gates(x0, pls, cmul_mode=cmul, tile_bits=0).amps
    try:
        for mode in (cmul, L.CMUL_CONTRACT):
            L.tune("fused_dyn", 0)
            static = D.run_gates(x0, pls, cmul_mode=mode).amps
            L.tune("fused_dyn", 1)
            dyn = D.run_gates(x0, pls, cmul_mode=mode).amps
            again = D.run_gates(x0, pls, cmul_mode=mode).amps  # fresh counter slots, same result
            assert np.array_equal(static, dyn) and np.array_equal(dyn, again), (seed, mode)
            if mode == cmul:
                assert np.array_equal(dyn, want), seed
    finally:
        L.tune("fused_dyn", 1)
