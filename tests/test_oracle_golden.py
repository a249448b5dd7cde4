"""Pin the CPU oracle (oracle/) to the reference's own outputs (tests/golden/).

These run without a GPU.  Every comparison is bitwise (array_equal, i.e.
values equal with signed zeros folded) except where noted: the oracle
restates the reference's exact operation order and rounding.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import GOLDEN, dense_from_pairs, digest, pairs_to_complex
from oracle import oracle as O
from paper_2405_01250_b200 import workloads as W


def flat_values(m: O.OMat) -> np.ndarray:
    parts = [m.diag(int(d)) for d in m.offs]
    if not parts:
        return np.zeros(0, np.complex128)
    return np.concatenate([r + 1j * i for r, i in parts])


@pytest.fixture(scope="module")
def cmul_mode(configs):
    return O.CMUL_FMA if configs["meta"]["numpy_cmul"] == "fma" else O.CMUL_PLAIN


# ---- KATs (reference unit tests' known answers) ----------------------------

def test_kat_corner_layout_and_spmv(kats):
    corner = np.array([[1, 0, 0, 2], [0, 3, 0, 0], [0, 0, 4, 0], [5, 0, 0, 6]], dtype=complex)
    a = O.from_dense(corner)
    k = kats["kats"]["corner"]
    assert a.offs.tolist() == k["offsets"] == [-3, 0, 3]
    for d in k["offsets"]:
        assert a.diag(d)[0].tolist() == k["re"][str(d)]
    y = O.spmv(a, np.ones(4, dtype=complex))
    assert np.array_equal(y, pairs_to_complex(kats["kats"]["corner_spmv_ones"]))


def test_kat_cx_layout_and_products(kats):
    cx = np.array([[1, 0, 0, 0], [0, 1, 0, 0], [0, 0, 0, 1], [0, 0, 1, 0]], dtype=complex)
    a = O.from_dense(cx)
    k = kats["kats"]["cx_layout"]
    assert a.offs.tolist() == k["offsets"]
    for d in k["offsets"]:
        assert a.diag(d)[0].tolist() == k["re"][str(d)]
    x = O.from_dense(np.array([[0, 1], [1, 0]], dtype=complex))
    assert O.matmul(x, x).offs.tolist() == kats["kats"]["xx_offsets"] == [0]
    z = O.from_dense(np.diag([1.0, -1.0]))
    zz = O.matmul(z, z)
    assert zz.offs.tolist() == kats["kats"]["zz"]["offsets"]
    assert zz.diag(0)[0].tolist() == kats["kats"]["zz"]["re"]


def test_kat_kron_identity(kats):
    z = O.from_dense(np.diag([1.0, -1.0]))
    kz = O.kron_identity(2, z, 1)
    assert kz.offs.tolist() == kats["kats"]["kron_identity_z"]["offsets"]
    assert kz.diag(0)[0].tolist() == kats["kats"]["kron_identity_z"]["re"]
    h = np.array([[1, 1], [1, -1]]) / np.sqrt(2)
    kh = O.kron_identity(2, O.from_dense(h), 2)
    assert kh.offs.tolist() == kats["kats"]["kron_identity_h"]["offsets"]
    assert np.array_equal(kh.to_dense(), dense_from_pairs(kats["kats"]["kron_identity_h"]["dense"]))


def test_kat_span_embeddings(kats):
    for case in kats["kats"]["span"]:
        g = dense_from_pairs(case["g"])
        u = O.span_unitary(g, case["positions"], case["span"])
        assert u.offs.tolist() == case["offsets"], case["name"]
        assert np.array_equal(flat_values(u), pairs_to_complex(case["values"])), case["name"]


def test_kat_catalog_gates(kats):
    for name, rec in kats["kats"]["catalog"].items():
        g = O.from_dense(O.GATES[name](*rec["params"]))
        assert g.offs.tolist() == rec["offsets"], name
        assert np.array_equal(flat_values(g), pairs_to_complex(rec["values"])), name


def test_kat_kernel_protocol(kats):
    proto = kats["kernel_protocol"]
    mc = proto["matmul_case"]
    a = O.from_dense(dense_from_pairs(mc["a_dense"]))
    b = O.from_dense(dense_from_pairs(mc["b_dense"]))
    c = O.matmul(a, b)
    assert [int(d) for d in c.offs] == sorted(int(k) for k in mc["c"]["diags"])
    for d, pairs in mc["c"]["diags"].items():
        r, i = c.diag(int(d))
        assert np.array_equal(r + 1j * i, pairs_to_complex(pairs))
    y = O.spmv(a, pairs_to_complex(mc["x"]))
    assert np.array_equal(y, pairs_to_complex(mc["y"]))


def test_kat_ghz_states_and_counts(kats, cmul_mode):
    for n, rec in kats["kats"]["ghz"].items():
        n = int(n)
        ops = [("h", (0,), ())] + [("cx", (i, i + 1), ()) for i in range(n - 1)]
        st = O.run_circuit(n, ops, cmul_mode=cmul_mode)
        assert digest(st) == rec["digest"]
        assert O.measure_all_sample(st, n, 1024, 0) == rec["counts"]
    sim = kats["kernel_protocol"]["ghz4_simulate"]
    st = O.run_circuit(sim["n_qubits"], sim["ops"], cmul_mode=cmul_mode)
    assert np.array_equal(st, pairs_to_complex(sim["result"]["state"]))
    assert O.measure_all_sample(st, 4, sim["shots"], sim["seed"]) == sim["result"]["counts"]


# ---- BASELINE configs ------------------------------------------------------

def test_config1_spmv_bitwise():
    g = np.load(os.path.join(GOLDEN, "config1_spmv.npz"))
    c1 = W.config1(0)
    assert np.array_equal(c1["u"], g["u"]) and np.array_equal(c1["x"], g["x"])
    a = O.kron_identity(c1["left"], O.from_dense(c1["u"]), c1["right"])
    assert a.offs.tolist() == g["offsets"].tolist() == [-32, 0, 32]
    assert np.array_equal(flat_values(a), g["a_values"])
    assert np.array_equal(O.spmv(a, c1["x"]), g["y"])


def _c2(seed):
    p = W.config2(seed)
    span = O.span_unitary(p["u4"], p["u4_positions"], p["u4_span"])
    A = O.kron_identity(p["a_left"], span, p["a_right"])
    B1 = O.kron_identity(p["b1_left"], O.from_dense(p["u2"]), p["b1_right"])
    B0 = O.kron_identity(p["b0_left"], O.from_dense(W.rz(p["theta"])), p["b0_right"])
    B = O.matmul(B1, B0)
    return A, B1, B0, B, O.matmul(A, B)


def test_config2_spgemm_bitwise():
    g = np.load(os.path.join(GOLDEN, "config2_spgemm.npz"))
    A, B1, B0, B, C = _c2(0)
    assert A.offs.tolist() == g["a_offsets"].tolist()
    assert B1.offs.tolist() == g["b1_offsets"].tolist()
    assert B0.offs.tolist() == g["b0_offsets"].tolist()
    assert B.offs.tolist() == g["b_offsets"].tolist()
    assert np.array_equal(flat_values(B), g["b_values"])
    assert C.offs.tolist() == g["c_offsets"].tolist()
    assert len(C.offs) == 27
    assert np.array_equal(flat_values(C), g["c_values"])


def test_config2_sweep_digests(configs):
    for rec in configs["config2_sweep"]:
        _, _, _, B, C = _c2(rec["seed"])
        assert B.offs.tolist() == rec["b_offsets"]
        assert digest(flat_values(B)) == rec["b_digest"]
        assert C.offs.tolist() == rec["c_offsets"]
        assert digest(flat_values(C)) == rec["c_digest"], rec["seed"]


def test_random_kernel_cases(random_cases, configs, cmul_mode):
    rc = random_cases
    for i in range(48):
        c = O.matmul(O.from_dense(rc[f"mm{i}_a"]), O.from_dense(rc[f"mm{i}_b"]))
        assert c.offs.tolist() == rc[f"mm{i}_c_offsets"].tolist()
        assert np.array_equal(flat_values(c), rc[f"mm{i}_c_values"])
    for i in range(100):
        y = O.spmv(O.from_dense(rc[f"mv{i}_a"]), rc[f"mv{i}_x"])
        assert np.array_equal(y, rc[f"mv{i}_y"])
    for i in range(100):
        dim_a, dim_b = (int(v) for v in rc[f"ap{i}_dims"])
        y = O.apply_placed(dim_a, O.from_dense(rc[f"ap{i}_m"]), dim_b, rc[f"ap{i}_x"], cmul_mode)
        assert np.array_equal(y, rc[f"ap{i}_y"])


@pytest.mark.parametrize("n", [8, 12])
def test_circuit_full_state(configs, cmul_mode, n):
    rec = configs["circuits"][str(n)]
    ops = W.random_layered_ops(n, rec["layers"], rec["seed"])
    assert [[a, list(b), list(c)] for a, b, c in ops] == rec["ops"]
    st = O.run_circuit(n, ops, cmul_mode=cmul_mode)
    want = np.load(os.path.join(GOLDEN, f"circuit_n{n}_state.npy"))
    assert np.array_equal(st, want)
    assert digest(st) == rec["digest"]
    assert O.measure_all_sample(st, n, 1024, 0) == rec["counts"]


def test_circuit_n20_digest(configs, cmul_mode):
    rec = configs["circuits"]["20"]
    ops = W.random_layered_ops(20, rec["layers"], rec["seed"])
    st = O.run_circuit(20, ops, cmul_mode=cmul_mode)
    assert digest(st) == rec["digest"]


def test_fusion_case(configs, cmul_mode):
    rec = configs["circuits"]["fusion_case"]
    for fusion in (False, True):
        st = O.run_circuit(rec["n"], rec["ops"], fusion=fusion, cmul_mode=cmul_mode)
        want = pairs_to_complex(rec["runs"][str(fusion)]["state"])
        assert np.array_equal(st, want), fusion
        assert len(O.compile_ops(rec["n"], rec["ops"], fusion)) == rec["runs"][str(fusion)]["gates"]
        assert O.measure_all_sample(st, rec["n"], 512, 3) == rec["runs"][str(fusion)]["counts"]


def test_config4_n22_slice(configs):
    rec = configs["config4_n22"]
    c4 = W.config4(22, seed=0)
    assert digest(c4["x"]) == rec["x_digest"]
    span = O.span_unitary(c4["u4"], c4["positions"], c4["span"])
    a = O.kron_identity(c4["left"], span, c4["right"])
    assert a.offs.tolist() == rec["offsets"]
    assert a.offs.tolist() == [-(2**21) - 8, -(2**21), -(2**21) + 8, -8, 0, 8, 2**21 - 8, 2**21,
                               2**21 + 8]
    assert digest(flat_values(a)) == rec["a_digest"]
    y = O.spmv(a, c4["x"])
    assert digest(y) == rec["y_digest"]
