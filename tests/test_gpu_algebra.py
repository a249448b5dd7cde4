"""GPU: the matrix algebra around the hot path and the round-2 API gaps,
bitwise against goldens produced by the reference itself
(tests/golden/make_golden_algebra.py):

  * single-precision matmul (float32 products, sums and prune) and mixed
    precision -> float64 (reference result_type, matrix.py:231);
  * add / scale / kron / adjoint / transpose as device kernels (transpose a
    zero-copy relabel of the same arena);
  * build_span_unitary of a 5-qubit gate;
  * apply_placed of an explicit placement with 90 stored diagonals;
  * the batched sweep and the device plan (structure never read back until
    asked), and matrices whose caches must see edits.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

import paper_2405_01250_b200 as D
from paper_2405_01250_b200 import _lib as L

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "algebra_cases.npz"))


def mat(key) -> D.DiaqMatrix:
    """A host-built (reference-style) matrix from a golden."""
    n = int(G[key + "_n"][0])
    dt = np.dtype(str(G[key + "_dtype"][0]))
    m = D.DiaqMatrix(n, dt)
    pos = 0
    for d in G[key + "_offs"].tolist():
        ln = n - abs(d)
        m.set_diag(d, G[key + "_re"][pos:pos + ln], G[key + "_im"][pos:pos + ln])
        pos += ln
    return m


def same(got: D.DiaqMatrix, key: str) -> None:
    want = mat(key)
    assert got.n_dim == want.n_dim
    assert got.dtype == want.dtype, (got.dtype, want.dtype)
    assert got.diag_indices() == want.diag_indices()
    for a, b in zip(got.diagonals(), want.diagonals()):
        assert a.re.dtype == want.dtype
        assert np.array_equal(a.re, b.re) and np.array_equal(a.im, b.im), a.index


@pytest.mark.parametrize("i", range(24))
def test_matmul_single_and_mixed_precision(i):
    a, b = mat(f"mm{i}_a"), mat(f"mm{i}_b")
    same(D.matmul(a, b), f"mm{i}_c")


def test_matmul_batch_matches_per_call():
    pairs = [(mat(f"mm{i}_a"), mat(f"mm{i}_b")) for i in range(24)]
    for i, c in enumerate(D.matrix.matmul_batch(pairs)):
        same(c, f"mm{i}_c")


@pytest.mark.parametrize("i", range(12))
@pytest.mark.parametrize("op", ["add", "scale", "kron", "adjoint", "transpose"])
def test_algebra_ops(i, op):
    a, b, k = mat(f"alg{i}_a"), mat(f"alg{i}_b"), mat(f"alg{i}_k")
    s = complex(G[f"alg{i}_s"][0])
    got = {"add": lambda: D.add(a, b), "scale": lambda: D.scale(a, s), "kron": lambda: D.kron(a, k),
           "adjoint": lambda: D.adjoint(a), "transpose": lambda: D.transpose(a)}[op]()
    same(got, f"alg{i}_{op}")


def test_transpose_is_a_relabel_of_the_same_arena():
    a = mat("alg0_a")
    dev = a._device().vals
    t = D.transpose(a)
    assert t._dev.vals.data_ptr() == dev.data_ptr()
    assert D.transpose(t) == a


def test_span_embedding_five_qubits():
    g = D.from_dense(G["span5_g"], 0.0)
    same(D.build_span_unitary(g, G["span5_positions"].tolist(), 7), "span5_out")


def test_placement_with_more_than_64_diagonals():
    m = mat("wide_m")
    assert m.diag_count() == 90
    p = D.Placement(dim_a=2, m=m, dim_b=4, span_lo=1, span_hi=6, name="wide")
    y = D.apply_placed(p, D.StateVector(9, G["wide_x"]))
    assert np.array_equal(y.amps, G["wide_y"])


def test_device_plan_structure_resolves_lazily():
    """A product of a product: planned on the device, structure read back
    only when asked; equal to the host-planned path."""
    a, b = mat("mm3_a"), mat("mm3_b")
    ab = D.matmul(a, b)
    assert ab._dev.offs is None  # structure still only on the device
    abb = D.matmul(ab, b)
    host = D.matrix._matmul_host(D.matrix._matmul_host(a, b, ab.dtype), b, ab.dtype)
    assert abb == host


def test_edits_invalidate_device_and_program_caches():
    """set_diag after a device upload, p.m reassignment and
    edited gates are seen by later kernels."""
    x = np.zeros(8, dtype=np.complex128)
    x[1] = 1.0
    m = D.from_dense(np.eye(2), 0.0)
    p = D.Placement(dim_a=1, m=m, dim_b=4, span_lo=0, span_hi=0, name="m")
    y1 = D.run_gates(D.StateVector(3, x), [p]).amps
    m.set_diag(0, [2.0, 3.0])  # edit after the first upload
    y2 = D.run_gates(D.StateVector(3, x), [p]).amps
    assert y1[1] == 1.0 and y2[1] == 2.0
    p.m = D.from_dense(np.array([[0, 1], [1, 0]]), 0.0)
    y3 = D.run_gates(D.StateVector(3, x), [p]).amps
    assert y3[5] == 1.0 and y3[1] == 0.0
    st = D.StateVector(3, x)
    host = st.amps
    st.device_amps  # upload: the host copy becomes a read-only snapshot
    with pytest.raises(ValueError):
        host[0] = 1.0
    st.amps = np.ones(8)
    assert D.run_gates(st, [p]).amps.sum() == 8.0


def test_spmv_rejects_out_aliasing_x():
    import torch
    a = mat("alg0_a")
    x = torch.zeros(a.n_dim, dtype=torch.complex128, device="cuda")
    with pytest.raises(ValueError):
        D.spmv(a, x, out=x)
