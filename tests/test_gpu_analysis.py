"""Chain-product / timestep analysis and memory models on the device vs the
reference's records (tests/golden/configs.json "analysis")."""
from __future__ import annotations

import numpy as np
import pytest

import paper_2405_01250_b200 as D

pytestmark = pytest.mark.gpu


def recs(rs):
    return [[r.timestep, r.gate_name, r.sparsity, r.diag_count, r.nnz, r.memory_map()] for r in rs]


def test_ghz10_chain_and_timestep(configs):
    a = configs["analysis"]
    c = D.Circuit(10, [D.GateOp("h", (0,))] + [D.GateOp("cx", (i, i + 1)) for i in range(9)])
    chain = D.chain_product_analysis(c)
    assert recs(chain) == a["ghz10_chain"]
    assert min(r.sparsity for r in chain) >= 0.998  # reference acceptance claim (test_acceptance.py:155-162)
    assert recs(D.timestep_analysis(c)) == a["ghz10_timestep"]
    csv = D.emit_analysis_csv(chain, mode="chain")
    assert csv.splitlines()[0] == "mode," + D.CSV_HEADER and len(csv.splitlines()) == 11
    assert D.chain_memory_totals(chain)["dense"] == 10 * (2**10) ** 2 * 16


def test_random_circuit_chains(configs):
    a = configs["analysis"]
    ops = [(o[0], tuple(o[1]), tuple(o[2])) for o in a["rl6_ops"]]
    c = D.Circuit(6, [D.GateOp(*o) for o in ops])
    assert recs(D.chain_product_analysis(c, span_limit=6)) == a["rl6_chain_left"]
    assert recs(D.chain_product_analysis(c, span_limit=6, order="right")) == a["rl6_chain_right"]
    assert recs(D.timestep_analysis(c, eps=1e-3, span_limit=6)) == a["rl6_timestep_eps"]


def test_memory_models(configs):
    m = configs["analysis"]["memory"]
    corner = np.array([[1, 0, 0, 2], [0, 3, 0, 0], [0, 0, 4, 0], [5, 0, 0, 6]], dtype=complex)
    cx = np.array([[1, 0, 0, 0], [0, 1, 0, 0], [0, 0, 0, 1], [0, 0, 1, 0]], dtype=complex)
    h = np.array([[1, 1], [1, -1]]) / np.sqrt(2)
    assert D.estimate_map(D.from_dense(corner, 0.0)) == m["corner"]
    assert D.estimate_map(D.from_dense(cx, 0.0)) == m["cx"]
    assert D.estimate_map(D.kron_identity(2, D.from_dense(h, 0.0), 2)) == m["kron_h"]
    assert D.nnz(D.from_dense(cx, 0.0), 1e-15) == 4  # stored structural zeros never count
    assert D.nnz(D.identity(1024)) == 1024
    assert D.sparsity(D.DiaqMatrix(16)) == 1.0
