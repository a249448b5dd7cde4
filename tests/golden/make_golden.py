#!/usr/bin/env python3
"""Regenerate tests/golden/ by running the REFERENCE diaqsim package.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py [--reference /root/reference/pkg/src]

Every stored output comes from the reference's own public API
(/root/reference/pkg/src/diaqsim), never from this repo's code, so the
fixtures pin the oracle (oracle/) and the CUDA path to the reference.
Inputs come from paper_2405_01250_b200.workloads (seeded generators).
Large outputs are stored as a SHA-256 digest of the canonicalised complex128
bytes (signed zeros folded to +0) plus a strided sample and the norm.
"""
from __future__ import annotations

import argparse
import contextlib
import hashlib
import io
import json
import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from paper_2405_01250_b200 import workloads as W  # noqa: E402


def canon(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.complex128) + np.complex128(0)


def digest(a) -> str:
    return hashlib.sha256(canon(a).tobytes()).hexdigest()


def sample_idx(n: int, count: int = 256) -> np.ndarray:
    return np.unique(np.linspace(0, n - 1, count).astype(np.int64))


def diaq_to_arrays(m):
    offs = np.asarray(m.diag_indices(), dtype=np.int64)
    vals = [m.get(int(d)).re + 1j * m.get(int(d)).im for d in offs]
    flat = np.concatenate(vals) if vals else np.zeros(0, np.complex128)
    return offs, flat


def ops_to_json(ops):
    return [[name, list(q), list(p)] for name, q, p in ops]


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--reference", default="/root/reference/pkg/src")
    args = ap.parse_args()
    sys.path.insert(0, args.reference)
    import diaqsim as R  # the reference
    from diaqsim import cli as RCLI

    t_start = time.time()
    meta = {
        "generator": "tests/golden/make_golden.py",
        "reference": args.reference,
        "numpy": np.__version__,
    }
    # which complex-multiply formula this host's numpy uses
    rng = np.random.default_rng(7)
    a = rng.normal(size=64) + 1j * rng.normal(size=64)
    b = rng.normal(size=64) + 1j * rng.normal(size=64)
    meta["numpy_cmul"] = "plain" if np.array_equal((a * b).real, a.real * b.real - a.imag * b.imag) else "fma"

    # ---- KATs: the reference unit tests' known answers, recomputed by the reference
    kats = {}
    corner = np.array([[1, 0, 0, 2], [0, 3, 0, 0], [0, 0, 4, 0], [5, 0, 0, 6]], dtype=complex)
    cx = np.array([[1, 0, 0, 0], [0, 1, 0, 0], [0, 0, 0, 1], [0, 0, 1, 0]], dtype=complex)
    ca = R.from_dense(corner, 0.0)
    kats["corner"] = {"offsets": ca.diag_indices(),
                      "re": {str(d): ca.get(d).re.tolist() for d in ca.diag_indices()}}
    kats["corner_spmv_ones"] = [[v.real, v.imag] for v in R.spmv(ca, np.ones(4, dtype=complex))]
    md = R.multiply_diagonals(ca.get(3), ca.get(-3), 4)
    kats["multiply_diagonals_corner"] = {"d_c": md[0], "re": md[1].re.tolist(), "im": md[1].im.tolist()}
    cxa = R.from_dense(cx, 0.0)
    kats["cx_layout"] = {"offsets": cxa.diag_indices(),
                         "re": {str(d): cxa.get(d).re.tolist() for d in cxa.diag_indices()}}
    x = R.from_dense(np.array([[0, 1], [1, 0]], dtype=complex), 0.0)
    kats["xx_offsets"] = R.matmul(x, x).diag_indices()
    z = R.from_dense(np.diag([1.0, -1.0]), 0.0)
    zz = R.matmul(z, z)
    kats["zz"] = {"offsets": zz.diag_indices(), "re": zz.get(0).re.tolist()}
    kz = R.kron_identity(2, z, 1)
    kats["kron_identity_z"] = {"offsets": kz.diag_indices(), "re": kz.get(0).re.tolist()}
    h = np.array([[1, 1], [1, -1]]) / np.sqrt(2)
    kh = R.kron_identity(2, R.from_dense(h, 0.0), 2)
    kats["kron_identity_h"] = {"offsets": kh.diag_indices(),
                               "dense": [[[v.real, v.imag] for v in row] for row in R.to_dense(kh)]}
    span_cases = [("cx", [0, 2], 3), ("cx", [2, 0], 3), ("cx", [1, 3], 4), ("swap", [3, 0], 4),
                  ("ccx", [0, 2, 4], 5), ("ccx", [4, 1, 2], 5), ("h", [1], 3)]
    kats["span"] = []
    for name, pos, span in span_cases:
        nq = R.gates.GATE_DEFS[name][0]
        g = R.gate_matrix(R.GateOp(name, tuple(range(nq))))
        u = R.build_span_unitary(g, pos, span)
        offs, flat = diaq_to_arrays(u)
        gd = R.to_dense(g)
        kats["span"].append({"name": name, "positions": pos, "span": span,
                             "g": [[[v.real, v.imag] for v in row] for row in gd],
                             "offsets": offs.tolist(),
                             "values": [[v.real, v.imag] for v in flat]})
    # catalog gate layouts (reference gates.py:81-101), params 0.3 + 0.2 i
    kats["catalog"] = {}
    for name, (nq, npar, _) in R.gates.GATE_DEFS.items():
        params = tuple(0.3 + 0.2 * i for i in range(npar))
        g = R.gate_matrix(R.GateOp(name, tuple(range(nq)), params))
        offs, flat = diaq_to_arrays(g)
        kats["catalog"][name] = {"params": list(params), "offsets": offs.tolist(),
                                 "values": [[v.real, v.imag] for v in flat]}
    # GHZ states and 1024-shot counts (reference test_acceptance.py:220-242)
    kats["ghz"] = {}
    for n in (2, 3, 4, 8, 12):
        ops = [("h", (0,), ())] + [("cx", (i, i + 1), ()) for i in range(n - 1)]
        c = R.Circuit(n, [R.GateOp(*o) for o in ops])
        res = R.run(c, backend="diaq", shots=1024, seed=0, emit_state=True)
        kats["ghz"][str(n)] = {"counts": res.counts, "digest": digest(res.state)}

    # ---- kernel JSON protocol (reference cli.py:251-287, frontend goldens)
    def kernel(op, request):
        buf = io.StringIO()
        old_in = sys.stdin
        sys.stdin = io.StringIO(json.dumps(request))
        try:
            with contextlib.redirect_stdout(buf):
                rc = RCLI.main(["kernel", op])
        finally:
            sys.stdin = old_in
        assert rc == 0
        return json.loads(buf.getvalue())

    def pairs(rows):
        return [[[float(v), 0.0] for v in row] for row in rows]

    proto = {}
    cd = pairs(corner.real.astype(int).tolist())
    wire = kernel("from-dense", {"dense": cd})
    proto["corner"] = {"dense": cd, "wire": wire, "round_trip": kernel("to-dense", {"a": wire})["dense"]}
    a_rows = [[(i + 1 if i == j else (i + 2 if j == i + 2 else 0)) for j in range(8)] for i in range(8)]
    b_rows = [[(2 * i + 1 if i == j else (i + 3 if j == i - 1 else 0)) for j in range(8)] for i in range(8)]
    aw = kernel("from-dense", {"dense": pairs(a_rows)})
    bw = kernel("from-dense", {"dense": pairs(b_rows)})
    cw = kernel("matmul", {"a": aw, "b": bw})
    xv = [[float(k % 5 - 2), float((k * k) % 3)] for k in range(8)]
    proto["matmul_case"] = {"a_dense": pairs(a_rows), "b_dense": pairs(b_rows), "a": aw, "b": bw,
                            "c": cw, "c_dense": kernel("to-dense", {"a": cw})["dense"], "x": xv,
                            "y": kernel("spmv", {"a": aw, "x": xv})["y"]}
    ghz4 = R.ghz_qasm(4)
    sim = kernel("simulate", {"qasm": ghz4, "seed": 7, "shots": 1024, "emit_state": True})
    circ = R.parse_circuit(ghz4)
    proto["ghz4_simulate"] = {"ops": [[op.name, list(op.qubits), list(op.params)] for op in circ.ops],
                              "n_qubits": circ.n_qubits, "seed": 7, "shots": 1024, "result": sim}
    with open(os.path.join(HERE, "kats.json"), "w") as f:
        json.dump({"meta": meta, "kats": kats, "kernel_protocol": proto}, f)

    # ---- config 1: spmv n=14
    c1 = W.config1(0)
    A1 = R.kron_identity(c1["left"], R.from_dense(c1["u"], 0.0), c1["right"])
    y1 = R.spmv(A1, c1["x"])
    np.savez(os.path.join(HERE, "config1_spmv.npz"), u=c1["u"], x=c1["x"], y=y1,
             offsets=np.asarray(A1.diag_indices()), a_values=diaq_to_arrays(A1)[1])

    # ---- config 2: spgemm n=12 + 64-pair sweep
    def c2_mats(seed):
        p = W.config2(seed)
        span = R.build_span_unitary(R.from_dense(p["u4"], 0.0), p["u4_positions"], p["u4_span"])
        A = R.kron_identity(p["a_left"], span, p["a_right"])
        B1 = R.kron_identity(p["b1_left"], R.from_dense(p["u2"], 0.0), p["b1_right"])
        B0 = R.kron_identity(p["b0_left"], R.from_dense(W.rz(p["theta"]), 0.0), p["b0_right"])
        B = R.matmul(B1, B0)
        return p, A, B1, B0, B, R.matmul(A, B)

    p, A, B1, B0, B, C = c2_mats(0)
    co, cv = diaq_to_arrays(C)
    bo, bv = diaq_to_arrays(B)
    np.savez(os.path.join(HERE, "config2_spgemm.npz"), u4=p["u4"], u2=p["u2"], theta=p["theta"],
             a_offsets=np.asarray(A.diag_indices()), b1_offsets=np.asarray(B1.diag_indices()),
             b0_offsets=np.asarray(B0.diag_indices()), b_offsets=bo, b_values=bv,
             c_offsets=co, c_values=cv)
    sweep = []
    for seed in range(64):
        _, _, _, _, Bs, Cs = c2_mats(seed)
        o, v = diaq_to_arrays(Cs)
        ob, vb = diaq_to_arrays(Bs)
        sweep.append({"seed": seed, "c_offsets": o.tolist(), "c_digest": digest(v),
                      "b_offsets": ob.tolist(), "b_digest": digest(vb)})

    # ---- random kernel cases (acceptance-suite style, test_acceptance.py:61-96)
    rng = np.random.default_rng(12345)

    def random_banded(n, n_diags):
        m = np.zeros((n, n), dtype=complex)
        offs = rng.choice(np.arange(-(n - 1), n), size=min(n_diags, 2 * n - 1), replace=False)
        for d in offs:
            ln = n - abs(int(d))
            vals = rng.normal(size=ln) + 1j * rng.normal(size=ln)
            if d >= 0:
                m[np.arange(ln), np.arange(ln) + d] = vals
            else:
                m[np.arange(ln) - d, np.arange(ln)] = vals
        return m

    cases = {}
    for i in range(48):
        n = int(rng.integers(2, 65))
        ma = random_banded(n, int(rng.integers(1, min(n, 9))) if n > 2 else 1)
        mb = random_banded(n, int(rng.integers(1, min(n, 9))) if n > 2 else 1)
        Cm = R.matmul(R.from_dense(ma, 0.0), R.from_dense(mb, 0.0))
        o, v = diaq_to_arrays(Cm)
        cases[f"mm{i}_a"] = ma
        cases[f"mm{i}_b"] = mb
        cases[f"mm{i}_c_offsets"] = o
        cases[f"mm{i}_c_values"] = v
    for i in range(100):
        n = int(rng.integers(2, 65))
        ma = random_banded(n, int(rng.integers(1, min(n, 9))) if n > 2 else 1)
        xv = rng.normal(size=n) + 1j * rng.normal(size=n)
        cases[f"mv{i}_a"] = ma
        cases[f"mv{i}_x"] = xv
        cases[f"mv{i}_y"] = R.spmv(R.from_dense(ma, 0.0), xv)
    for i in range(100):
        n_q = int(rng.integers(1, 4))
        lo = int(rng.integers(0, 4))
        hi_pad = int(rng.integers(0, 4))
        mm = random_banded(2**n_q, int(rng.integers(1, 2**n_q + 1)))
        dim_a, dim_b = 2**lo, 2**hi_pad
        xv = rng.normal(size=dim_a * 2**n_q * dim_b) + 1j * rng.normal(size=dim_a * 2**n_q * dim_b)
        pl = R.Placement(dim_a, R.from_dense(mm, 0.0), dim_b, lo, lo + n_q - 1, "rand")
        yv = R.apply_placed(pl, R.StateVector(lo + n_q + hi_pad, xv)).amps
        cases[f"ap{i}_m"] = mm
        cases[f"ap{i}_dims"] = np.array([dim_a, dim_b])
        cases[f"ap{i}_x"] = xv
        cases[f"ap{i}_y"] = yv
    np.savez_compressed(os.path.join(HERE, "random_cases.npz"), **cases)

    # ---- config 3: random layered circuit; n=12 full state, n=20 digest
    circuits = {}
    for n, layers, full in ((8, 10, True), (12, 40, True), (20, 40, False)):
        ops = W.random_layered_ops(n, layers, seed=0)
        c = R.Circuit(n, [R.GateOp(*o) for o in ops])
        t0 = time.time()
        res = R.run(c, backend="diaq", shots=1024, seed=0, span_limit=n, emit_state=True)
        rec = {"n": n, "layers": layers, "seed": 0, "ops": ops_to_json(ops),
               "digest": digest(res.state), "norm": float(np.linalg.norm(res.state)),
               "counts": res.counts, "ref_apply_s": res.timings_ns["apply_total"] * 1e-9,
               "wall_s": time.time() - t0}
        idx = sample_idx(2**n)
        rec["sample_idx"] = idx.tolist()
        rec["sample"] = [[v.real, v.imag] for v in res.state[idx]]
        if full:
            np.save(os.path.join(HERE, f"circuit_n{n}_state.npy"), res.state)
        circuits[str(n)] = rec
    # fusion case: repeated same-span gates so fuse_pass (-> matmul) fires
    fops = []
    for q in range(6):
        fops += [("rx", (q,), (0.3 + q,)), ("ry", (q,), (1.1 * q,)), ("rz", (q,), (0.7,))]
    fops += [("cx", (0, 3), ()), ("cx", (0, 3), ()), ("cx", (4, 1), ()), ("h", (2,), ()),
             ("u3", (5,), (0.1, 0.2, 0.3)), ("u3", (5,), (0.4, 0.5, 0.6)), ("swap", (1, 2), ()),
             ("cz", (2, 3), ()), ("ccx", (0, 2, 5), ()), ("ccx", (0, 2, 5), ())]
    fc = R.Circuit(6, [R.GateOp(*o) for o in fops])
    fus = {}
    for fusion in (False, True):
        res = R.run(fc, shots=512, seed=3, fusion=fusion, emit_state=True, span_limit=6)
        fus[str(fusion)] = {"state": [[v.real, v.imag] for v in res.state], "counts": res.counts,
                            "gates": len(res.timings_ns["per_gate"])}
    circuits["fusion_case"] = {"n": 6, "ops": ops_to_json(fops), "runs": fus}

    # ---- config 4 parity slice n=22
    c4 = W.config4(22, seed=0)
    span = R.build_span_unitary(R.from_dense(c4["u4"], 0.0), c4["positions"], c4["span"])
    A4 = R.kron_identity(c4["left"], span, c4["right"])
    t0 = time.perf_counter()
    y4 = R.spmv(A4, c4["x"])
    t_spmv = time.perf_counter() - t0
    idx = sample_idx(2**22)
    o4, v4 = diaq_to_arrays(A4)
    c4rec = {"n": 22, "offsets": o4.tolist(), "a_digest": digest(v4), "x_digest": digest(c4["x"]),
             "y_digest": digest(y4), "y_norm": float(np.linalg.norm(y4)),
             "sample_idx": idx.tolist(), "y_sample": [[v.real, v.imag] for v in y4[idx]],
             "ref_spmv_s": t_spmv, "u4": [[[v.real, v.imag] for v in row] for row in c4["u4"]]}
    # ---- analysis / memory models (reference analysis.py, memory.py)
    def recs(rs):
        return [[r.timestep, r.gate_name, r.sparsity, r.diag_count, r.nnz, r.memory_map()] for r in rs]

    ghz10 = R.Circuit(10, [R.GateOp("h", (0,))] + [R.GateOp("cx", (i, i + 1)) for i in range(9)])
    rl6_ops = W.random_layered_ops(6, 2, seed=2)
    rl6 = R.Circuit(6, [R.GateOp(*o) for o in rl6_ops])
    analysis = {
        "ghz10_chain": recs(R.chain_product_analysis(ghz10)),
        "ghz10_timestep": recs(R.timestep_analysis(ghz10)),
        "rl6_ops": ops_to_json(rl6_ops),
        "rl6_chain_left": recs(R.chain_product_analysis(rl6, span_limit=6)),
        "rl6_chain_right": recs(R.chain_product_analysis(rl6, span_limit=6, order="right")),
        "rl6_timestep_eps": recs(R.timestep_analysis(rl6, eps=1e-3, span_limit=6)),
        "memory": {
            "corner": R.estimate_map(R.from_dense(corner, 0.0)),
            "cx": R.estimate_map(R.from_dense(cx, 0.0)),
            "kron_h": R.estimate_map(kh),
        },
    }
    with open(os.path.join(HERE, "configs.json"), "w") as f:
        json.dump({"meta": meta, "config2_sweep": sweep, "circuits": circuits, "config4_n22": c4rec,
                   "analysis": analysis}, f)
    print(f"goldens written in {time.time() - t_start:.1f}s")
    return 0


if __name__ == "__main__":
    sys.exit(main())
