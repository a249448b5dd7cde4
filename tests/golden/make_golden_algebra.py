#!/usr/bin/env python3
"""Goldens for the matrix algebra around the hot path and the round-2 API
gaps, produced by running the REFERENCE diaqsim package (build container):

    python tests/golden/make_golden_algebra.py [--reference /root/reference/pkg/src]

Cases (inputs and the reference's outputs, all in algebra_cases.npz):
  * matmul of single-precision pairs (float32 x float32 -> float32 products
    and prune, matrix.py:218-250) and of mixed pairs (-> float64);
  * add / scale / kron / adjoint / transpose (matrix.py:281-355), float64
    and float32 operands;
  * build_span_unitary of a 5-qubit gate (gates.py:169-219);
  * apply_placed of an explicit Placement whose m stores 90 diagonals
    (sim.py:69-105, more than one 64-diagonal chunk).
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def banded(rng, n, nd, dtype):
    m = np.zeros((n, n), dtype=np.complex128)
    offs = rng.choice(np.arange(-(n - 1), n), size=min(nd, 2 * n - 1), replace=False)
    for d in offs:
        length = n - abs(int(d))
        v = rng.normal(size=length) + 1j * rng.normal(size=length)
        if rng.random() < 0.2:
            v[rng.integers(length)] = 0
        idx = np.arange(length)
        r = idx - min(int(d), 0)
        m[r, r + int(d)] = v
    if dtype == np.float32:
        m = m.real.astype(np.float32).astype(np.float64) + 1j * m.imag.astype(np.float32).astype(np.float64)
    return m


def flat(R, m):
    offs = np.asarray(m.diag_indices(), dtype=np.int64)
    re = np.concatenate([m.get(int(d)).re.astype(np.float64) for d in offs]) if len(offs) else np.zeros(0)
    im = np.concatenate([m.get(int(d)).im.astype(np.float64) for d in offs]) if len(offs) else np.zeros(0)
    return offs, re, im, str(m.dtype)


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--reference", default="/root/reference/pkg/src")
    args = ap.parse_args()
    sys.path.insert(0, args.reference)
    import diaqsim as R

    rng = np.random.default_rng(2024)
    out = {}
    cases = []

    def put(key, arr):
        out[key] = np.asarray(arr)

    def put_mat(key, m):
        offs, re, im, dt = flat(R, m)
        put(key + "_offs", offs)
        put(key + "_re", re)
        put(key + "_im", im)
        put(key + "_n", np.array([m.n_dim]))
        put(key + "_dtype", np.array([dt]))

    # matmul: single x single, single x double, with an exact-cancellation pair
    for i in range(24):
        n = int(rng.integers(4, 48))
        da = np.float32 if i % 3 != 2 else np.float64
        db = np.float32
        ma, mb = banded(rng, n, int(rng.integers(1, 7)), da), banded(rng, n, int(rng.integers(1, 7)), db)
        if i == 0:  # X @ X cancellation (prune) in single precision
            n = 2
            ma = mb = np.array([[0, 1], [1, 0]], dtype=np.complex128)
        A, B = R.from_dense(ma, dtype=da), R.from_dense(mb, dtype=db)
        put_mat(f"mm{i}_a", A)
        put_mat(f"mm{i}_b", B)
        put_mat(f"mm{i}_c", R.matmul(A, B))
        cases.append(("matmul", i))
    # add / scale / kron / adjoint / transpose
    for i in range(12):
        dt1 = np.float32 if i % 2 else np.float64
        dt2 = np.float32 if i % 4 in (1, 2) else np.float64
        n = int(rng.integers(3, 24))
        A = R.from_dense(banded(rng, n, int(rng.integers(1, 6)), dt1), dtype=dt1)
        B = R.from_dense(banded(rng, n, int(rng.integers(1, 6)), dt2), dtype=dt2)
        s = complex(rng.normal(), rng.normal())
        nb = int(rng.integers(2, 6))
        K = R.from_dense(banded(rng, nb, int(rng.integers(1, 5)), dt2), dtype=dt2)
        put_mat(f"alg{i}_a", A)
        put_mat(f"alg{i}_b", B)
        put_mat(f"alg{i}_k", K)
        put(f"alg{i}_s", np.array([s]))
        put_mat(f"alg{i}_add", R.add(A, B))
        put_mat(f"alg{i}_scale", R.scale(A, s))
        put_mat(f"alg{i}_kron", R.kron(A, K))
        put_mat(f"alg{i}_adjoint", R.adjoint(A))
        put_mat(f"alg{i}_transpose", R.transpose(A))
        cases.append(("algebra", i))
    # 5-qubit span embedding
    g = rng.normal(size=(32, 32)) + 1j * rng.normal(size=(32, 32))
    g[rng.random((32, 32)) < 0.3] = 0
    put("span5_g", g)
    put("span5_positions", np.array([6, 0, 3, 1, 5]))
    put_mat("span5_out", R.build_span_unitary(R.from_dense(g), [6, 0, 3, 1, 5], 7))
    # explicit placement with 90 stored diagonals
    m = banded(rng, 64, 90, np.float64)
    M = R.from_dense(m)
    p = R.Placement(dim_a=2, m=M, dim_b=4, span_lo=1, span_hi=6, name="wide")
    x = rng.normal(size=2 * 64 * 4) + 1j * rng.normal(size=2 * 64 * 4)
    y = R.sim.apply_placed(p, R.sim.StateVector(9, x.copy())).amps
    put_mat("wide_m", M)
    put("wide_x", x)
    put("wide_y", y)
    np.savez_compressed(os.path.join(HERE, "algebra_cases.npz"), **out)
    print(f"wrote {len(out)} arrays ({len(cases)} matmul/algebra cases) to tests/golden/algebra_cases.npz")
    return 0


if __name__ == "__main__":
    sys.exit(main())
