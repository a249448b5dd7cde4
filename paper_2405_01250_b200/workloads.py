"""Seeded synthetic inputs for the BASELINE.json configs.

BASELINE.json names no public suite; these generators produce inputs with
the configs' shapes and value distributions.  All randomness is
numpy.random.default_rng(seed); draw order is gate unitaries first, then
the state vector x.

* Haar(k): QR of a complex Ginibre matrix, columns re-phased by
  r_ii/|r_ii| (so the distribution is exactly Haar).
* x: normal(N) + 1j*normal(N), L2-normalised.

Qubit convention is the reference's: qubit 0 is the most significant basis
bit (reference gates.py:8-9), so a gate on qubit q has offsets
+-2^(n-1-q).
"""
from __future__ import annotations

import math

import numpy as np


def haar(rng: np.random.Generator, dim: int) -> np.ndarray:
    """Haar unitary by modified Gram-Schmidt in plain Python arithmetic.

    Same distribution as QR with the r_ii phase fix (MGS yields a positive
    real diagonal of R), but no LAPACK/BLAS: every operation is a correctly
    rounded IEEE op in a fixed order, so the gate is bit-identical on every
    host (fixtures stay valid on any GPU box).
    """
    z = rng.normal(size=(dim, dim)) + 1j * rng.normal(size=(dim, dim))
    cols = [[complex(z[i, j]) for i in range(dim)] for j in range(dim)]
    q = []
    for v in cols:
        v = list(v)
        for u in q:
            proj = sum((u[i].conjugate() * v[i] for i in range(dim)), 0j)
            v = [v[i] - proj * u[i] for i in range(dim)]
        nrm = math.sqrt(math.fsum(c.real * c.real + c.imag * c.imag for c in v))
        q.append([c / nrm for c in v])
    return np.ascontiguousarray(np.array(q, dtype=np.complex128).T)


def random_state(rng: np.random.Generator, n_amps: int) -> np.ndarray:
    """normal + 1j*normal, L2-normalised with an exactly rounded norm (math.fsum),
    so x is bit-identical on every host (no BLAS reduction order)."""
    re = rng.normal(size=n_amps)
    im = rng.normal(size=n_amps)
    nrm = math.sqrt(math.fsum(re * re) + math.fsum(im * im))
    x = np.empty(n_amps, dtype=np.complex128)
    x.real = re / nrm
    x.imag = im / nrm
    return x


def rz(theta: float) -> np.ndarray:
    """Reference gates.py:40-41."""
    return np.diag([np.exp(-0.5j * theta), np.exp(0.5j * theta)])


# -- config 1: single spmv, n=14 -------------------------------------------

def config1(seed: int = 0) -> dict:
    """kron_identity(2^8, from_dense(Haar2), 2^5) and a random x (n=14)."""
    rng = np.random.default_rng(seed)
    u = haar(rng, 2)
    x = random_state(rng, 2**14)
    return {"n": 14, "u": u, "left": 2**8, "right": 2**5, "x": x}


# -- config 2: spgemm gate fusion, n=12 ------------------------------------

def config2(seed: int = 0) -> dict:
    """A = kron_identity(2^2, span(Haar4,[0,5],6), 2^4);
    B = kron_identity(2^9, Haar2, 2^2) @ kron_identity(1, RZ(theta), 2^11)."""
    rng = np.random.default_rng(seed)
    u4 = haar(rng, 4)
    u2 = haar(rng, 2)
    theta = float(rng.uniform(0.0, 2.0 * math.pi))
    return {
        "n": 12,
        "u4": u4, "u4_positions": [0, 5], "u4_span": 6, "a_left": 2**2, "a_right": 2**4,
        "u2": u2, "b1_left": 2**9, "b1_right": 2**2,
        "theta": theta, "b0_left": 1, "b0_right": 2**11,
    }


# -- config 3 / 5: random layered circuit -----------------------------------

def random_layered_ops(n: int, layers: int, seed: int = 0) -> list[tuple[str, tuple, tuple]]:
    """Per layer: RX/RY/RZ (type uniform, angle U[0,2pi)) on every qubit,
    then CX on a seeded random perfect matching (perm pairs)."""
    rng = np.random.default_rng(seed)
    ops = []
    kinds = ["rx", "ry", "rz"]
    for _ in range(layers):
        for q in range(n):
            kind = kinds[int(rng.integers(3))]
            theta = float(rng.uniform(0.0, 2.0 * math.pi))
            ops.append((kind, (q,), (theta,)))
        perm = rng.permutation(n)
        for i in range(n // 2):
            ops.append(("cx", (int(perm[2 * i]), int(perm[2 * i + 1])), ()))
    return ops


# -- config 4: bandwidth-bound large spmv ------------------------------------

def config4(n: int = 28, seed: int = 0, with_x: bool = True) -> dict:
    """Offsets {0, +-8, +-2^21, +-(2^21 +- 8)}: kron_identity(2^(n-22),
    build_span_unitary(Haar4, [18, 0], 19), 2^3).  n=22 is the parity slice
    (same offsets), n=28 the measured size."""
    if n < 22:
        raise ValueError("config 4 needs n >= 22")
    rng = np.random.default_rng(seed)
    u4 = haar(rng, 4)
    out = {"n": n, "u4": u4, "positions": [18, 0], "span": 19, "left": 2 ** (n - 22),
           "right": 2**3}
    if with_x:
        out["x"] = random_state(rng, 2**n)
    return out


def algorithmic_spmv_bytes(n_dim: int, offsets) -> int:
    """16 * sum(N - |d|) + 32 * N (diagonals + x + y)."""
    return 16 * sum(n_dim - abs(int(d)) for d in offsets) + 32 * n_dim
