"""GPU: the sharded path (multi-source kernel + exchange plans) emulated on
one device with P = 2, 4, 8 ranks, against the reference goldens (bitwise)
and the unsharded run.  Multi-process host logic: tests/test_shard_cpu.py."""
from __future__ import annotations

import os

import numpy as np
import pytest

import paper_2405_01250_b200 as D
from conftest import GOLDEN, digest
from paper_2405_01250_b200 import _lib as L
from paper_2405_01250_b200 import workloads as W
from paper_2405_01250_b200.shard import run_emulated

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cmul(configs):
    return L.CMUL_FMA if configs["meta"]["numpy_cmul"] == "fma" else L.CMUL_PLAIN


@pytest.fixture(params=[0, 11, 12], ids=["gate-by-gate", "fused11", "fused12"], autouse=True)
def fuse_mode(request):
    old = D.sim.FUSE_TILE_BITS
    D.sim.FUSE_TILE_BITS = request.param
    yield request.param
    D.sim.FUSE_TILE_BITS = old


def _full(shards):
    import torch
    return torch.cat(shards).cpu().numpy()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_n12_matches_reference(configs, cmul, world):
    rec = configs["circuits"]["12"]
    ops = W.random_layered_ops(12, rec["layers"], rec["seed"])
    pls = D.compile_circuit(D.Circuit(12, [D.GateOp(*o) for o in ops]), span_limit=12)
    shards, stats = run_emulated(12, world, pls, cmul_mode=cmul)
    want = np.load(os.path.join(GOLDEN, "circuit_n12_state.npy"))
    assert np.array_equal(_full(shards), want)
    assert stats["exchanged"] > 0


@pytest.mark.parametrize("remap", [False, True], ids=["plain", "remap"])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_n20_matches_reference_digest(configs, cmul, world, remap):
    """remap: global qubits swapped into local positions before cross-shard
    gates (shard.remap_plan) -- still bitwise the reference (config-5 mix)."""
    rec = configs["circuits"]["20"]
    ops = W.random_layered_ops(20, rec["layers"], rec["seed"])
    pls = D.compile_circuit(D.Circuit(20, [D.GateOp(*o) for o in ops]), span_limit=20)
    shards, stats = run_emulated(20, world, pls, cmul_mode=cmul, remap=remap)
    assert digest(_full(shards)) == rec["digest"]
    if remap:
        assert stats["swaps"] > 0


def test_sharded_mixed_gates_match_unsharded(cmul):
    n = 10
    ops = W.random_layered_ops(n, 2, seed=9)
    ops += [("ccx", (0, 1, 2), ()), ("ccx", (2, 0, 9), ()), ("ccx", (9, 8, 0), ()), ("swap", (0, 9), ()),
            ("swap", (1, 0), ()), ("cz", (0, 1), ()), ("u3", (0,), (0.1, 0.2, 0.3)), ("h", (2,), ()),
            ("cx", (2, 1), ()), ("y", (1,), ())]
    pls = D.compile_circuit(D.Circuit(n, [D.GateOp(*o) for o in ops]), span_limit=n)
    want = D.run_gates(D.init_state(n), pls, cmul_mode=cmul).amps
    for world in (2, 4, 8):
        shards, _ = run_emulated(n, world, pls, cmul_mode=cmul)
        assert np.array_equal(_full(shards), want), world
        shards, _ = run_emulated(n, world, pls, cmul_mode=cmul, remap=True)
        assert np.array_equal(_full(shards), want), ("remap", world)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_spmv_config4_slice(world):
    """Row-sharded spmv with x read across shard boundaries (config-4
    offsets +-2^21 +-8 cross every boundary at n=22), emulated on one GPU:
    the concatenated rank outputs are bitwise the single-GPU spmv."""
    import torch
    from paper_2405_01250_b200.shard import ShardedDiaq
    c4 = W.config4(22, seed=0, with_x=True)
    span = D.build_span_unitary(D.from_dense(c4["u4"], 0.0), c4["positions"], c4["span"])
    a = D.kron_identity(1, span, c4["right"])
    x = torch.from_numpy(c4["x"]).cuda()
    want = D.spmv(a, x).cpu().numpy()
    parts = list(x.chunk(world))
    got = [ShardedDiaq.from_matrix(a, r, world).spmv(parts) for r in range(world)]
    assert np.array_equal(torch.cat(got).cpu().numpy(), want)


def test_sharded_spmv_ragged_offsets():
    """Offsets of every sign and size, including |d| > one shard."""
    import torch
    from paper_2405_01250_b200.shard import ShardedDiaq
    rng = np.random.default_rng(3)
    n = 256
    offs = [-200, -65, -64, -3, 0, 1, 63, 64, 130, 255]
    m = np.zeros((n, n), dtype=complex)
    for d in offs:
        k = np.arange(n - abs(d))
        r, c = (k, k + d) if d >= 0 else (k - d, k)
        m[r, c] = rng.normal(size=len(k)) + 1j * rng.normal(size=len(k))
    a = D.from_dense(m, 0.0)
    x = torch.from_numpy(rng.normal(size=n) + 1j * rng.normal(size=n)).cuda()
    want = D.spmv(a, x).cpu().numpy()
    for world in (2, 4, 8):
        parts = list(x.chunk(world))
        got = torch.cat([ShardedDiaq.from_matrix(a, r, world).spmv(parts) for r in range(world)])
        assert np.array_equal(got.cpu().numpy(), want), world


@pytest.mark.parametrize("seed", range(4))
def test_sharded_fuzz(cmul, seed):
    """Seeded random circuits (rotations, CX/SWAP chains with controls and
    targets on global bits, CZ, CCX, Haar4) on emulated shards: fused local
    runs with rank-dependent controls, permutation tails, and exchanges,
    bitwise against the single-state run."""
    n, pls = _shard_fuzz_circuit(seed, 12, 17)
    want = D.run_gates(D.init_state(n), pls, cmul_mode=cmul).amps
    for world in (2, 4):
        shards, _ = run_emulated(n, world, pls, cmul_mode=cmul)
        assert np.array_equal(_full(shards), want), (seed, n, world)


@pytest.mark.parametrize("seed", range(4, 10))
def test_sharded_fuzz_specialised_passes(cmul, seed):
    """The same circuits on shards large enough for tiled passes, with the
    NVRTC-specialised kernels compiled before they run (fused_jit 2: rank
    bits in the selector base, rank-dependent constants of the permutation
    maps): bitwise against the single-state run, and within 1e-12 under the
    contracted arithmetic."""
    from paper_2405_01250_b200 import _lib as L
    n, pls = _shard_fuzz_circuit(seed, 15, 19)
    want = D.run_gates(D.init_state(n), pls, cmul_mode=cmul).amps
    try:
        L.tune("fused_jit", 2)
        for world in (2, 4):
            shards, _ = run_emulated(n, world, pls, cmul_mode=cmul)
            assert np.array_equal(_full(shards), want), (seed, n, world)
            shards, _ = run_emulated(n, world, pls, cmul_mode=L.CMUL_CONTRACT)
            got = _full(shards)
            assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-12, (seed, n, world)
    finally:
        L.tune("fused_jit", 1)


def _shard_fuzz_circuit(seed, nlo, nhi):
    rng = np.random.default_rng(500 + seed)
    n = int(rng.integers(nlo, nhi))
    ops = []
    for _ in range(int(rng.integers(30, 60))):
        q = [int(v) for v in rng.choice(np.arange(2, n), size=3, replace=False)]  # qubits 0, 1: the global bits
        if rng.integers(3) == 0:
            q[0] = int(rng.integers(2))
        k = int(rng.integers(6))
        if k == 0:
            ops.append((["rx", "ry", "rz", "h"][int(rng.integers(4))], (q[0],), (0.4,) if k == 0 else ()))
        elif k == 1:
            ops += [("cx", (q[0], q[1]), ()), ("cx", (1 - (q[0] & 1) if q[0] < 2 else 0, q[2]), ()),
                    ("cx", (q[2], 1), ())]
        elif k == 2:
            ops += [("swap", (q[0], q[1]), ()), ("x", (q[2],), ())]
        elif k == 3:
            ops += [("cz", (q[0], q[1]), ()), ("ccx", tuple(q), ())]
        else:
            ops += [("ry", (q[1],), (1.3,)), ("rz", (0,), (0.9,))]
    ops = [(a, b, c if a in ("rx", "ry", "rz") else ()) for a, b, c in ops]
    pls = D.compile_circuit(D.Circuit(n, [D.GateOp(*o) for o in ops]), span_limit=n)
    a, b = (int(v) for v in rng.choice(n, size=2, replace=False))
    lo, hi = min(a, b), max(a, b)
    pls.append(D.Placement(2**lo, None, 2 ** (n - 1 - hi), lo, hi, "haar", gate=(W.haar(rng, 4), [a - lo, b - lo])))
    return n, pls
