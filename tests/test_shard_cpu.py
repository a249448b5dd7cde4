"""Multi-process (gloo, world_size 2 and 4) tests of the sharded-state host logic.

The ranks run the real planning/exchange code of paper_2405_01250_b200.shard
(diaq_shard_plan from the C-ABI, partner schedule, batched send/recv); the
per-rank arithmetic is a numpy stand-in of the CUDA multi-source kernel
defined here (the device kernel itself is covered by tests/test_gpu_shard.py).
The gathered state must equal the single-process oracle bitwise.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2405_01250_b200 import workloads as W


def numpy_apply(n_bits, local_bits, g, shifts, rank, srcs, y, cmul_mode):
    """CPU stand-in of diaq_apply_gate_sharded: rows of this rank, columns
    gathered from the source blocks, summed in ascending embedding order."""
    from paper_2405_01250_b200.shard import global_shifts
    k = len(shifts)
    g = np.asarray(g)
    idx = (rank << local_bits) + np.arange(1 << local_bits, dtype=np.int64)
    emb = [sum(((c >> (k - 1 - i)) & 1) << shifts[i] for i in range(k)) for c in range(1 << k)]
    gate_mask = sum(1 << s for s in shifts)
    rg = np.zeros_like(idx)
    for i, s in enumerate(shifts):
        rg |= ((idx >> s) & 1) << (k - 1 - i)
    free = idx & ~gate_mask
    gs = global_shifts(shifts, local_bits)
    acc = np.zeros(len(idx), dtype=np.complex128)
    xs = [None if t is None else t.numpy() for t in srcs]
    for cg in sorted(range(1 << k), key=lambda c: emb[c]):
        coef = g[rg, cg]
        nz = coef != 0
        if not nz.any():
            continue
        col = free | emb[cg]
        block = np.zeros_like(idx)
        for j, s in enumerate(gs):
            block |= ((col >> s) & 1) << (len(gs) - 1 - j)
        vals = np.zeros(len(idx), dtype=np.complex128)
        for b in np.unique(block[nz]):
            sel = nz & (block == b)
            vals[sel] = xs[int(b)][col[sel] & ((1 << local_bits) - 1)]
        term = coef * vals  # numpy complex multiply: the reference's rounding on this host
        acc[nz] = acc[nz] + term[nz]
    y.copy_(torch.from_numpy(acc))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, ops, out_q, remap=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2405_01250_b200 as D
        from paper_2405_01250_b200.shard import ShardedState, TorchDistComm
        comm = TorchDistComm()
        st = ShardedState.basis(n, comm, device=torch.device("cpu"), apply_fn=numpy_apply)
        pls = D.compile_circuit(D.Circuit(n, [D.GateOp(*o) for o in ops]), span_limit=n)
        st.apply_placements(pls, cmul_mode=O.numpy_cmul_mode(), remap=remap)
        nrm = st.norm()
        full = st.gather()
        if rank == 0:
            out_q.put((full.numpy(), nrm, st.stats))
    finally:
        dist.destroy_process_group()


def run_world(world: int, n: int, ops, remap: bool = False):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, ops, q, remap)) for r in range(world)]
    for p in procs:
        p.start()
    import queue
    import time
    deadline = time.time() + 300
    res = None
    while res is None:
        try:
            res = q.get(timeout=2)
        except queue.Empty:
            if any(p.exitcode not in (None, 0) for p in procs) or time.time() > deadline:
                for p in procs:
                    p.kill()
                raise AssertionError("a sharded worker failed") from None
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_random_layered_circuit_matches_oracle(world):
    n = 8
    ops = W.random_layered_ops(n, 3, seed=4)
    ops += [("ccx", (0, 5, 1), ()), ("swap", (1, 6), ()), ("cz", (0, 1), ()), ("rz", (0,), (0.3,)),
            ("u3", (1,), (0.1, 0.2, 0.3)), ("cx", (7, 0), ()), ("cx", (0, 7), ())]
    full, nrm, stats = run_world(world, n, ops)
    want = O.run_circuit(n, ops, cmul_mode=O.numpy_cmul_mode())
    assert np.array_equal(full, want)
    assert abs(nrm - 1.0) < 1e-12
    assert stats["gates"] == len(ops)
    assert stats["exchanged"] > 0 and stats["local"] > 0


def test_exchange_schedule_rules():
    """Cross-shard rules of SURVEY 8(e): diagonal gates and global controls
    need no partner; a flip of global bit g needs rank r ^ (1 << (g-L))."""
    from paper_2405_01250_b200 import gates as G
    from paper_2405_01250_b200.shard import exchange_schedule
    n, lb, world = 6, 4, 4
    rx = G.GATE_DEFS["rx"][2](0.7)
    rz = G.GATE_DEFS["rz"][2](0.7)
    cx = G.GATE_DEFS["cx"][2]()
    # RX on global bit 5 (reference qubit 0)
    needs = exchange_schedule(n, lb, rx, [5], world)
    for r in range(world):
        assert sorted(needs[r].values()) == sorted({r, r ^ 2})
    # RZ on a global bit: own block only
    needs = exchange_schedule(n, lb, rz, [4], world)
    assert all(list(nd.values()) == [r] for r, nd in enumerate(needs))
    # CX with global control (bit 5) and local target (bit 0): no communication
    needs = exchange_schedule(n, lb, cx, [5, 0], world)
    assert all(list(nd.values()) == [r] for r, nd in enumerate(needs))
    # CX with local control, global target (bit 4): partner r ^ 1
    needs = exchange_schedule(n, lb, cx, [0, 4], world)
    for r in range(world):
        assert sorted(needs[r].values()) == sorted({r, r ^ 1})
    # CX with both operands global: control=1 ranks read the target partner
    needs = exchange_schedule(n, lb, cx, [5, 4], world)
    for r in range(world):
        want = {r} if not (r >> 1) & 1 else {r ^ 1}
        assert set(needs[r].values()) == want


def test_cross_shard_fraction_matches_survey():
    """Counts quoted in SURVEY 8(e) for the config-5 generator (seed 0, 20 layers)."""
    from paper_2405_01250_b200 import gates as G
    from paper_2405_01250_b200.shard import exchange_schedule
    for n, world, want in ((31, 2, 18), (32, 4, 44), (33, 8, 65)):
        lb = n - (world.bit_length() - 1)
        ops = W.random_layered_ops(n, 20, seed=0)
        crosses = 0
        for name, qubits, params in ops:
            g = G.GATE_DEFS[name][2](*params)
            shifts = [n - 1 - q for q in qubits]
            if all(s < lb for s in shifts):
                continue
            needs = exchange_schedule(n, lb, g, shifts, world)
            if any(src != r for r in range(world) for src in needs[r].values()):
                crosses += 1
        assert crosses == want, (n, world, crosses)


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_remap_matches_oracle(world):
    """Qubit remapping (shard.remap_plan): global qubits swapped into local
    positions before cross-shard gates, layout restored at the end; the
    gathered state is still bitwise the oracle's (one-qubit and permutation
    gates only), with fewer partner reads than without remapping."""
    n = 8
    ops = W.random_layered_ops(n, 4, seed=7)
    ops += [("ccx", (0, 5, 1), ()), ("swap", (1, 6), ()), ("cz", (0, 1), ()), ("cx", (7, 0), ())]
    full, nrm, stats = run_world(world, n, ops, remap=True)
    want = O.run_circuit(n, ops, cmul_mode=O.numpy_cmul_mode())
    assert np.array_equal(full, want)
    assert abs(nrm - 1.0) < 1e-12
    assert stats["swaps"] > 0
    _, _, base = run_world(world, n, ops)
    assert stats["bytes_received"] < base["bytes_received"]
    # staged transport: a remapping swap moves half a shard, packed
    shard = 16 * 2 ** (n - (world.bit_length() - 1))
    assert stats["bytes_received"] % (shard // 2) == 0
    assert stats["bytes_received"] < stats["exchanged"] * shard


def _dense_apply(x, g, shifts):
    """numpy reference of one compact gate on a full 2^n vector (host test)."""
    n = int(np.log2(len(x)))
    k = len(shifts)
    idx = np.arange(len(x))
    rg = np.zeros_like(idx)
    for i, s in enumerate(shifts):
        rg |= ((idx >> s) & 1) << (k - 1 - i)
    free = idx & ~sum(1 << s for s in shifts)
    y = np.zeros_like(x)
    for c in range(1 << k):
        col = free.copy()
        for i, s in enumerate(shifts):
            col |= ((c >> (k - 1 - i)) & 1) << s
        y += np.asarray(g)[rg, c] * x[col]
    return y


@pytest.mark.parametrize("n,world", [(8, 2), (9, 4), (10, 8)])
def test_remap_plan_is_a_relabelling(n, world):
    """The physical program (swaps + relabelled gates, layout restored)
    computes the logical circuit; swaps are SWAP gates on one global and one
    local bit, and every remaining cross-shard gate still needs its partner."""
    from paper_2405_01250_b200 import gates as G
    from paper_2405_01250_b200.shard import remap_plan
    rng = np.random.default_rng(n)
    ops = W.random_layered_ops(n, 3, seed=n)
    ops.append(("u3", (0,), (0.1, 0.2, 0.3)))
    comps = [(np.asarray(G.GATE_DEFS[nm][2](*pr), dtype=np.complex128), [n - 1 - q for q in qs]) for nm, qs, pr in ops]
    lb = n - (world.bit_length() - 1)
    phys, nsw = remap_plan(n, lb, world, comps)
    assert nsw > 0 and len(phys) == len(comps) + nsw
    x = rng.normal(size=2**n) + 1j * rng.normal(size=2**n)
    a, b = x.copy(), x.copy()
    for g, sh in comps:
        a = _dense_apply(a, g, sh)
    for g, sh in phys:
        b = _dense_apply(b, g, sh)
    assert np.allclose(a, b, rtol=0, atol=1e-12)
    # no remapping needed on one shard
    same, k = remap_plan(n, n, 1, comps)
    assert k == 0 and all(sa == sb for (_, sa), (_, sb) in zip(same, comps))


def test_remap_cuts_partner_reads_config5():
    """Config-5 generator (seed 0, 20 layers) at n=33 on 8 shards: remapping
    turns 65 cross-shard gates reading 52 partner shards into 36 cross-shard
    operations (mostly half-shard swaps) reading 17.5 shards' worth."""
    from paper_2405_01250_b200 import gates as G
    from paper_2405_01250_b200.shard import exchange_schedule, partner_rows, remap_plan
    n, world = 33, 8
    lb = n - 3
    ops = W.random_layered_ops(n, 20, seed=0)
    comps = [(np.asarray(G.GATE_DEFS[nm][2](*pr), dtype=np.complex128), [n - 1 - q for q in qs]) for nm, qs, pr in ops]

    def reads(prog):
        cross, shards = 0, 0.0
        for g, sh in prog:
            if all(s < lb for s in sh):
                continue
            needs = exchange_schedule(n, lb, g, sh, world)
            if any(src != r for r in range(world) for src in needs[r].values()):
                cross += 1
                fr = partner_rows(lb, g, sh, 0)
                shards += sum(f for b, f in fr.items() if needs[0].get(b, 0) != 0)
        return cross, shards

    assert reads(comps) == (65, 52.0)
    phys, nsw = remap_plan(n, lb, world, comps)
    assert reads(phys) == (36, 17.5)


def test_collective_device_follows_backend():
    """host-side collectives must use CUDA tensors under NCCL
    (torch registers NCCL for "cuda" only) and CPU tensors under gloo."""
    from paper_2405_01250_b200.shard import collective_device
    assert collective_device("nccl", torch.device("cuda", 3)) == torch.device("cuda", 3)
    assert collective_device("NCCL", "cuda:1").type == "cuda"
    assert collective_device("gloo", torch.device("cuda", 0)).type == "cpu"
    assert collective_device("gloo", None).type == "cpu"


def _order_worker(rank, world, port, out_q):
    """PeerComm.order() protocol with the device calls recorded instead of
    issued: record own event k, gloo barrier, wait on every partner's event
    k; k alternates between consecutive cross-shard gates."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2405_01250_b200 import _lib as L
        from paper_2405_01250_b200.shard import PeerComm
        log = []
        made = []
        L.ipc_event_create = lambda: made.append(1000 * (rank + 1) + len(made)) or made[-1]
        L.ipc_event_handle = lambda ev: str(ev).encode()
        L.ipc_event_open = lambda h: int(h.decode())
        L.event_record = lambda ev: log.append(("record", ev))
        L.stream_wait_event = lambda ev: log.append(("wait", ev))
        comm = PeerComm()
        assert comm.host_group is None or comm.backend == "gloo"
        for _ in range(3):
            comm.order()
        out_q.put((rank, log))
    finally:
        dist.destroy_process_group()


def test_peer_order_protocol_gloo():
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_order_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    logs = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r, log in logs.items():
        assert len(log) == 3 * world  # per gate: 1 record + (world - 1) waits
        for g in range(3):
            step = log[g * world:(g + 1) * world]
            # own event g % 2 (two alternate), then event g % 2 of every partner
            assert step[0] == ("record", 1000 * (r + 1) + g % 2)
            assert sorted(ev for _, ev in step[1:]) == [1000 * (q + 1) + g % 2 for q in range(world) if q != r]
            assert all(kind == "wait" for kind, _ in step[1:])
