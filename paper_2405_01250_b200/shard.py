"""Sharded state vector over several GPUs (no reference counterpart).

The 2^n state is split over P = 2^p ranks by its top p bits (reference
qubits 0..p-1, since qubit 0 is the most significant bit): rank r owns
indices [r*2^L, (r+1)*2^L), L = n - p.  For every gate:

* all operands local (bits < L): no communication, the single-GPU kernel;
* some operands global: diaq_shard_plan tells each rank which column blocks
  its rows read.  Block-diagonal gates in the global bits (RZ/diagonal gates
  on any qubit, CX with a global control) read only the rank's own block --
  no communication.  Otherwise every rank sends its shard to the ranks that
  read it and receives the partner shards it reads (NCCL send/recv over
  NVLink/NVSwitch via torch.distributed, or any comm with the same
  interface), then diaq_apply_gate_sharded combines own + partner blocks.

The per-amplitude summation order equals the single-GPU path's, so a sharded
run is bitwise equal to the unsharded one.  Norms are an all-reduce (sum)
of local |x|^2.  Timing is by CUDA events, max over ranks.

The host logic (plans, partner schedule, exchange) is independent of the
device: `apply_fn` defaults to the CUDA kernel; CPU tests inject a numpy
stand-in and run it over gloo with world_size 2 and 4.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib as L
from .gates import Placement


def gate_plan(n_bits: int, local_bits: int, g: np.ndarray, shifts, rank: int) -> tuple[int, int, int]:
    """(need_mask, n_global, own_block) for `rank` (host-only C-ABI call)."""
    gd = np.ascontiguousarray(g, dtype=np.complex128)
    sh = np.ascontiguousarray(shifts, dtype=np.int32)
    need = ctypes.c_uint32(0)
    kg = ctypes.c_int(0)
    vr = ctypes.c_uint32(0)
    L.call("diaq_shard_plan", n_bits, local_bits, len(sh), gd.ctypes.data, sh.ctypes.data, int(rank),
           ctypes.addressof(need), ctypes.addressof(kg), ctypes.addressof(vr))
    return int(need.value), int(kg.value), int(vr.value)


def global_shifts(shifts, local_bits: int) -> list[int]:
    """Global operand shifts in block-index order (descending shift = MSB first)."""
    return sorted((s for s in shifts if s >= local_bits), reverse=True)


def block_rank(rank: int, block: int, gshifts: list[int], local_bits: int) -> int:
    """Rank holding column block `block` for the rows of `rank`."""
    kg = len(gshifts)
    r = rank
    for j, s in enumerate(gshifts):
        bit = (block >> (kg - 1 - j)) & 1
        pos = s - local_bits
        r = (r & ~(1 << pos)) | (bit << pos)
    return r


def exchange_schedule(n_bits: int, local_bits: int, g, shifts, world: int):
    """needs[r] = {block: source rank} every rank reads, for all ranks."""
    gs = global_shifts(shifts, local_bits)
    needs = []
    for r in range(world):
        mask, _, _ = gate_plan(n_bits, local_bits, g, shifts, r)
        needs.append({b: block_rank(r, b, gs, local_bits) for b in range(1 << len(gs)) if (mask >> b) & 1})
    return needs


def partner_rows(local_bits: int, g: np.ndarray, shifts, rank: int) -> dict[int, float]:
    """{column block: fraction of this rank's rows that read it} -- what a
    kernel reading partner data in place (peer transport) fetches: RX on a
    global bit reads the whole partner shard, SWAP(global, local) half."""
    g = np.asarray(g)
    k = len(shifts)
    gs = global_shifts(shifts, local_bits)
    loc = [i for i in range(k) if shifts[i] < local_bits]
    glo = {i: (rank >> (shifts[i] - local_bits)) & 1 for i in range(k) if shifts[i] >= local_bits}
    use: dict[int, int] = {}
    for pat in range(1 << len(loc)):
        rg = 0
        for i in range(k):
            bit = glo[i] if i in glo else (pat >> loc.index(i)) & 1
            rg |= bit << (k - 1 - i)
        blocks = set()
        for c in np.nonzero(g[rg])[0]:
            b = 0
            for j, sh in enumerate(gs):
                i = list(shifts).index(sh)
                b |= ((int(c) >> (k - 1 - i)) & 1) << (len(gs) - 1 - j)
            blocks.add(b)
        for b in blocks:
            use[b] = use.get(b, 0) + 1
    return {b: u / (1 << len(loc)) for b, u in use.items()}


_SWAP = np.array([[1, 0, 0, 0], [0, 0, 1, 0], [0, 1, 0, 0], [0, 0, 0, 1]], dtype=np.complex128)


def mixing_operands(g: np.ndarray, k: int) -> list[int]:
    """Operands a k-qubit gate mixes: i is NOT mixing when g is block
    diagonal in it (g[r, c] == 0 whenever bit i of r and c differ) -- a
    control or a diagonal operand, which selects rows but moves nothing."""
    g = np.asarray(g)
    idx = np.arange(1 << k)
    out = []
    for i in range(k):
        b = (idx >> (k - 1 - i)) & 1
        if np.any(g[b[:, None] != b[None, :]] != 0):
            out.append(i)
    return out


def remap_plan(n_bits: int, local_bits: int, world: int, comps, restore: bool = True):
    """Qubit remapping for cross-shard gates ("ways to push
    toward linear"): before a gate that would read a partner shard because
    it mixes global bit g, swap g with a local bit v, so the gate (and every
    later gate on that qubit until it is displaced) runs locally.  The swap is
    a SWAP(g, v) gate through the ordinary exchange path; it moves half a
    shard each way (rows whose v bit differs from the rank's g bit) instead
    of the whole partner shard a cross-shard rotation reads.  Victim v:
    the local bit whose qubit's next mixing use is farthest ahead (Belady;
    controls and diagonal gates do not count), ties to the highest bit.
    Host-only and deterministic, so every rank plans the same swaps.

    comps: logical (g, shifts).  Returns (physical (g, shifts) list,
    number of swaps).  restore: end with the identity layout (swaps back),
    so the caller's amplitudes are in logical order after the run.

    Rounding: one-qubit and permutation gates are bitwise the unremapped
    path; a dense multi-qubit gate whose operands change relative order is
    summed in the physical column order (equal within fp64 rounding)."""
    l2p = list(range(n_bits))
    p2l = list(range(n_bits))
    mix = [[shifts[i] for i in mixing_operands(g, len(shifts))] for g, shifts in comps]
    # next mixing use of each logical bit after gate i (scanned backwards)
    nxt = [None] * len(comps)
    far = [len(comps)] * n_bits
    for i in range(len(comps) - 1, -1, -1):
        nxt[i] = far.copy()
        for s in mix[i]:
            far[s] = i
    out = []
    swaps = 0

    def swap(a: int, b: int):
        nonlocal swaps
        out.append((_SWAP, [a, b]))
        la, lb_ = p2l[a], p2l[b]
        p2l[a], p2l[b] = lb_, la
        l2p[la], l2p[lb_] = b, a
        swaps += 1

    for i, (g, shifts) in enumerate(comps):
        phys = [l2p[s] for s in shifts]
        if world > 1 and any(l2p[s] >= local_bits for s in mix[i]):
            needs = exchange_schedule(n_bits, local_bits, g, phys, world)
            if any(src != r for r, nd in enumerate(needs) for src in nd.values()):
                busy = set(phys)
                for s in mix[i]:
                    if l2p[s] < local_bits:
                        continue
                    cand = [v for v in range(local_bits) if v not in busy]
                    if not cand:
                        break
                    v = max(cand, key=lambda v: (nxt[i][p2l[v]], v))
                    busy.add(v)
                    swap(l2p[s], v)
                phys = [l2p[s] for s in shifts]
        out.append((g, phys))
    if restore:
        for q in range(n_bits):
            if l2p[q] != q:
                swap(l2p[q], q)
    return out, swaps


def _ptr(t):
    """device address of a source block: a tensor, a raw (peer) pointer, or None"""
    if t is None:
        return None
    return int(t) if isinstance(t, int) else t.data_ptr()


def _cuda_apply(n_bits, local_bits, g, shifts, rank, srcs, y, cmul_mode):
    gd = np.ascontiguousarray(g, dtype=np.complex128)
    sh = np.ascontiguousarray(shifts, dtype=np.int32)
    arr = (ctypes.c_void_p * len(srcs))(*[_ptr(t) for t in srcs])
    L.call("diaq_apply_gate_sharded", n_bits, local_bits, len(sh), gd.ctypes.data, sh.ctypes.data, int(rank),
           arr, y.data_ptr(), int(cmul_mode), L.stream_handle())


def collective_device(backend: str, like_device):
    """Device the tensors of a host-side collective must live on for
    `backend`: NCCL only moves CUDA tensors (torch registers it for "cuda"
    only), gloo moves CPU tensors everywhere and CUDA tensors for some ops
    only -- so CPU for everything but NCCL."""
    import torch
    if str(backend).lower() == "nccl":
        if like_device is not None and torch.device(like_device).type == "cuda":
            return torch.device(like_device)
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


class TorchDistComm:
    """torch.distributed transport (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.backend = str(dist.get_backend(group))

    def _dev(self, like=None):
        return collective_device(self.backend, getattr(like, "device", None))

    def exchange(self, sends, recvs) -> None:
        """sends: [(peer, tensor)], recvs: [(peer, tensor)] -- one batched group."""
        import torch
        re = torch.view_as_real  # complex128 travels as float64 pairs (gloo has no complex)
        ops = [self.dist.P2POp(self.dist.isend, re(t), p, self.group) for p, t in sends]
        ops += [self.dist.P2POp(self.dist.irecv, re(t), p, self.group) for p, t in recvs]
        if ops:
            for req in self.dist.batch_isend_irecv(ops):
                req.wait()

    def allreduce_sum(self, value: float, like=None) -> float:
        import torch
        t = torch.tensor([value], dtype=torch.float64, device=self._dev(like))
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return float(t.item())

    def allreduce_max(self, value: float, like=None) -> float:
        import torch
        t = torch.tensor([value], dtype=torch.float64, device=self._dev(like))
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return float(t.item())

    def gather(self, local):
        """Full state on rank 0 (tests only): every shard travels on the
        backend's device, the result is returned on `local`'s device."""
        import torch
        dev = self._dev(local)
        lr = torch.view_as_real(local).to(dev)
        parts = [torch.empty_like(lr) for _ in range(self.world)] if self.rank == 0 else None
        self.dist.gather(lr, parts, dst=0, group=self.group)
        return torch.view_as_complex(torch.cat(parts)).to(local.device) if self.rank == 0 else None


class PeerComm(TorchDistComm):
    """Peer-memory transport: every rank maps its partners' shard buffers
    (CUDA IPC, NVLink/NVSwitch peer access) and the multi-source kernel reads
    partner amplitudes directly inside the gate pass -- no staging copy, the
    transfer overlaps the arithmetic.  Cross-shard gates then run out of
    place into a second buffer (partners read this rank's current one): a
    rank only overwrites a buffer after every partner finished reading it,
    and only reads a partner's buffer after the partner finished writing it.

    That ordering is device-side (order()): each rank records an
    interprocess CUDA event on its stream, the ranks pass a host barrier on
    a gloo side group (it orders the enqueueing only -- no GPU is drained),
    and each stream waits on the partners' events.  Two events per rank
    alternate between consecutive cross-shard gates, so a fast rank cannot
    re-record an event a slow partner has yet to wait on.  torch.distributed
    (any backend; collectives on the backend's device) carries the handles
    and the reductions."""

    peer = True

    def __init__(self, group=None):
        super().__init__(group)
        self._opened: list[int] = []
        # host barriers on a CPU side group: an NCCL barrier would launch a
        # device collective and block the host on it
        if self.backend.lower() == "gloo":
            self.host_group = group
        else:
            ranks = list(range(self.dist.get_world_size())) if group is None else \
                self.dist.get_process_group_ranks(group)
            self.host_group = self.dist.new_group(ranks=ranks, backend="gloo")
        self._events = None  # ([own event x2], [[partner event x2] per rank])
        self._phase = 0

    def host_barrier(self) -> None:
        self.dist.barrier(group=self.host_group)

    def _share_events(self) -> None:
        own = [L.ipc_event_create() for _ in range(2)]
        handles = [L.ipc_event_handle(e) for e in own]
        allh = [None] * self.world
        self.dist.all_gather_object(allh, handles, group=self.host_group)
        peers = [[None, None] if q == self.rank else [L.ipc_event_open(h) for h in hs] for q, hs in enumerate(allh)]
        self._events = (own, peers)

    def order(self) -> None:
        """Device-side ordering before a cross-shard gate (see the class doc)."""
        if self._events is None:
            self._share_events()
        own, peers = self._events
        k = self._phase
        L.event_record(own[k])
        self.host_barrier()
        for q in range(self.world):
            if q != self.rank:
                L.stream_wait_event(peers[q][k])
        self._phase ^= 1

    def share(self, ptrs: list[int]) -> list[list[int]]:
        """table[q][i] = this process's address of rank q's buffer i.  Every
        rank learns whether every other one could map its partners, and all
        raise DeviceError together if one could not (no rank is left waiting
        in a collective the others skipped)."""
        err = None
        try:
            mine = [L.ipc_handle(p) for p in ptrs]
        except Exception as e:  # noqa: BLE001 -- reported to every rank below
            mine, err = None, repr(e)
        allh = [None] * self.world
        self.dist.all_gather_object(allh, mine, group=self.host_group)
        table, opened = [], []
        if err is None and all(h is not None for h in allh):
            try:
                for q, hs in enumerate(allh):
                    if q == self.rank:
                        table.append(list(ptrs))
                        continue
                    row = []
                    for h in hs:
                        row.append(L.ipc_open(h))
                        opened.append(row[-1])
                    table.append(row)
            except Exception as e:  # noqa: BLE001
                err = repr(e)
        else:
            err = err or "a partner could not export its buffers"
        errs = [None] * self.world
        self.dist.all_gather_object(errs, err, group=self.host_group)
        bad = [e for e in errs if e is not None]
        if bad:
            for ptr in opened:
                L.ipc_close(ptr)
            raise L.DeviceError(f"peer mapping failed: {bad[0]}")
        self._opened += opened
        return table

    def barrier(self) -> None:
        """Full barrier (setup and teardown): every rank's device work done."""
        L.torch().cuda.synchronize()
        self.host_barrier()

    def close(self) -> None:
        for p in self._opened:
            L.ipc_close(p)
        self._opened = []
        if self._events is not None:
            own, _ = self._events
            for e in own:
                L.event_destroy(e)
            self._events = None


class ShardedState:
    """This rank's 2^L amplitudes of a 2^n state split over `comm.world` ranks."""

    def __init__(self, n_qubits: int, local, comm, apply_fn=None):
        self.n_qubits = int(n_qubits)
        self.comm = comm
        world = comm.world
        if world & (world - 1):
            raise ValueError(f"world size {world} is not a power of two")
        self.p = world.bit_length() - 1
        self.local_bits = self.n_qubits - self.p
        if self.local_bits < 1:
            raise ValueError("more shards than amplitudes")
        self.apply_fn = apply_fn or _cuda_apply
        self.stats = {"gates": 0, "local": 0, "no_comm_global": 0, "exchanged": 0, "bytes_received": 0}
        self._recv = {}
        self.peer = bool(getattr(comm, "peer", False))
        if self.peer:  # two exportable buffers: the current state and the next cross-shard result
            bufs = [L.shared_c128(local.numel()) for _ in range(2)]
            self._bufs = [t for t, _ in bufs]
            self._bufs[0].copy_(local)
            self._peer = comm.share([p for _, p in bufs])  # [rank][buffer] -> address here
            self._cur = 0
            local = self._bufs[0]
        self.local = local

    @classmethod
    def basis(cls, n_qubits: int, comm, device=None, apply_fn=None) -> "ShardedState":
        """|0...0> split over the ranks (reference init_state, sim.py:53-59)."""
        import torch
        world = comm.world
        lb = n_qubits - (world.bit_length() - 1)
        dev = device if device is not None else L.device()
        local = torch.zeros(2**lb, dtype=torch.complex128, device=dev)
        if comm.rank == 0:
            local[0] = 1.0
        return cls(n_qubits, local, comm, apply_fn)

    def _recv_buffer(self, peer: int):
        import torch
        buf = self._recv.get(peer)
        if buf is None or buf.numel() != self.local.numel():
            buf = torch.empty_like(self.local)
            self._recv[peer] = buf
        return buf

    def apply_gate(self, g: np.ndarray, shifts, cmul_mode: int) -> None:
        """One compact gate (operand i on state bit shifts[i]) on the sharded state."""
        n, lb, me = self.n_qubits, self.local_bits, self.comm.rank
        self.stats["gates"] += 1
        if all(s < lb for s in shifts):
            self.stats["local"] += 1
            self.apply_fn(n, lb, g, shifts, me, [self.local], self.local, cmul_mode)
            return
        needs = exchange_schedule(n, lb, g, shifts, self.comm.world)
        if self.peer and any(src != r for r, nd in enumerate(needs) for src in nd.values()):
            self._apply_peer(g, shifts, needs, cmul_mode)
            return
        if g is _SWAP and sum(s >= lb for s in shifts) == 1:
            self._swap_staged(*sorted(shifts, reverse=True))
            return
        sends = [(q, self.local) for q in range(self.comm.world) if q != me and me in needs[q].values()]
        recvs = [(src, self._recv_buffer(src)) for src in sorted(set(needs[me].values())) if src != me]
        if recvs or sends:
            self.stats["exchanged"] += 1
            self.stats["bytes_received"] += 16 * self.local.numel() * len(recvs)
            self.comm.exchange(sends, recvs)
        else:
            self.stats["no_comm_global"] += 1
        kg = len(global_shifts(shifts, lb))
        srcs = [None] * (1 << kg)
        for b, src in needs[me].items():
            srcs[b] = self.local if src == me else self._recv[src]
        self.apply_fn(n, lb, g, shifts, me, srcs, self.local, cmul_mode)

    def _swap_staged(self, gbit: int, vbit: int) -> None:
        """Remapping swap of global bit gbit and local bit vbit over the staged
        transport: only the half shard whose v bit differs from this rank's g
        bit crosses (packed, one send/recv with the partner), in place --
        pure copies, bitwise the SWAP gate."""
        lb, me = self.local_bits, self.comm.rank
        a = (me >> (gbit - lb)) & 1
        partner = me ^ (1 << (gbit - lb))
        view = self.local.view(-1, 2, 1 << vbit)[:, 1 - a, :]
        send = view.contiguous()
        recv = self._recv_buffer(partner)[: send.numel()].view_as(send)
        self.stats["exchanged"] += 1
        self.stats["bytes_received"] += 16 * send.numel()
        self.comm.exchange([(partner, send)], [(partner, recv)])
        view.copy_(recv)

    def _apply_peer(self, g, shifts, needs, cmul_mode) -> None:
        """Cross-shard gate reading partner shards in place over peer memory."""
        n, lb, me = self.n_qubits, self.local_bits, self.comm.rank
        self.comm.order()  # partners finished writing their current buffers / reading our next one (device-side)
        kg = len(global_shifts(shifts, lb))
        srcs = [None] * (1 << kg)
        for b, src in needs[me].items():
            srcs[b] = self.local if src == me else self._peer[src][self._cur]
        frac = partner_rows(lb, g, shifts, me)
        self.stats["exchanged"] += 1
        self.stats["bytes_received"] += int(16 * self.local.numel() *
                                            sum(f for b, f in frac.items() if needs[me].get(b, me) != me))
        nxt = self._bufs[self._cur ^ 1]
        self.apply_fn(n, lb, g, shifts, me, srcs, nxt, cmul_mode)
        self._cur ^= 1
        self.local = nxt

    def _needs_exchange(self, g, shifts) -> bool:
        lb = self.local_bits
        if all(s < lb for s in shifts):
            return False
        needs = exchange_schedule(self.n_qubits, lb, g, shifts, self.comm.world)
        return any(src != r for r, nd in enumerate(needs) for src in nd.values())

    def apply_placements(self, placements: list[Placement], cmul_mode: int | None = None,
                         remap: bool = False) -> None:
        """Apply gates in order.  On the GPU every maximal run of gates that
        needs no partner data (the same decision on every rank) goes through
        one fused native call (diaq_run_gates_local: shared-memory multi-gate
        passes, global-bit controls read from the rank index); cross-shard
        gates exchange and use the multi-source kernel.  remap: swap a
        global qubit with a local one before a gate that would read a
        partner shard (remap_plan); the layout is restored at the end."""
        from . import sim
        mode = sim.CMUL_MODE if cmul_mode is None else cmul_mode
        comps = []
        for p in placements:
            comp = p.compact()
            if comp is None:
                raise ValueError(f"sharded apply needs compact placements, got {p!r}")
            comps.append(comp)
        if remap:
            comps, nsw = remap_plan(self.n_qubits, self.local_bits, self.comm.world, comps)
            self.stats["swaps"] = self.stats.get("swaps", 0) + nsw
        if self.apply_fn is not _cuda_apply or sim.FUSE_TILE_BITS == 0:
            for g, shifts in comps:
                self.apply_gate(g, shifts, mode)
            return
        i = 0
        while i < len(comps):
            j = i
            while j < len(comps) and not self._needs_exchange(*comps[j]):
                j += 1
            if j > i:
                run = comps[i:j]
                prog = sim._GateProgram(run)
                L.call("diaq_run_gates_local", self.n_qubits, self.local_bits, self.comm.rank, prog.n, prog.arr,
                       self.local.data_ptr(), int(mode), int(sim.FUSE_TILE_BITS), None, None, L.stream_handle())
                self.stats["gates"] += len(run)
                self.stats["local"] += sum(all(s < self.local_bits for s in sh) for _, sh in run)
                self.stats["no_comm_global"] += sum(not all(s < self.local_bits for s in sh) for _, sh in run)
                i = j
                continue
            g, shifts = comps[i]
            self.apply_gate(g, shifts, mode)
            i += 1

    def norm(self) -> float:
        """||psi|| over all ranks (all-reduce of local |x|^2)."""
        if self.local.device.type == "cuda":
            from .sim import norm2
            local = norm2(self.local)
        else:
            local = float((self.local.abs() ** 2).sum().item())
        return float(np.sqrt(self.comm.allreduce_sum(local, self.local)))

    def gather(self):
        """Full state on rank 0 (tests only: 2^n amplitudes)."""
        return self.comm.gather(self.local)


class EmulatedComm:
    """P ranks driven by ONE process on one device (tests/benchmarks with fewer
    GPUs than ranks).  Ranks run one after another per gate; the exchange
    is a device copy of the partner's pre-gate shard, so nothing waits on
    another kernel (no cross-rank spin)."""

    def __init__(self, world: int):
        self.world = world
        self.rank = 0


def run_emulated(n_qubits: int, world: int, placements: list[Placement], cmul_mode: int | None = None,
                 device=None, remap: bool = False):
    """Apply placements to |0..0> split over `world` emulated ranks on one
    device; returns (list of local shards, stats).  Same plans and kernels as
    the multi-process path (remap: ShardedState.apply_placements)."""
    import torch

    from . import sim
    mode = sim.CMUL_MODE if cmul_mode is None else cmul_mode
    comms = []
    states = []
    for r in range(world):
        c = EmulatedComm(world)
        c.rank = r
        comms.append(c)
        states.append(ShardedState.basis(n_qubits, c, device=device))
    lb = states[0].local_bits
    stats = {"gates": 0, "local": 0, "no_comm_global": 0, "exchanged": 0}
    comps = [p.compact() for p in placements]
    if remap:
        comps, stats["swaps"] = remap_plan(n_qubits, lb, world, comps)
    fuse = sim.FUSE_TILE_BITS != 0

    def crosses(g, shifts):
        if all(s < lb for s in shifts):
            return False, None
        needs = exchange_schedule(n_qubits, lb, g, shifts, world)
        return any(src != r for r in range(world) for src in needs[r].values()), needs

    i = 0
    while i < len(comps):
        if fuse:
            j = i
            while j < len(comps) and not crosses(*comps[j])[0]:
                j += 1
            if j > i:
                prog = sim._GateProgram(comps[i:j])
                for r in range(world):
                    L.call("diaq_run_gates_local", n_qubits, lb, r, prog.n, prog.arr, states[r].local.data_ptr(),
                           int(mode), int(sim.FUSE_TILE_BITS), None, None, L.stream_handle())
                for g, shifts in comps[i:j]:
                    stats["gates"] += 1
                    stats["local" if all(s < lb for s in shifts) else "no_comm_global"] += 1
                i = j
                continue
        g, shifts = comps[i]
        stats["gates"] += 1
        cross, needs = crosses(g, shifts)
        if needs is None:
            stats["local"] += 1
            for r in range(world):
                _cuda_apply(n_qubits, lb, g, shifts, r, [states[r].local], states[r].local, mode)
            i += 1
            continue
        stats["exchanged" if cross else "no_comm_global"] += 1
        if cross:  # shard-equivalents each rank reads from partners (in-place peer reads)
            rd = sum(f for r in range(world) for b, f in partner_rows(lb, g, shifts, r).items()
                     if needs[r].get(b, r) != r) / world
            stats["partner_shards_read"] = round(stats.get("partner_shards_read", 0.0) + rd, 6)
        snap = {}
        if cross:  # partner data as it was before this gate
            for r in range(world):
                for src in needs[r].values():
                    if src != r and src not in snap:
                        snap[src] = states[src].local.clone()
        kg = len(global_shifts(shifts, lb))
        for r in range(world):
            srcs = [None] * (1 << kg)
            for b, src in needs[r].items():
                srcs[b] = states[r].local if src == r else snap[src]
            _cuda_apply(n_qubits, lb, g, shifts, r, srcs, states[r].local, mode)
        i += 1
    return [s.local for s in states], stats


class ShardedDiaq:
    """This rank's rows of a DiaQ matrix split like a sharded state: rank q
    owns rows [q*2^B, (q+1)*2^B), B = n_bits - p.  `rows[i]` holds diagonal
    offs[i] at those rows (row-indexed, so an offset crossing the shard
    boundary needs no index shuffle).  spmv reads x from every rank's slice
    -- its own and partners' through peer mappings (PeerComm.share) -- inside
    the kernel (diaq_spmv_sharded); bitwise the single-GPU spmv."""

    def __init__(self, n: int, offs, rows, row0: int, nrows: int):
        self.n = int(n)
        self.offs = np.ascontiguousarray(offs, dtype=np.int64)
        self.rows = list(rows)
        self.row0 = int(row0)
        self.nrows = int(nrows)

    @classmethod
    def from_matrix(cls, a, rank: int, world: int) -> "ShardedDiaq":
        """Row slice of a (device) DiaqMatrix for `rank` of `world` (tests and
        single-node setups; at scale each rank builds its slice directly)."""
        import torch
        n = a.n_dim
        if world & (world - 1) or n % world:
            raise ValueError(f"{world} ranks do not split n_dim={n} into power-of-two slices")
        nrows = n // world
        row0 = rank * nrows
        dev = a._device()
        rows = []
        for d, st in zip(dev.offs.tolist(), dev.starts.tolist()):
            t = torch.zeros(nrows, dtype=torch.complex128, device=dev.vals.device)
            lo, hi = max(0, -d, row0), min(n, n - d, row0 + nrows)
            if hi > lo:  # element of row r sits at k = r + min(d, 0)
                k0 = st + lo + min(d, 0)
                t[lo - row0:hi - row0] = dev.vals[k0:k0 + (hi - lo)]
            rows.append(t)
        return cls(n, dev.offs, rows, row0, nrows)

    @classmethod
    def from_block(cls, a, rank: int, world: int) -> "ShardedDiaq":
        """This rank's rows of kron(I_world, a) -- a matrix whose shards are
        diagonal blocks (e.g. kron_identity with the left identity spanning
        the shard bits): the rank builds only its own 2^B block `a`; global
        diagonal entries outside the block are the stored zeros of the
        Kronecker expansion, and their x reads still go to the partner (so
        the signs of zero match the single-GPU product)."""
        import torch
        nloc = a.n_dim
        dev = a._device()
        rows = []
        for d, st in zip(dev.offs.tolist(), dev.starts.tolist()):
            t = torch.zeros(nloc, dtype=torch.complex128, device=dev.vals.device)
            lo, hi = max(0, -d), min(nloc, nloc - d)
            if hi > lo:
                k0 = st + lo + min(d, 0)
                t[lo:hi] = dev.vals[k0:k0 + (hi - lo)]
            rows.append(t)
        return cls(nloc * world, dev.offs, rows, rank * nloc, nloc)

    def spmv(self, x_parts, y=None):
        """y (this rank's rows) = A x; x_parts[q]: rank q's x slice (tensor or address)."""
        nparts = len(x_parts)
        part_bits = (self.n // nparts).bit_length() - 1
        if y is None:
            y = L.empty_c128(self.nrows)
        rows = (ctypes.c_void_p * max(1, len(self.rows)))(*[t.data_ptr() for t in self.rows])
        parts = (ctypes.c_void_p * nparts)(*[_ptr(t) for t in x_parts])
        L.call("diaq_spmv_sharded", self.n, len(self.offs), self.offs.ctypes.data if len(self.offs) else None,
               rows, self.row0, self.nrows, parts, part_bits, nparts, y.data_ptr(), L.stream_handle())
        return y
