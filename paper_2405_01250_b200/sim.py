"""State-vector simulation on the device (drop-in for diaqsim.sim).

Reference: /root/reference/pkg/src/diaqsim/sim.py.  The diaq backend applies
every Placement on the B200:

* compact gates (everything compile_circuit emits, and explicit placements
  whose m is a small power-of-two block) go through the group kernel
  (apply.cu gate_kernel): read each amplitude once, write it once;
* any other explicit Placement goes through the diagonal kernel
  (apply.cu placed_kernel), the direct analogue of _apply_diags_block.

Both reproduce the reference's per-amplitude summation order and numpy's
complex multiply rounding (CMUL_MODE), so states match the reference
bitwise on hosts whose numpy uses the same complex multiply (see
DESIGN.md; the contract is 1e-12 relative L2).

run() compiles on the host, then hands the whole gate list to the native
loop diaq_run_gates (one C call, in-place updates, CUDA events around every
gate resolved after the loop -- no per-gate host sync).  Sampling is the
reference's splitmix64 inverse-CDF sampler, on the device with the
reference's sequential CDF reproduced exactly (sample.cu).
"""
from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .errors import NormalizationError, ResourceError, ShapeError
from .gates import Circuit, Placement, compile_circuit, fuse_pass
from .matrix import kron_identity, spmv, to_dense

MAX_QUBITS = 30

BACKENDS = ("dense", "diaq")


def _probe_numpy_cmul() -> int:
    """Which complex-multiply rounding this host's numpy uses."""
    rng = np.random.default_rng(7)
    a = rng.normal(size=64) + 1j * rng.normal(size=64)
    b = rng.normal(size=64) + 1j * rng.normal(size=64)
    plain = a.real * b.real - a.imag * b.imag
    return L.CMUL_PLAIN if np.array_equal((a * b).real, plain) else L.CMUL_FMA


# rounding of the gate-apply complex multiply; defaults to this host's numpy
CMUL_MODE = _probe_numpy_cmul()
_REFERENCE_CMUL = CMUL_MODE


def set_numerics(kind: str) -> None:
    """Arithmetic of the gate loop (extension; the default is "reference").

    "reference": every gate with numpy's complex-multiply rounding, states
    bitwise equal to the reference simulator.  "contracted": fused
    multiply-add chains (a rotation costs 4 FP64 operations per amplitude
    instead of 6; runs of diagonal gates on non-register bits fold into one
    factor), within 1e-12 relative L2 of the reference (the north-star
    tolerance) but not bitwise.
    """
    global CMUL_MODE
    if kind == "reference":
        CMUL_MODE = _REFERENCE_CMUL
    elif kind == "contracted":
        CMUL_MODE = L.CMUL_CONTRACT
    else:
        raise ValueError(f"numerics must be 'reference' or 'contracted', got {kind!r}")

# shared-memory tile of the fused multi-gate passes (diaq_run_gates_fused):
# 11 or 12 bits, -1 lets the library pick per circuit (12 only with >12%
# fewer HBM passes: its passes cost ~1.14x); 0 applies every gate as its own
# HBM sweep.  Results are identical.
FUSE_TILE_BITS = -1


class StateVector:
    """2^n complex128 amplitudes, resident on the device.

    `amps` is the host view (downloaded lazily, like the reference's numpy
    array); `device_amps` the CUDA tensor.  Construct from either.
    """

    def __init__(self, n_qubits: int, amps):
        self.n_qubits = int(n_qubits)
        self._set(amps)

    def _set(self, amps) -> None:
        t = L.torch()
        if isinstance(amps, t.Tensor) and amps.device.type == "cuda":
            self._dev = L.to_device_c128(amps.reshape(-1))
            self._host = None
        else:
            # the caller's array is copied: the state owns its amplitudes, and
            # the copy is the authoritative one until the first upload
            self._host = np.array(amps, dtype=np.complex128, copy=True).reshape(-1)
            self._dev = None

    @property
    def device_amps(self):
        if self._dev is None:
            self._dev = L.to_device_c128(self._host)
            # from now on the device copy is authoritative: the host copy is a
            # read-only snapshot (an edit could not reach the device)
            self._host.flags.writeable = False
        return self._dev

    def _device_modified(self) -> None:
        """The device amplitudes changed in place: drop the host snapshot."""
        self._host = None

    @property
    def amps(self) -> np.ndarray:
        """Host view of the amplitudes.  Writable only while the state has
        never been uploaded; afterwards a read-only snapshot of the device
        copy.  Assign `state.amps = array` to replace the amplitudes."""
        if self._host is None:
            self._host = self._dev.cpu().numpy()
            self._host.flags.writeable = False
        return self._host

    @amps.setter
    def amps(self, value) -> None:
        value = np.asarray(value)
        if value.size != len(self):
            raise ShapeError(f"state has {len(self)} amplitudes, got {value.size}")
        self._set(value)

    def __len__(self) -> int:
        return int(self._dev.numel()) if self._dev is not None else len(self._host)

    def norm(self) -> float:
        return float(np.sqrt(norm2(self.device_amps)))


def norm2(x) -> float:
    """sum |x_i|^2 of a device vector (deterministic two-pass reduction)."""
    t = L.torch()
    work = t.empty(L.DIAQ_NORM_WORK, dtype=t.float64, device=x.device)
    L.call("diaq_norm2", int(x.numel()), x.data_ptr(), work.data_ptr(), L.stream_handle())
    return float(work[0].item())


@dataclass
class RunResult:
    counts: dict[str, int]
    timings_ns: dict
    backend: str
    seed: int
    shots: int
    n_qubits: int
    state: np.ndarray | None = None


def init_state(n_qubits: int, max_qubits: int = MAX_QUBITS) -> StateVector:
    """|0...0>: amplitude 1 at index 0 (sim.py:53-59)."""
    if not 1 <= n_qubits <= max_qubits:
        raise ResourceError(f"n_qubits {n_qubits} outside 1..{max_qubits}")
    x = L.empty_c128(2**n_qubits)
    L.call("diaq_init_basis", 2**n_qubits, x.data_ptr(), 0, L.stream_handle())
    return StateVector(n_qubits, x)


def _check_dims(p: Placement, x: StateVector) -> None:
    if p.n_dim != len(x):
        raise ShapeError(
            f"placement covers {p.n_dim} amplitudes, state has {len(x)}"
        )


def _apply_into(p: Placement, xd, yd, cmul_mode: int) -> None:
    """y = placement(x) on the device; y must not alias x for the generic path."""
    n = int(xd.numel())
    comp = p.compact()
    s = L.stream_handle()
    if comp is not None:
        g, shifts = comp
        k = len(shifts)
        gd = np.ascontiguousarray(g, dtype=np.complex128)
        sh = np.ascontiguousarray(shifts, dtype=np.int32)
        L.call("diaq_apply_gate", n.bit_length() - 1, k, gd.ctypes.data, sh.ctypes.data,
               xd.data_ptr(), yd.data_ptr(), int(cmul_mode), s)
        return
    st = p.m._struct()
    L.call("diaq_apply_placed", p.dim_a, ctypes.byref(st), p.dim_b, xd.data_ptr(), yd.data_ptr(),
           int(cmul_mode), s)


def apply_placed(p: Placement, x: StateVector, threads: int = 1,
                 cmul_mode: int | None = None) -> StateVector:
    """Apply I_dim_a (x) m (x) I_dim_b to x on the device (sim.py:81-105).

    Returns a fresh state (x is not modified).  `threads` is accepted for API
    compatibility; results never depend on it (the reference guarantees the
    same, sim.py:84-87).
    """
    _check_dims(p, x)
    xd = x.device_amps
    yd = L.empty_c128(xd.numel())
    _apply_into(p, xd, yd, CMUL_MODE if cmul_mode is None else cmul_mode)
    return StateVector(x.n_qubits, yd)


def apply_dense(p: Placement, x: StateVector) -> StateVector:
    """Dense backend: materialise the span operator and contract it (sim.py:108-120).

    Reference/oracle backend only (4^span cost); runs as a torch contraction
    on the device.
    """
    _check_dims(p, x)
    t = L.torch()
    g = t.from_numpy(np.ascontiguousarray(to_dense(p.m))).to(L.device())
    x3 = x.device_amps.reshape(p.dim_a, p.m.n_dim, p.dim_b)
    y3 = t.tensordot(g, x3, dims=([1], [1])).permute(1, 0, 2).contiguous()
    return StateVector(x.n_qubits, y3.reshape(-1))


# -- sampling ------------------------------------------------------------------

# splitmix64: golden-gamma counter increment and the two mixing constants
_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_MIX1 = np.uint64(0xBF58476D1CE4E5B9)
_MIX2 = np.uint64(0x94D049BB133111EB)


def splitmix64_uniforms(seed: int, count: int) -> np.ndarray:
    """`count` doubles in [0, 1) from the splitmix64 stream for `seed` (sim.py:131-139)."""
    idx = np.arange(1, count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + idx * _GAMMA
        z = (z ^ (z >> np.uint64(30))) * _MIX1
        z = (z ^ (z >> np.uint64(27))) * _MIX2
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * 2.0**-53


def measure_all_sample(x: StateVector, shots: int, seed: int) -> dict[str, int]:
    """Sample `shots` bitstrings (q0..q(n-1), MSB first) from |amps|^2 (sim.py:142-161).

    On the device (sample.cu): probabilities rounded to 1e-12 and the
    SEQUENTIAL float64 CDF of the reference are reproduced bit for bit, so
    counts equal the reference's for the same state and seed.
    """
    if shots < 0:
        raise ValueError(f"shots must be >= 0, got {shots}")
    xd = x.device_amps
    u = splitmix64_uniforms(seed, shots)
    hits = np.empty(max(shots, 1), dtype=np.int64)
    norm2 = ctypes.c_double(0.0)
    L.call("diaq_sample_hits", int(xd.numel()), xd.data_ptr(), u.ctypes.data if shots else None, int(shots),
           hits.ctypes.data if shots else None, ctypes.addressof(norm2), L.stream_handle())
    if abs(norm2.value - 1.0) > 1e-6:
        raise NormalizationError(f"state norm^2 = {norm2.value:.9f}, cannot sample")
    if shots == 0:
        return {}
    outcomes, freq = np.unique(hits[:shots], return_counts=True)
    width = x.n_qubits
    # bitstrings q0..q(n-1), MSB first, formatted in one numpy pass
    bits = (outcomes[:, None] >> np.arange(width - 1, -1, -1, dtype=np.int64)) & 1
    keys = (bits.astype(np.uint8) + ord("0")).view(f"S{width}").ravel()
    return {k.decode(): int(c) for k, c in zip(keys, freq.tolist())}


# -- driver ----------------------------------------------------------------------


_GATE_DTYPE = np.dtype({"names": ["k", "shifts", "g"], "formats": ["<i4", ("<i4", 5), "<u8"],
                        "offsets": [0, 4, 24], "itemsize": 32})  # diaq_gate_t


class _GateProgram:
    """Compact gates packed for diaq_run_gates (keeps host buffers alive).
    Packed with numpy into the diaq_gate_t layout; the last program is
    cached per run of Placement objects (held, so their ids stay theirs)."""

    _last: tuple | None = None

    def __init__(self, comps):
        n = len(comps)
        self.buf = np.zeros(max(1, n), dtype=_GATE_DTYPE)
        if n:
            # every gate matrix in one contiguous host block; g = base + offset
            mats, ks, flat_sh = [], [], []
            for g, sh in comps:
                mats.append(g.reshape(-1))
                ks.append(len(sh))
                flat_sh.extend(sh)
            self.mats = np.concatenate(mats).astype(np.complex128, copy=False)
            k = np.asarray(ks, dtype=np.int64)
            sizes = np.left_shift(1, 2 * k)
            offs = np.zeros(n, dtype=np.int64)
            np.cumsum(sizes[:-1], out=offs[1:])
            sh = np.zeros((n, 5), dtype=np.int32)
            rows = np.repeat(np.arange(n), k)
            cols = np.arange(len(flat_sh)) - np.repeat(np.cumsum(k) - k, k)
            sh[rows, cols] = flat_sh
            self.buf["k"][:n] = k
            self.buf["shifts"][:n] = sh
            self.buf["g"][:n] = self.mats.ctypes.data + 16 * offs
        self.arr = self.buf.ctypes.data_as(ctypes.POINTER(L.Gate))
        self.n = n

    @classmethod
    def for_placements(cls, pls):
        # keyed by each placement's identity AND the state its compact form
        # depends on (dims, gate, matrix edit version): reassigning p.m or
        # editing m with set_diag rebuilds the program
        key = tuple((id(p), p._token()) for p in pls)
        last = cls._last
        if last is not None and last[0] == key:
            return last[2]
        prog = cls([p.compact() for p in pls])
        cls._last = (key, list(pls), prog)
        return prog


def run_gates(state: StateVector, placements: list[Placement], cmul_mode: int | None = None,
              timer: "L.Timer | None" = None, inplace: bool = False,
              tile_bits: int | None = None) -> StateVector:
    """Apply placements in order on the device; each maximal run of compact
    gates goes through one native call (diaq_run_gates, in place).  The input
    state is left untouched unless inplace=True.  `timer` (len(placements)+1
    events) records the boundaries of every gate."""
    mode = CMUL_MODE if cmul_mode is None else cmul_mode
    n_bits = len(state).bit_length() - 1
    xd = state.device_amps
    if inplace:
        state._device_modified()
    else:
        xd = xd.clone()
    i = 0
    s = L.stream_handle()
    while i < len(placements):
        j = i
        while j < len(placements) and placements[j].compact() is not None:
            j += 1
        if j > i:
            prog = _GateProgram.for_placements(placements[i:j])
            evs = timer.slice_ptr(i) if timer is not None else None
            tb = FUSE_TILE_BITS if tile_bits is None else tile_bits
            if tb != 0:
                L.call("diaq_run_gates_fused", n_bits, prog.n, prog.arr, xd.data_ptr(), int(mode), int(tb), evs,
                       None, s)
            else:
                L.call("diaq_run_gates", n_bits, prog.n, prog.arr, xd.data_ptr(), int(mode), evs, s)
            i = j
            continue
        p = placements[i]
        yd = L.empty_c128(xd.numel())
        if timer is not None:
            timer.record(i)
        _apply_into(p, xd, yd, mode)
        xd = yd
        if timer is not None:
            timer.record(i + 1)
        i += 1
    return StateVector(state.n_qubits, xd)


_RUN_CACHE: dict = {}


def run(
    circuit: Circuit,
    backend: str = "diaq",
    shots: int = 1024,
    seed: int = 0,
    fusion: bool = False,
    span_limit: int | None = None,
    emit_state: bool = False,
    threads: int = 1,
) -> RunResult:
    """Compile, apply, and sample a circuit (sim.py:167-221).

    Timings are nanoseconds per phase; per-gate application times come from
    CUDA events recorded around every gate and resolved after the loop.
    """
    if backend not in BACKENDS:
        raise ValueError(f"backend must be one of {BACKENDS}, got '{backend}'")
    kwargs = {} if span_limit is None else {"span_limit": span_limit}
    t0 = time.perf_counter_ns()
    # run() never hands its placements out, so a repeated run of the same
    # circuit (same ops, span limit, fusion) reuses the compiled list -- and
    # with it the packed native program and the per-gate timer
    key = (circuit.n_qubits, kwargs.get("span_limit"), bool(fusion), tuple(circuit.ops))
    hit = _RUN_CACHE.get(key)
    if hit is None:
        placements = fuse_pass(compile_circuit(circuit, **kwargs), enabled=fusion)
        names = [f"{i}:{p.name}" for i, p in enumerate(placements)]
        comps = [p.compact() for p in placements]
        # the placements are private to this cache, so the packed program
        # cannot go stale: it is built once and replayed
        prog = _GateProgram(comps) if all(c is not None for c in comps) else None
        hit = (placements, names, L.Timer(len(placements) + 1), prog)
        if len(_RUN_CACHE) >= 4:
            _RUN_CACHE.pop(next(iter(_RUN_CACHE)))
        _RUN_CACHE[key] = hit
    placements, names, timer, prog = hit
    t_compile = time.perf_counter_ns() - t0

    state = init_state(circuit.n_qubits)
    t0 = time.perf_counter_ns()
    if backend == "diaq" and prog is not None and prog.n:
        xd = state.device_amps
        state._device_modified()
        n_bits = len(state).bit_length() - 1
        if FUSE_TILE_BITS != 0:
            L.call("diaq_run_gates_fused", n_bits, prog.n, prog.arr, xd.data_ptr(), int(CMUL_MODE),
                   int(FUSE_TILE_BITS), timer.slice_ptr(0), None, L.stream_handle())
        else:
            L.call("diaq_run_gates", n_bits, prog.n, prog.arr, xd.data_ptr(), int(CMUL_MODE), timer.slice_ptr(0),
                   L.stream_handle())
    elif backend == "diaq":
        state = run_gates(state, placements, timer=timer, inplace=True)
    else:
        timer.record(0)
        for i, p in enumerate(placements):
            state = apply_dense(p, state)
            timer.record(i + 1)
    ms = timer.elapsed_ms()  # one host sync after the whole loop
    t_apply = time.perf_counter_ns() - t0
    per_gate = dict(zip(names, np.rint(ms.astype(np.float64) * 1e6).astype(np.int64).tolist()))

    t0 = time.perf_counter_ns()
    counts = measure_all_sample(state, shots, seed)
    t_sample = time.perf_counter_ns() - t0

    timings = {
        "compile": t_compile,
        "apply_total": t_apply,
        "sample": t_sample,
        "total": t_compile + t_apply + t_sample,
        "per_gate": per_gate,
    }
    return RunResult(
        counts=counts,
        timings_ns=timings,
        backend=backend,
        seed=seed,
        shots=shots,
        n_qubits=circuit.n_qubits,
        state=state.amps if emit_state else None,
    )
