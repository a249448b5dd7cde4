#!/usr/bin/env python3
"""Benchmark of the B200 DiaQ hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[3], the metric's config): the config-4 DiaQ
matrix at n=28 -- kron_identity(2^6, build_span_unitary(Haar4, [18, 0], 19),
2^3), 9 diagonals at offsets {0, +-8, +-2^21, +-(2^21 +- 8)}, 38.45 GB of
complex128 diagonals, built on the device -- times a normalised random x.
One step = one spmv.  value = algorithmic bytes (16*sum(N-|d|) + 32*N =
47,043,313,408 B per step per GPU) / device time, summed over ranks (each
rank runs its own replica: the spmv does not shard, so N>1 is weak-scaling
replicas; the sharded circuit path is measured separately).  Inputs are far
larger than the 126 MB L2, so no flush is needed between steps.

Also reported on the same line: gate applications/s at n=28 (the metric's
second half: one random layer of RX/RY/RZ + CX matching per step through the
native run loop), e2e through the public API with pinned host buffers,
the roofline of the dominant kernel, the CPU baseline (the pinned C oracle,
OpenMP over all host cores, on an n=24 sample with the same offsets), SM
clocks sampled during the timed region, and our kernel-launch count.

--impl reference times the reference algorithm's CPU implementation (the
oracle port, oracle/) on the same metric; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "DiaQ spmv HBM GB/s and gate-applications/sec at n=28 c128; % of HBM roofline"
N_QUBITS = 28


def alg_bytes(n_dim: int, offsets) -> int:
    return 16 * sum(n_dim - abs(int(d)) for d in offsets) + 32 * n_dim


def measured_peak() -> tuple[float, str]:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def profiled_traffic() -> dict:
    """dram bytes per launch from the committed ncu summary, if any."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return {}


class ClockSampler:
    """SM clock and throttle reasons sampled every 10 ms (NVML) during the timed region."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index: int, period_s: float = 0.01):
        self.index = index
        self.period = period_s
        self.sm: list[float] = []
        self.reasons: set[str] = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self.error = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM))
            self.thread = threading.Thread(target=self._run, daemon=True)
            self.thread.start()
        except Exception as e:  # no NVML: report without clocks
            self.error = repr(e)
            self._nv = None
        return self

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)))
                mask = int(nv.nvmlDeviceGetCurrentClocksEventReasons(self._h))
                for name, bit in self.REASONS.items():
                    if mask & bit:
                        self.reasons.add(name)
            except Exception as e:
                self.error = repr(e)
                return
            time.sleep(self.period)

    def __exit__(self, *exc):
        self._stop.set()
        if self._nv is not None:
            self.thread.join(timeout=2)

    def summary(self) -> dict:
        out = {"sm_mhz": statistics.median(self.sm) if self.sm else None, "sm_max_mhz": self.max_mhz,
               "reasons": sorted(self.reasons), "samples": len(self.sm), "source": "nvml 10 ms"}
        if self.error:
            out["error"] = self.error
        return out


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("DIAQ_BENCH_SAME_GPU"):  # functional check of the N>1 code on one GPU (not a measurement)
        local = 0
    return rank, world, local


def init_dist(world: int, backend: str):
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend=backend)
        return dist
    return None


def max_over_ranks(dist, value: float, device) -> float:
    if dist is None:
        return value
    import torch
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------- CPU baseline
#
# The reference's algorithm on the box's host cores.  The reference itself is
# numpy (single-threaded ufuncs, ~1 GB/s); the pinned C oracle
# (oracle/, bitwise the reference spmv) with OpenMP over every host core is
# a stronger CPU baseline and is what the reference arm reports, at the
# metric's own config (n=28).  Threads are pinned (OMP_PROC_BIND=close,
# OMP_PLACES=cores, set before the oracle library loads) and every figure is
# the median of >= 5 timed reps after a warm-up.

CPU_SPMV_REPS = 5


def _cpu_env() -> None:
    os.environ.setdefault("OMP_PROC_BIND", "close")
    os.environ.setdefault("OMP_PLACES", "cores")


def _fast_state(n_amps: int, seed: int = 1) -> np.ndarray:
    """Normalised Gaussian complex vector (timing input; numpy's own sum)."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(2 * n_amps).view(np.complex128)
    x /= np.linalg.norm(x)
    return x


def cpu_spmv_measure(n: int, reps: int = CPU_SPMV_REPS, warmup: int = 1) -> dict:
    """The C oracle spmv on the config-4 matrix at n (OpenMP, all cores)."""
    _cpu_env()
    from oracle import oracle as O
    from paper_2405_01250_b200 import workloads as W
    c4 = W.config4(22, seed=0, with_x=False)  # the gate and offsets are those of every n >= 22
    t0 = time.perf_counter()
    span = O.span_unitary(c4["u4"], c4["positions"], c4["span"])
    a = O.kron_identity(2 ** (n - 22), span, c4["right"])
    x = _fast_state(2**n)
    build_s = time.perf_counter() - t0
    nb = alg_bytes(2**n, a.offs)
    for _ in range(warmup):
        O.spmv(a, x)
    times = []
    for _ in range(reps):
        t1 = time.perf_counter()
        O.spmv(a, x)
        times.append(time.perf_counter() - t1)
    med = statistics.median(times)
    del a, x
    return {"value": round(nb / med / 1e9, 3), "unit": "GB/s", "cores": O.num_threads(), "kind": "port",
            "sample": f"config-4 spmv at n={n} (the metric's config), median of {reps} after {warmup} warm-up; "
                      f"C oracle -O3 OpenMP (bitwise reference matrix.py:253-278), "
                      f"OMP_PROC_BIND={os.environ.get('OMP_PROC_BIND')} OMP_PLACES={os.environ.get('OMP_PLACES')}",
            "times_s": [round(t, 4) for t in times], "build_s": round(build_s, 2), "alg_bytes_per_step": nb,
            "cpu_model": _cpu_model()}


def cpu_gates_measure(n: int = N_QUBITS, count: int = 4) -> dict:
    """The oracle's apply_placed (reference sim.py:81-105, numpy complex
    multiply rounding) on the first `count` one-qubit gates of the n=28 random
    layer, at 1 thread and at every host core: gates/s."""
    _cpu_env()
    from oracle import oracle as O
    from paper_2405_01250_b200 import workloads as W
    ops = [o for o in W.random_layered_ops(n, 1, seed=0) if len(o[1]) == 1][:count]
    x = _fast_state(2**n, seed=2)
    out = {}
    for threads in (1, O.num_threads()):
        t_total = 0.0
        for name, (q,), params in ops:
            g = O.GATES[name](*params)
            m = O.from_dense(g)
            t1 = time.perf_counter()
            x = O.apply_placed(2**q, m, 2 ** (n - 1 - q), x, O.numpy_cmul_mode(), threads)
            t_total += time.perf_counter() - t1
        out[f"threads_{threads}"] = {"gates_per_s": round(len(ops) / t_total, 3), "s_per_gate": round(t_total / len(ops), 3)}
    return {"unit": "gates/s", "kind": "port", "n_qubits": n, "gates": [o[0] for o in ops], **out,
            "sample": f"first {len(ops)} one-qubit gates of the n={n} random layer, C oracle apply_placed "
                      "(reference sim.py:69-105), pinned OpenMP threads"}


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def numpy_reference_secondary() -> dict:
    """The real reference (numpy, baseline/_ref installed by
    tools/install_reference.py) on this host: its spmv on the config-4
    parity slice (n=22) and run() at n=20 (2 random layers) at threads=1 and
    at every core.  Bounded samples; absent install -> reported as such."""
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "diaqsim")):
        return {"unavailable": "baseline/_ref not installed (python tools/install_reference.py)"}
    import importlib
    if ref_dir not in sys.path:
        sys.path.insert(0, ref_dir)
    R = importlib.import_module("diaqsim")
    from paper_2405_01250_b200 import workloads as W
    out = {"kind": "reference (numpy, unmodified)", "cpu_model": _cpu_model(), "numpy": np.__version__}
    c4 = W.config4(22, seed=0, with_x=False)
    a = R.kron_identity(1, R.build_span_unitary(R.from_dense(c4["u4"]), c4["positions"], c4["span"]), c4["right"])
    x = _fast_state(2**22)
    nb = alg_bytes(2**22, a.diag_indices())
    R.spmv(a, x)
    ts = []
    for _ in range(3):
        t1 = time.perf_counter()
        R.spmv(a, x)
        ts.append(time.perf_counter() - t1)
    out["spmv_n22"] = {"GBs": round(nb / statistics.median(ts) / 1e9, 3), "s": round(statistics.median(ts), 3),
                       "cores": 1, "note": "numpy ufuncs, single-threaded; median of 3"}
    del a, x
    ops = W.random_layered_ops(20, 2, seed=0)
    circ = R.Circuit(20, [R.GateOp(*o) for o in ops])
    for threads in (1, os.cpu_count() or 1):
        t1 = time.perf_counter()
        res = R.run(circ, shots=0, span_limit=20, threads=threads)
        dt = time.perf_counter() - t1
        out[f"run_n20_threads_{threads}"] = {"gates": len(ops), "s": round(dt, 3),
                                             "apply_gates_per_s": round(len(ops) / (res.timings_ns["apply_total"] * 1e-9), 2)}
    return out


def run_reference(args):
    """--impl reference: the reference algorithm's CPU implementation at the
    metric's config (config-4 spmv, n=28) on all host cores; rank 0 only."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    n = args.n
    _cpu_env()
    from oracle import oracle as O
    from paper_2405_01250_b200 import workloads as W
    c4 = W.config4(22, seed=0, with_x=False)
    span = O.span_unitary(c4["u4"], c4["positions"], c4["span"])
    a = O.kron_identity(2 ** (n - 22), span, c4["right"])
    x = _fast_state(2**n)
    nb = alg_bytes(2**n, a.offs)
    for _ in range(args.warmup):
        O.spmv(a, x)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        O.spmv(a, x)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    value = nb * len(times) / total / 1e9
    del a, x
    secondary = {}
    if not args.no_secondary:
        try:
            secondary["numpy_reference"] = numpy_reference_secondary()
        except Exception as e:  # never lose the arm's line
            secondary["numpy_reference"] = {"error": repr(e)}
    line = {
        "metric": METRIC, "impl": "reference", "value": round(value, 3), "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * total / len(times), 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"config4 spmv n={n}: kron_identity(2^{n - 22}, span(Haar4,[18,0],19), 2^3)",
                   "n_qubits": n, "alg_bytes_per_step": nb, "same_config_as_ours": True},
        "cpu_baseline": {"value": round(value, 3), "unit": "GB/s", "cores": O.num_threads(), "kind": "port",
                         "sample": f"every step = one config-4 spmv at n={n}; the C oracle restating reference "
                                   "matrix.py:253-278 bitwise, OpenMP pinned (OMP_PROC_BIND=close, OMP_PLACES=cores)",
                         "step_s_median": round(statistics.median(times), 4), "cpu_model": _cpu_model()},
        "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "secondary": secondary,
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- GPU arm

def run_ours(args):
    import torch

    import paper_2405_01250_b200 as D
    from paper_2405_01250_b200 import _lib as L
    from paper_2405_01250_b200 import workloads as W

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = init_dist(world, os.environ.get("DIAQ_BENCH_DIST_BACKEND", "nccl"))
    lib = L.load()
    n = args.n
    N = 2**n

    # ---- build the config-4 matrix on the device
    c4 = W.config4(22, seed=0, with_x=False)  # the gate and offsets (identical for every n >= 22)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    span = D.build_span_unitary(D.from_dense(c4["u4"], 0.0), c4["positions"], c4["span"])
    a = D.kron_identity(2 ** (n - 22), span, c4["right"])
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t0
    offs = a.diag_indices()
    nbytes = alg_bytes(N, offs)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    x = torch.randn(N, dtype=torch.complex128, device=dev, generator=gen)
    x /= torch.linalg.vector_norm(x)
    y = torch.empty_like(x)
    st = a._struct()
    s = torch.cuda.current_stream()

    def spmv_launch():
        L.call("diaq_spmv", __import__("ctypes").byref(st), x.data_ptr(), y.data_ptr(), s.cuda_stream)

    # N>1: the 2^(n+p) product kron(I, A) with its rows sharded over the ranks
    # (each rank builds only its own block); x stays in place on its rank and
    # the offsets that cross a shard boundary read the partner's x through a
    # peer mapping inside the kernel.  Falls back to replicas (no data-path
    # communication) when the GPUs cannot map each other.
    spmv_mode = "replicas" if world > 1 else "single GPU"
    if world > 1 and not args.replicas:
        try:
            from paper_2405_01250_b200.shard import PeerComm, ShardedDiaq
            pcomm = PeerComm()
            sd = ShardedDiaq.from_block(a, rank, world)
            xs, xptr = L.shared_c128(N)
            xs.copy_(x)
            parts = [row[0] for row in pcomm.share([xptr])]
            pcomm.barrier()

            def spmv_launch():  # noqa: F811 -- the sharded product replaces the replica
                sd.spmv(parts, y)
            spmv_mode = f"rows of a 2^{n + world.bit_length() - 1} product sharded over {world} ranks, x via peer loads"
        except L.DeviceError as e:
            spmv_mode = f"replicas (peer mapping failed: {e})"

    for _ in range(args.warmup):
        spmv_launch()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    launches0 = L.launch_count()
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        ev[0].record(s)
        for i in range(args.steps):
            spmv_launch()
            ev[i + 1].record(s)
        torch.cuda.synchronize()
    launches = L.launch_count() - launches0
    if dist is not None:
        dist.barrier()
    step_ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(args.steps)]
    total_ms = ev[0].elapsed_time(ev[-1])
    total_ms = max_over_ranks(dist, total_ms, dev)
    ms_per_step = total_ms / args.steps
    value = nbytes * world * args.steps / (total_ms * 1e-3) / 1e9
    y_norm = float(torch.linalg.vector_norm(y).item())

    # ---- gate applications.  N=1: one random layer at n=28 per step (the
    # metric's config).  N>1 (default): config 5 -- the 20-layer random
    # circuit on a 2^(30+p) state sharded over the ranks (weak scaling);
    # --replicas: independent n=28 layers per rank instead
    if world > 1 and not args.replicas:
        gates_part = sharded_gates(args, D, L, W, torch, dist, n, world, x, s, dev)
    else:
        gates_part = replica_gates(args, D, L, W, torch, dist, n, world, x, s, dev)
    n_gates, g_ms, g_launches, g_norm, gate_n, gate_extra = gates_part
    ms_per_gate = g_ms / n_gates
    ms_per_pass = g_ms / max(1, g_launches)
    gate_bytes = 32 * N  # per GPU per gate (each rank's 2^n amplitudes read + written)

    # ---- e2e through the public API with pinned host buffers
    # (failures are caught per rank, then every rank joins the same collective)
    e2e = None
    if not args.no_e2e:
        e_local, e_err = float("inf"), None
        try:
            xh = torch.empty(N, dtype=torch.complex128, pin_memory=True)
            xh.copy_(x)
            yh = torch.empty(N, dtype=torch.complex128, pin_memory=True)
            torch.cuda.synchronize()
            e_steps = max(1, min(args.steps, 5))
            D.spmv(a, xh, out=yh)  # warm-up (allocator)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(e_steps):
                D.spmv(a, xh, out=yh)
            torch.cuda.synchronize()
            e_local = (time.perf_counter() - t0) / e_steps
            del xh, yh
        except Exception as ex:  # pinned-memory limits etc.: report, do not hang the other ranks
            e_err = repr(ex)
        e_s = max_over_ranks(dist, e_local, dev)
        if e_s == float("inf"):
            e2e = {"error": e_err or "e2e failed on another rank"}
        else:
            e2e = {"value": round(nbytes * world / e_s / 1e9, 3), "unit": "GB/s",
                   "h2d_bytes_per_step": 16 * N, "d2h_bytes_per_step": 16 * N,
                   "ms_per_step": round(1e3 * e_s, 3),
                   "path": "paper_2405_01250_b200.spmv(a, pinned host x, out=pinned host y)"}

    secondary = {}
    if not args.no_secondary:
        try:
            secondary = secondary_workloads(args, D, L, W, torch)
        except Exception as e:  # never lose the headline line
            secondary = {"error": repr(e)}

    peak, peak_src = measured_peak()
    prof = profiled_traffic()
    kern_ms = statistics.mean(step_ms)
    achieved = nbytes / (kern_ms * 1e-3) / 1e9
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "peak_source": peak_src,
                "traffic": prof.get("spmv_dram_bytes_per_launch") if n == N_QUBITS else None,
                "alg_bytes_per_launch": nbytes, "kernel": "diaq::spmv_async_kernel<9> (cp.async-staged banded spmv)",
                "frac_of_8TBs_spec": round(achieved / 8000.0, 4)}
    gates_scale = 1 if (world > 1 and not args.replicas) else world
    gates = {"gates_per_s": round(gates_scale * n_gates / (g_ms * 1e-3), 2), "ms_per_gate": round(ms_per_gate, 4),
             "n_qubits": gate_n, **gate_extra,
             "roofline": {"bound": "hbm", "achieved": round(gate_bytes / (ms_per_pass * 1e-3) / 1e9, 1),
                          "peak": peak, "unit": "GB/s",
                          "frac": round(gate_bytes / (ms_per_pass * 1e-3) / 1e9 / peak, 4),
                          "traffic": prof.get("gate_dram_bytes_per_launch") if n == N_QUBITS else None,
                          "alg_bytes_per_launch": gate_bytes,
                          "per": "HBM pass (one kernel launch = one read+write sweep of the state; "
                                 "a fused pass applies several gates)",
                          "ms_per_pass": round(ms_per_pass, 4)},
             "norm_after": g_norm, "gpu_launches": int(g_launches)}
    gates["roofline_fp64"] = fp64_roofline(prof.get("gate_fp64_warp_inst_per_launch"), ms_per_pass)
    if isinstance(gates.get("contracted"), dict) and n == N_QUBITS:
        gates["contracted"]["roofline_fp64"] = fp64_roofline(
            prof.get("gate_contracted_fp64_warp_inst_per_launch"), gates["contracted"]["ms_per_pass"])
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return 0
    cpu = None
    if world == 1 and not args.no_cpu:
        try:
            cpu = cpu_spmv_measure(n)
            gates["cpu_baseline"] = cpu_gates_measure(gate_n)
        except Exception as e:  # never lose the headline line
            cpu = {"error": repr(e)}
        if not args.no_secondary:
            try:
                secondary["numpy_reference"] = numpy_reference_secondary()
            except Exception as e:
                secondary["numpy_reference"] = {"error": repr(e)}
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: seeded Haar-random 2-qubit gate (config 4), normalised Gaussian x",
        "config": {"workload": f"config4 spmv n={n}: kron_identity(2^{n - 22}, span(Haar4,[18,0],19), 2^3)",
                   "n_qubits": n, "N": N, "offsets": offs, "alg_bytes_per_step": nbytes,
                   "matrix_bytes": 16 * sum(N - abs(d) for d in offs),
                   "l2": "inputs (47 GB/step) far larger than the 126 MB L2; no flush needed",
                   "parallelism": spmv_mode, "build_s": round(t_build, 3)},
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "gates": gates,
        "secondary": secondary,
        "check": {"y_norm": y_norm, "unitary_norm_err": abs(y_norm - 1.0)},
        "step_ms_minmax": [round(min(step_ms), 4), round(max(step_ms), 4)],
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def fp64_roofline(warp_inst, ms_per_pass) -> dict | None:
    """FP64-pipe roofline of a gate pass: DMUL+DADD+DFMA warp instructions
    per launch (committed ncu opcode mix) over the measured pass time,
    against 148 SMs x 2 FP64 warp instructions per clock at the max SM clock."""
    if not warp_inst:
        return None
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mhz = float(json.load(f).get("sm_max_mhz", 1965.0))
    except Exception:
        mhz = 1965.0
    peak = 148 * 2 * mhz * 1e6  # warp instructions / s
    achieved = warp_inst / (ms_per_pass * 1e-3)
    return {"bound": "fp64", "achieved": round(achieved * 32 / 1e12, 3), "peak": round(peak * 32 / 1e12, 3),
            "unit": "T FP64 instr/s (DFMA = 1)", "frac": round(achieved / peak, 4),
            "fp64_warp_inst_per_launch": int(warp_inst), "source": "profiles/ncu_summary.json (ncu opcode mix)"}


def jit_stats(L):
    import ctypes
    st = (ctypes.c_int64 * 6)()
    L.call("diaq_jit_stats", ctypes.addressof(st))
    return dict(zip(["compiled", "failed", "launches", "modules", "pending", "compile_ms"], list(st)))


def replica_gates(args, D, L, W, torch, dist, n, world, x, s, dev):
    """Each rank applies one random layer per step to its own 2^n state (fused
    shared-memory passes; bitwise equal to gate-by-gate)."""
    gl_ops = W.random_layered_ops(n, 1, seed=0)
    pls = D.compile_circuit(D.Circuit(n, [D.GateOp(*o) for o in gl_ops]), span_limit=n)
    state = D.StateVector(n, x.clone())
    for _ in range(max(1, args.warmup // 2)):
        state = D.run_gates(state, pls, inplace=True)
    # the passes' specialised kernels compile in the background during the
    # warm-up (one-time, per pass structure); time the steady state
    t_jit = time.perf_counter()
    L.call("diaq_jit_wait", -1.0)
    jit_wait_s = time.perf_counter() - t_jit
    state = D.run_gates(state, pls, inplace=True)
    torch.cuda.synchronize()
    jst0 = jit_stats(L)
    g_steps = max(2, min(args.steps, 10))
    ge0 = torch.cuda.Event(enable_timing=True)
    ge1 = torch.cuda.Event(enable_timing=True)
    gl0 = L.launch_count()
    ge0.record(s)
    for _ in range(g_steps):
        state = D.run_gates(state, pls, inplace=True)
    ge1.record(s)
    torch.cuda.synchronize()
    g_launches = L.launch_count() - gl0
    jst1 = jit_stats(L)
    g_ms = max_over_ranks(dist, ge0.elapsed_time(ge1), dev)
    g_norm = state.norm()
    contracted = contracted_gates(D, L, torch, dist, pls, x, g_steps, s, dev)
    extra = {"gates_per_step": len(pls), "steps": g_steps, "mode": f"replicas x{world}",
             "numerics": "reference (numpy complex-multiply rounding; bitwise the reference)",
             "contracted": contracted,
             "fused_tile_bits": D.sim.FUSE_TILE_BITS if D.sim.FUSE_TILE_BITS > 0 else "auto (11 or 12: 12 only with >12% fewer passes)", "hbm_passes": int(g_launches),
             "specialised_passes": {"launches_timed": jst1["launches"] - jst0["launches"], "compiled": jst1["compiled"],
                                    "failed": jst1["failed"], "compile_cpu_ms": jst1["compile_ms"],
                                    "wait_after_warmup_s": round(jit_wait_s, 3),
                                    "note": "NVRTC per pass structure, background thread; one-time"}}
    return len(pls) * g_steps, g_ms, g_launches, g_norm, n, extra


def contracted_gates(D, L, torch, dist, pls, x, g_steps, s, dev):
    """The same layer under the contracted arithmetic (DIAQ_CMUL_CONTRACT:
    FMA chains, folded diagonal runs; within 1e-12 rel L2 of the reference,
    not bitwise): device time per step, and its parity on one layer from x
    against the reference-rounded layer."""
    C = L.CMUL_CONTRACT
    ref1 = D.run_gates(D.StateVector(x.numel().bit_length() - 1, x), pls).device_amps
    st = D.StateVector(x.numel().bit_length() - 1, x.clone())
    st = D.run_gates(st, pls, cmul_mode=C, inplace=True)
    d = st.device_amps
    rel = float(torch.linalg.vector_norm(d - ref1).item() / torch.linalg.vector_norm(ref1).item())
    del ref1
    L.call("diaq_jit_wait", -1.0)
    st = D.run_gates(st, pls, cmul_mode=C, inplace=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = L.launch_count()
    e0.record(s)
    for _ in range(g_steps):
        st = D.run_gates(st, pls, cmul_mode=C, inplace=True)
    e1.record(s)
    torch.cuda.synchronize()
    launches = L.launch_count() - l0
    ms = max_over_ranks(dist, e0.elapsed_time(e1), dev)
    peak, _ = measured_peak()
    ms_pass = ms / max(1, launches)
    gbs = 32 * x.numel() / (ms_pass * 1e-3) / 1e9
    return {"numerics": "contracted (FMA chains, folded diagonal runs; 1e-12 rel L2 tolerance, not bitwise)",
            "gates_per_s": round(len(pls) * g_steps / (ms * 1e-3), 2), "ms_per_pass": round(ms_pass, 4),
            "hbm_passes": int(launches), "roofline_frac": round(gbs / peak, 4), "achieved_GBs": round(gbs, 1),
            "rel_l2_vs_reference_one_layer": rel, "norm_err": abs(1.0 - st.norm())}


def sharded_gates(args, D, L, W, torch, dist, n, world, x, s, dev):
    """Config 5: the 20-layer random circuit (config-3 gate mix, CX matching
    over ALL qubits) on a 2^(L+p) state sharded over the ranks, L =
    --circuit-qubits local bits (30: 16 GiB per GPU); weak scaling.  One
    step = the whole circuit from the current state.  Cross-shard gates read
    partner shards in place over peer memory (--transport peer: CUDA IPC over
    NVLink/NVSwitch, ordered by IPC events) or exchange them with NCCL
    send/recv first (--transport nccl).  Measured without and with qubit
    remapping (half-shard swaps before cross-shard gates); the headline is
    the plain run."""
    from paper_2405_01250_b200.shard import PeerComm, ShardedState, TorchDistComm
    p = world.bit_length() - 1
    ns = args.circuit_qubits + p
    lb = args.circuit_qubits
    layers = args.circuit_layers
    del x  # the circuit starts from |0...0>
    transport = args.transport
    comm = PeerComm() if transport == "peer" else TorchDistComm()
    try:
        st = ShardedState.basis(ns, comm)
    except L.DeviceError as e:  # no peer mapping between these GPUs: staged NCCL exchange
        transport = f"nccl (peer mapping failed: {e})"
        comm = TorchDistComm()
        st = ShardedState.basis(ns, comm)
    ops = W.random_layered_ops(ns, layers, seed=0)
    pls = D.compile_circuit(D.Circuit(ns, [D.GateOp(*o) for o in ops]), span_limit=ns)
    peak, _ = measured_peak()
    runs = {}
    g_launches = 0
    # plain and remapped with reference rounding (bitwise), then the
    # contracted arithmetic (1e-12 tolerance; commutation-aware scheduling of
    # the local runs) without remapping
    for remap, mode in ((False, None), (True, None), (False, L.CMUL_CONTRACT)):
        st.apply_placements(pls, cmul_mode=mode, remap=remap)  # warm-up: plans, specialised passes
        L.call("diaq_jit_wait", -1.0)
        torch.cuda.synchronize()
        dist.barrier()
        st.stats = {k: 0 for k in st.stats}
        g_steps = max(1, min(args.steps, 3))
        ge0 = torch.cuda.Event(enable_timing=True)
        ge1 = torch.cuda.Event(enable_timing=True)
        gl0 = L.launch_count()
        ge0.record(s)
        for _ in range(g_steps):
            st.apply_placements(pls, cmul_mode=mode, remap=remap)
        ge1.record(s)
        torch.cuda.synchronize()
        launches = L.launch_count() - gl0
        g_ms = max_over_ranks(dist, ge0.elapsed_time(ge1), dev)
        stats = {k: (v // g_steps if isinstance(v, int) else v) for k, v in st.stats.items()}
        passes = launches / g_steps
        # per-rank HBM: every launch sweeps the rank's shard (32 B per local
        # amplitude: read + write); partner reads arrive over NVLink, not HBM
        hbm_bytes = passes * 32 * 2**lb
        runs["contracted" if mode else ("remap" if remap else "plain")] = {
            "gates_per_s": round(len(pls) * g_steps / (g_ms * 1e-3), 2), "s_per_circuit": round(g_ms / g_steps / 1e3, 4),
            "launches_per_circuit": round(passes, 1), "cross_shard_ops": stats.get("exchanged", 0),
            "swaps": stats.get("swaps", 0), "partner_bytes_read_per_rank": stats.get("bytes_received", 0),
            "hbm_frac_per_rank": round(hbm_bytes / (g_ms / g_steps * 1e-3) / 1e9 / peak, 4), "stats": stats}
        if not remap and mode is None:
            g_launches = launches
            plain_ms, plain_steps = g_ms, g_steps
    norm = st.norm()
    extra = {"gates_per_step": len(pls), "steps": plain_steps, "layers": layers, "circuit_qubits": ns,
             "local_qubits": lb, "mode": f"config 5: sharded over {world} ranks (top {p} bits), weak scaling",
             "transport": transport, "runs": runs, "norm_err": abs(1.0 - norm),
             "norm_ok": abs(1.0 - norm) < 1e-10}
    return len(pls) * plain_steps, plain_ms, g_launches, norm, ns, extra


def secondary_workloads(args, D, L, W, torch) -> dict:
    """The other BASELINE configs (launch-bound sizes), device-timed."""
    out = {}
    s = torch.cuda.current_stream()

    def dev_time(fn, reps):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            fn()
        e1.record(s)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    # config 1: spmv n=14 (3 diagonals), latency-bound
    c1 = W.config1(0)
    a1 = D.kron_identity(c1["left"], D.from_dense(c1["u"], 0.0), c1["right"])
    x1 = torch.from_numpy(c1["x"]).cuda()
    for _ in range(500):  # steady state (allocator, launch caches, clocks)
        D.spmv(a1, x1)
    ms = dev_time(lambda: D.spmv(a1, x1), 2000)
    out["config1_spmv_n14"] = {"us_per_spmv": round(ms * 1e3, 2),
                               "GBs": round(alg_bytes(2**14, a1.diag_indices()) / ms / 1e6, 1),
                               "note": "public D.spmv(a, cuda x) per call, 2000 back-to-back calls after 500 warm-up "
                                       "(host-bound: the kernel itself is ~3.8 us)"}
    # config 2: spgemm n=12, sweep of 64 seeded pairs (products/s incl. plan + prune readback)
    pairs = []
    for seed in range(64):
        p = W.config2(seed)
        span = D.build_span_unitary(D.from_dense(p["u4"], 0.0), p["u4_positions"], p["u4_span"])
        A = D.kron_identity(p["a_left"], span, p["a_right"])
        B = D.matmul(D.kron_identity(p["b1_left"], D.from_dense(p["u2"], 0.0), p["b1_right"]),
                     D.kron_identity(p["b0_left"], D.from_dense(W.rz(p["theta"]), 0.0), p["b0_right"]))
        pairs.append((A, B))
    for A, B in pairs[:3]:
        D.matmul(A, B)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for A, B in pairs:
        C = D.matmul(A, B)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / len(pairs)
    D.matrix.matmul_batch(pairs)
    torch.cuda.synchronize()
    bt = []
    for _ in range(5):
        t0 = time.perf_counter()
        D.matrix.matmul_batch(pairs)
        torch.cuda.synchronize()
        bt.append((time.perf_counter() - t0) / len(pairs))
    db = statistics.median(bt)
    out["config2_spgemm_n12"] = {"us_per_product": round(dt * 1e6, 1), "products_per_s": round(1 / dt, 1),
                                 "c_diagonals": C.diag_count(), "note": "wall clock per matmul() call",
                                 "sweep_us_per_product": round(db * 1e6, 2),
                                 "sweep_products_per_s": round(1 / db, 1),
                                 "sweep_note": "matmul_batch(64 pairs): device plan + multiply + prune, "
                                               "wall clock incl. sync, median of 5"}
    # config 3: random layered circuit n=20, 40 layers, 1200 gates
    ops = W.random_layered_ops(20, 40, seed=0)
    pls = D.compile_circuit(D.Circuit(20, [D.GateOp(*o) for o in ops]), span_limit=20)
    st = D.init_state(20)
    D.run_gates(st, pls, inplace=True)
    L.call("diaq_jit_wait", -1.0)  # specialised passes (one-time compile)
    ms = dev_time(lambda: D.run_gates(st, pls, inplace=True), 3)
    circ3 = D.Circuit(20, [D.GateOp(*o) for o in ops])
    t0 = time.perf_counter()
    res = D.run(circ3, shots=1024, seed=0, span_limit=20)
    first_s = time.perf_counter() - t0  # compile_circuit + packing on a cold cache
    walls = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = D.run(circ3, shots=1024, seed=0, span_limit=20)
        walls.append(time.perf_counter() - t0)
    e2e_s = statistics.median(walls)
    # config 5 shape on one GPU: a 2^29-amplitude state split into 2 emulated
    # shards (same plans and kernels as the NCCL path; the exchange is a
    # device copy here), 4 random layers drawn over all 29 qubits, without
    # and with qubit remapping (shard.remap_plan)
    from paper_2405_01250_b200.shard import run_emulated
    ops5 = W.random_layered_ops(29, 4, seed=0)
    pls5 = D.compile_circuit(D.Circuit(29, [D.GateOp(*o) for o in ops5]), span_limit=29)
    for remap in (False, True):
        run_emulated(29, 2, pls5, remap=remap)  # warm-up
        L.call("diaq_jit_wait", -1.0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        shards, st5 = run_emulated(29, 2, pls5, remap=remap)
        torch.cuda.synchronize()
        dt5 = time.perf_counter() - t0
        key = "config5_sharded_emulated_n29_p2" + ("_remap" if remap else "")
        out[key] = {"gates": len(pls5), "layers": 4, "s_per_circuit": round(dt5, 4),
                    "gates_per_s": round(len(pls5) / dt5, 1), "stats": st5,
                    "note": "2 shards on one GPU, wall clock; exchange = device copy (NVLink unmeasured); "
                            "partner_shards_read = what in-place peer reads fetch"}
        del shards
    # the metric's Haar4 gate kind at n=28: a layer of 14 Haar-random two-qubit
    # gates on a seeded random matching (fused passes, device time per layer)
    rng = np.random.default_rng(0)
    perm = rng.permutation(28)
    pls_h = []
    for i in range(14):
        qa, qb = int(perm[2 * i]), int(perm[2 * i + 1])
        lo, hi = min(qa, qb), max(qa, qb)
        pls_h.append(D.Placement(2**lo, None, 2 ** (27 - hi), lo, hi, "haar",
                                 gate=(W.haar(rng, 4), [qa - lo, qb - lo])))
    for mode, tag in ((None, ""), (L.CMUL_CONTRACT, "_contracted")):
        st_h = D.init_state(28)
        D.run_gates(st_h, pls_h, cmul_mode=mode, inplace=True)
        L.call("diaq_jit_wait", -1.0)
        ms_h = dev_time(lambda: D.run_gates(st_h, pls_h, cmul_mode=mode, inplace=True), 3)
        out["haar4_layer_n28" + tag] = {"gates": len(pls_h), "ms_per_layer": round(ms_h, 3),
                                        "gates_per_s": round(len(pls_h) / ms_h * 1e3, 1)}
        del st_h
    # the benchmark's layer kind as a deep program at the metric's size: n=28, 20
    # layers (840 gates) in one run_gates call -- the schedule packs several
    # layers into a pass (contracted arithmetic: lookahead tile bits, phase
    # slots), which a one-layer step cannot show
    ops28 = W.random_layered_ops(28, 20, seed=0)
    pls28 = D.compile_circuit(D.Circuit(28, [D.GateOp(*o) for o in ops28]), span_limit=28)
    for mode, tag in ((None, ""), (L.CMUL_CONTRACT, "_contracted")):
        st28 = D.init_state(28)
        D.run_gates(st28, pls28, cmul_mode=mode, inplace=True)
        L.call("diaq_jit_wait", -1.0)
        spec0 = jit_stats(L)["launches"]
        D.run_gates(st28, pls28, cmul_mode=mode, inplace=True)
        npass28 = jit_stats(L)["launches"] - spec0
        ms28 = dev_time(lambda: D.run_gates(st28, pls28, cmul_mode=mode, inplace=True), 3)
        out["layered_n28_20layers" + tag] = {
            "gates": len(pls28), "ms_per_circuit": round(ms28, 3), "gates_per_s": round(len(pls28) / ms28 * 1e3, 1),
            "hbm_passes": npass28, "ms_per_pass": round(ms28 / max(1, npass28), 3),
            "numerics": "contracted" if mode else "reference rounding (bitwise)",
            "norm_err": abs(1.0 - st28.norm())}
        del st28
    # config 5 at its 1-GPU size: n=30 (16 GB state), 20 random layers, norm check
    ops30 = W.random_layered_ops(30, 20, seed=0)
    pls30 = D.compile_circuit(D.Circuit(30, [D.GateOp(*o) for o in ops30]), span_limit=30)
    for mode, tag in ((None, ""), (L.CMUL_CONTRACT, "_contracted")):
        st30 = D.init_state(30, max_qubits=30)
        D.run_gates(st30, pls30, cmul_mode=mode, inplace=True)  # warm-up (program cache, specialised passes)
        L.call("diaq_jit_wait", -1.0)
        del st30
        reps30 = []
        for _ in range(3):  # each rep from |0..0>: device time of the whole 900-gate circuit
            st30 = D.init_state(30, max_qubits=30)
            spec0 = jit_stats(L)["launches"]
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(s)
            D.run_gates(st30, pls30, cmul_mode=mode, inplace=True)
            e1.record(s)
            torch.cuda.synchronize()
            reps30.append((e0.elapsed_time(e1), jit_stats(L)["launches"] - spec0))
            if len(reps30) < 3:
                del st30
        ms30 = sorted(r[0] for r in reps30)[1]
        out["config5_n30_1gpu" + tag] = {
            "gates": len(pls30), "layers": 20, "s_per_circuit": round(ms30 / 1e3, 4),
            "gates_per_s": round(len(pls30) / ms30 * 1e3, 1), "norm_err": abs(1.0 - st30.norm()),
            "reps_s": [round(r[0] / 1e3, 4) for r in reps30], "specialised_launches": [r[1] for r in reps30],
            "numerics": "contracted" if mode else "reference rounding (bitwise)",
            "note": "device time (CUDA events) of run_gates on |0..0>, fused passes; median of 3"}
        del st30
    out["config3_circuit_n20"] = {"gates": len(pls), "ms_per_circuit": round(ms, 3),
                                  "gates_per_s": round(len(pls) / ms * 1e3, 1),
                                  "run_api_wall_s": round(e2e_s, 4),
                                  "run_api_first_call_s": round(first_s, 4),
                                  "run_api_apply_ms": round(res.timings_ns["apply_total"] / 1e6, 3),
                                  "run_api_sample_ms": round(res.timings_ns["sample"] / 1e6, 3),
                                  "run_api_note": "run(circuit, shots=1024): wall median of 5 after a cold first call"}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--qubits", "--n", dest="n", type=int, default=N_QUBITS)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--replicas", action="store_true",
                    help="N>1: independent spmv / n=28 layer replicas instead of the sharded product and circuit")
    ap.add_argument("--circuit-qubits", type=int, default=30,
                    help="N>1: local qubits per rank of the sharded config-5 circuit (n = this + log2 N)")
    ap.add_argument("--circuit-layers", type=int, default=20, help="N>1: layers of the config-5 circuit")
    ap.add_argument("--transport", default="peer", choices=["peer", "nccl"],
                    help="sharded gates: partner shards read in place over peer memory, or NCCL-staged")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
