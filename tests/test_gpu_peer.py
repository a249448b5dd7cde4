"""GPU: the peer-memory transport of the sharded state (CUDA IPC mappings of
the partner shards read in place by the multi-source kernel).  Two ranks run
as two processes on the one GPU of the test box -- host barriers only, no
kernel waits on another -- and must equal the unsharded run bitwise."""
from __future__ import annotations

import ast
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import paper_2405_01250_b200 as D
from conftest import ROOT
from paper_2405_01250_b200 import _lib as L
from paper_2405_01250_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("n,tile,remap", [(12, 12, 0), (14, 0, 0), (16, 11, 0), (14, 0, 1), (16, 11, 1)])
def test_peer_sharded_matches_unsharded(tmp_path, configs, n, tile, remap):
    cmul = L.CMUL_FMA if configs["meta"]["numpy_cmul"] == "fma" else L.CMUL_PLAIN
    out = str(tmp_path / "state.npy")
    port = _port()
    worker = os.path.join(ROOT, "tests", "_peer_worker.py")
    procs = [subprocess.Popen([sys.executable, worker, "--rank", str(r), "--world", "2", "--port", str(port),
                               "--n", str(n), "--cmul", str(cmul), "--tile", str(tile), "--out", out,
                               "--remap", str(remap)],
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True) for r in range(2)]
    logs = []
    try:
        for p in procs:
            logs.append(p.communicate(timeout=300)[0])
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    assert all(p.returncode == 0 for p in procs), "\n".join(logs)
    got = np.load(out)
    info = ast.literal_eval(open(out + ".stats").read())
    assert info["stats"]["exchanged"] > 0 and abs(info["norm"] - 1.0) < 1e-12
    if remap:  # half-shard swaps instead of whole-shard partner reads
        assert info["stats"]["swaps"] > 0
    ops = W.random_layered_ops(n, 2, seed=0)
    ops += [("h", (0,), ()), ("cx", (0, n - 1), ()), ("ry", (1,), (0.7,)), ("swap", (0, 2), ()),
            ("cx", (n - 1, 0), ()), ("u3", (0,), (0.3, 0.2, 0.1))]
    pls = D.compile_circuit(D.Circuit(n, [D.GateOp(*o) for o in ops]), span_limit=n)
    want = D.run_gates(D.init_state(n), pls, cmul_mode=cmul).amps
    assert np.array_equal(got, want)


def test_peer_sharded_spmv_config4(tmp_path):
    """Sharded spmv whose +-2^21 offsets cross the shard boundary: partner x
    read in place through a CUDA IPC mapping, bitwise the single-GPU spmv."""
    import torch
    out = str(tmp_path / "y.npy")
    port = _port()
    worker = os.path.join(ROOT, "tests", "_peer_worker.py")
    procs = [subprocess.Popen([sys.executable, worker, "--rank", str(r), "--world", "2", "--port", str(port),
                               "--n", "22", "--mode", "spmv", "--out", out],
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True) for r in range(2)]
    logs = []
    try:
        for p in procs:
            logs.append(p.communicate(timeout=300)[0])
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    assert all(p.returncode == 0 for p in procs), "\n".join(logs)
    c4 = W.config4(22, seed=0, with_x=True)
    span = D.build_span_unitary(D.from_dense(c4["u4"], 0.0), c4["positions"], c4["span"])
    a = D.kron_identity(1, span, c4["right"])
    want = D.spmv(a, torch.from_numpy(c4["x"]).cuda()).cpu().numpy()
    assert np.array_equal(np.load(out), want)


def test_bench_multi_rank_paths_on_one_gpu(tmp_path):
    """bench.py's N>1 code (row-sharded spmv with peer x loads, sharded gates
    over the peer transport) end to end with two ranks on the one GPU
    (gloo, host barriers only): a functional check, not a measurement."""
    import json
    env = dict(os.environ, DIAQ_BENCH_SAME_GPU="1", DIAQ_BENCH_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "3", "--no-e2e", "--no-cpu", "--no-secondary",
           "--qubits", "23", "--circuit-qubits", "16", "--circuit-layers", "3"]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-3000:]
    line = json.loads(p.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and "peer loads" in line["config"]["parallelism"]
    g = line["gates"]
    # the default N>1 gate measurement is the sharded config-5 circuit
    assert g["mode"].startswith("config 5") and g["circuit_qubits"] == 17 and g["transport"] == "peer"
    assert g["runs"]["plain"]["cross_shard_ops"] > 0 and g["runs"]["remap"]["swaps"] > 0
    assert g["runs"]["contracted"]["gates_per_s"] > 0  # the contracted arithmetic on the sharded path
    assert g["norm_ok"] and abs(g["norm_after"] - 1.0) < 1e-10


_NCCL_SCRIPT = r"""
import sys
sys.path.insert(0, {root!r})
import torch, torch.distributed as dist
import paper_2405_01250_b200 as D
from paper_2405_01250_b200 import workloads as W
from paper_2405_01250_b200.shard import PeerComm, ShardedState, TorchDistComm
torch.cuda.set_device(0)
dist.init_process_group("nccl", init_method="tcp://127.0.0.1:{port}", rank=0, world_size=1)
for comm in (PeerComm(), TorchDistComm()):
    st = ShardedState.basis(10, comm)
    ops = W.random_layered_ops(10, 2, seed=0)
    st.apply_placements(D.compile_circuit(D.Circuit(10, [D.GateOp(*o) for o in ops]), span_limit=10))
    if isinstance(comm, PeerComm):
        comm.order()   # events + gloo side-group barrier under an NCCL default group
    n = st.norm()      # all-reduce on the backend's device
    full = st.gather() # gather on the backend's device
    assert abs(n - 1.0) < 1e-12 and full.numel() == 1024 and full.device.type == "cuda", (n, full.device)
    assert comm.allreduce_max(3.0, st.local) == 3.0
    if isinstance(comm, PeerComm):
        comm.close()
dist.destroy_process_group()
print("nccl-ok")
"""


def test_peer_comm_collectives_under_nccl():
    """under an NCCL process group every host-side collective of
    PeerComm / TorchDistComm must hand CUDA tensors to NCCL (CPU tensors
    raise "No backend type associated with device type cpu"); the event
    ordering's host barrier runs on a gloo side group.  One rank (NCCL
    refuses two ranks on one GPU)."""
    script = _NCCL_SCRIPT.format(root=ROOT, port=_port())
    p = subprocess.run([sys.executable, "-c", script], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert p.returncode == 0 and "nccl-ok" in p.stdout, p.stdout[-2000:] + p.stderr[-3000:]
