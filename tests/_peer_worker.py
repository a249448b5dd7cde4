"""One rank of the peer-memory sharded run (launched by test_gpu_peer.py):
gloo for handles/barriers, CUDA IPC mappings of the partner shards, and the
multi-source kernel reading them in place.  Rank 0 writes the gathered
state to --out."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rank", type=int, required=True)
    ap.add_argument("--world", type=int, required=True)
    ap.add_argument("--port", type=int, required=True)
    ap.add_argument("--n", type=int, required=True)
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--cmul", type=int, default=1)
    ap.add_argument("--tile", type=int, default=12)
    ap.add_argument("--out", required=True)
    ap.add_argument("--mode", default="gates", choices=["gates", "spmv"])
    ap.add_argument("--remap", type=int, default=0)
    a = ap.parse_args()
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2405_01250_b200 as D
    from paper_2405_01250_b200 import workloads as W
    from paper_2405_01250_b200.shard import PeerComm, ShardedState

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{a.port}", rank=a.rank, world_size=a.world)
    torch.cuda.set_device(0)
    D.sim.FUSE_TILE_BITS = a.tile
    comm = PeerComm()
    if a.mode == "spmv":
        run_spmv(a, comm)
        return
    ops = W.random_layered_ops(a.n, a.layers, seed=a.seed)
    ops += [("h", (0,), ()), ("cx", (0, a.n - 1), ()), ("ry", (1,), (0.7,)), ("swap", (0, 2), ()),
            ("cx", (a.n - 1, 0), ()), ("u3", (0,), (0.3, 0.2, 0.1))]
    pls = D.compile_circuit(D.Circuit(a.n, [D.GateOp(*o) for o in ops]), span_limit=a.n)
    st = ShardedState.basis(a.n, comm)
    st.apply_placements(pls, cmul_mode=a.cmul, remap=bool(a.remap))
    norm = st.norm()
    full = st.gather()
    comm.barrier()  # nobody unmaps or frees while a partner may still read
    if a.rank == 0:
        np.save(a.out, full.cpu().numpy())
        with open(a.out + ".stats", "w") as f:
            f.write(repr({"stats": st.stats, "norm": norm}))
    comm.close()
    dist.destroy_process_group()


def run_spmv(a, comm):
    """config-4 offsets at n=22: every rank's x slice in an exportable buffer,
    partners' slices mapped, the sharded kernel reads them in place."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2405_01250_b200 as D
    from paper_2405_01250_b200 import _lib as L
    from paper_2405_01250_b200 import workloads as W
    from paper_2405_01250_b200.shard import ShardedDiaq

    c4 = W.config4(22, seed=0, with_x=True)
    span = D.build_span_unitary(D.from_dense(c4["u4"], 0.0), c4["positions"], c4["span"])
    full = D.kron_identity(1, span, c4["right"])
    sd = ShardedDiaq.from_matrix(full, a.rank, a.world)
    xs, ptr = L.shared_c128(sd.nrows)
    xs.copy_(torch.from_numpy(c4["x"][sd.row0:sd.row0 + sd.nrows]).cuda())
    table = comm.share([ptr])
    comm.barrier()  # every slice written before anyone reads it
    y = sd.spmv([row[0] for row in table])
    comm.barrier()  # partners done reading our slice
    parts = comm.gather(y)
    if a.rank == 0:
        np.save(a.out, parts.cpu().numpy())
    comm.barrier()
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
