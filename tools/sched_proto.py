"""Prototype of the fused-pass scheduler's pass-count model (host only, no
device): first-fit tile bits (what csrc/fused.cu does under the contracted
arithmetic) against a lookahead choice of the tile bits.
  python tools/sched_proto.py [n] [layers] [seed]"""
import sys
import itertools

sys.path.insert(0, '/root/repo')
from paper_2405_01250_b200 import workloads as W

T, LOW = 11, 3
MAXMEM = int(sys.argv[4]) if len(sys.argv) > 4 else 24


def gates_of(ops):
    out = []
    for name, qs, _ in ops:
        if name == "cx":
            out.append(("p", qs[1], qs[0]))       # target (mixing), control
        elif name == "rz":
            out.append(("z", qs[0], None))
        else:
            out.append(("d", qs[0], None))
    return out


def sweep(gates, pending, n, B=None, tail_insert=False, maxmem=MAXMEM, count_perm=True):
    """One pass.  B None: first-fit growth.  Returns (members, deferred)."""
    inb = set(range(LOW)) if B is None else set(B)
    grow = B is None
    blocked = 0
    members, deferred = [], []
    tail_on = False
    tailq = 0
    nm = 0
    allq = (1 << n) - 1
    for idx, i in enumerate(pending):
        if blocked == allq:
            deferred.extend(pending[idx:])
            break
        kind, q, c = gates[i]
        qm = (1 << q) | ((1 << c) if c is not None else 0)
        if qm & blocked:
            deferred.append(i); blocked |= qm; continue
        full = nm >= maxmem
        if kind == "p":
            if not tail_on and q in inb and not full:
                members.append(i); nm += 1 if count_perm else 0; continue
            if not tail_on and grow and len(inb) < T and not full:
                inb.add(q); members.append(i); nm += 1 if count_perm else 0; continue
            if not members:
                # opens the pass: would take its bits
                if grow:
                    inb.add(q)
                    members.append(i); nm += 1 if count_perm else 0; continue
                deferred.append(i); blocked |= qm; continue
            tail_on = True
            tailq |= qm
            members.append(i)
            continue
        if tail_on and (not tail_insert or (qm & tailq)):
            deferred.append(i); blocked |= qm; continue
        if full:
            deferred.append(i); blocked |= qm; continue
        if kind == "z" or q in inb:
            members.append(i); nm += 1; continue
        if grow and len(inb) < T:
            inb.add(q); members.append(i); nm += 1; continue
        deferred.append(i); blocked |= qm
    return members, deferred, inb


def score(gates, members):
    return sum(1.0 if gates[i][0] == "d" else 0.25 for i in members)


def choose_bits(gates, pending, n, **kw):
    m0, _, B = sweep(gates, pending, n, None, **kw)
    B = set(B)
    for b in range(n):
        if len(B) >= T:
            break
        B.add(b)
    best = score(gates, sweep(gates, pending, n, B, **kw)[0])
    # candidates: qubits of the next few hundred pending gates
    improved = True
    it = 0
    while improved and it < 6:
        improved = False
        it += 1
        for out in sorted(B - set(range(LOW))):
            for inn in range(LOW, n):
                if inn in B:
                    continue
                C = (B - {out}) | {inn}
                s = score(gates, sweep(gates, pending, n, C, **kw)[0])
                if s > best + 1e-9:
                    best, B, improved = s, C, True
                    break
            if improved:
                break
    return B


def schedule(gates, n, lookahead, **kw):
    pending = list(range(len(gates)))
    passes = []
    while pending:
        B = choose_bits(gates, pending, n, **kw) if lookahead else None
        mem, pending2, _ = sweep(gates, pending, n, B, **kw)
        if not mem:   # preset bits admit nothing: fall back to first fit
            mem, pending2, _ = sweep(gates, pending, n, None, **kw)
        assert mem
        passes.append(mem)
        pending = pending2
    return passes


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    layers = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    seed = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    g = gates_of(W.random_layered_ops(n, layers, seed=seed))
    for la, ti, cp in itertools.product([False, True], [False, True], [True, False]):
        p = schedule(g, n, la, tail_insert=ti, count_perm=cp)
        sizes = [len(m) for m in p]
        print(f"lookahead={la} tail_insert={ti} count_perm={cp}: passes {len(p)}  max members {max(sizes)}")
