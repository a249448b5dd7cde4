#!/usr/bin/env python3
"""Summarise an ncu --set full report of the fused passes for profiles/:
per kernel the duration, DRAM bytes, pipe utilisation (FP64, issue, shared
memory), occupancy and the warp-stall breakdown (raw page), plus the
dynamic opcode mix and an excerpt of the hottest SASS (source page).
  python tools/ncu_pass_summary.py REPORT.ncu-rep OUT_PREFIX [UNITS]
UNITS: thread-level work units per launch for the per-unit opcode mix
(default 2^28 amplitudes / 16 per thread = 2^24 threads-tiles)."""
import csv
import io
import json
import subprocess
import sys
from collections import Counter


def page(rep, name, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", name, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main(rep, prefix, units=float(2**24)):
    rows = page(rep, "raw")
    h = rows[0]
    summary = []
    for r in rows[2:]:
        g = lambda k: r[h.index(k)] if k in h else None  # noqa: E731
        f = lambda k: float(g(k).replace(",", "")) if g(k) not in (None, "") else None  # noqa: E731
        stalls = {}
        for i, k in enumerate(h):
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    stalls[k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(r[i])
                except ValueError:
                    pass
        summary.append({
            "kernel": g("Kernel Name"), "duration_ms": f("gpu__time_duration.sum"),
            "dram_bytes_read": f("dram__bytes_read.sum"), "dram_bytes_write": f("dram__bytes_write.sum"),
            "fp64_pipe_pct_active": f("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "issue_slots_pct": f("sm__instruction_throughput.avg.pct_of_peak_sustained_active"),
            "smem_wavefronts_pct": f("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
            "smem_bank_conflicts": f("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
            "warps_active_per_sm": f("sm__warps_active.avg.per_cycle_active"),
            "registers": f("launch__registers_per_thread"), "grid": f("launch__grid_size"),
            "block": f("launch__block_size"), "warp_instructions": f("smsp__inst_executed.sum"),
            "stall_cycles_per_issue": dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:12]),
        })
    with open(prefix + "_ncu_summary.json", "w") as fo:
        json.dump(summary, fo, indent=1)
    lines = []
    for s in summary:
        k = s["kernel"]
        src = page(rep, "source", ("--print-source", "sass", "-k", k))
        if len(src) < 3:
            continue
        hh = src[1]
        ie, sc, ws = hh.index("Instructions Executed"), hh.index("Source"), hh.index("Warp Stall Sampling (All Samples)")
        ops, body = Counter(), []
        for r in src[2:]:
            if len(r) <= ie or not r[ie].isdigit():
                continue
            toks = r[sc].split()
            op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
            ops[op] += int(r[ie])
            body.append((int(r[ie]), int(r[ws] or 0), r[sc].strip()))
        tot = sum(ops.values())
        # the source page's "Instructions Executed" sums to a multiple of
        # smsp__inst_executed.sum on this ncu (2x for these kernels): scale
        # the per-unit figures to the raw counter
        norm = (s["warp_instructions"] or tot) / tot
        lines.append(f"== {k}: dynamic opcode mix (per unit = warp instructions x32 / {units:.0f} thread-tiles; "
                     f"source-page counts scaled by {norm:.3f} to smsp__inst_executed.sum)")
        for op, v in ops.most_common(24):
            lines.append(f"  {op:12s} {int(v * norm):14d} {100 * v / tot:5.1f}%  per-unit {v * norm * 32 / units:8.1f}")
        hot = max(b[0] for b in body)
        seg = [b for b in body if b[0] == hot]
        lines.append(f"-- hottest straight-line block ({len(seg)} instructions executed {hot} times), first 60:")
        lines += [f"  {c:12d} {w:6d}  {t}" for c, w, t in seg[:60]]
    with open(prefix + "_sass_opmix.txt", "w") as fo:
        fo.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], *(float(a) for a in sys.argv[3:]))
