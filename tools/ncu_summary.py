#!/usr/bin/env python3
"""Summarise ncu captures into profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py --tag r01 --full gpurun_out/spmv_full.ncu-rep gpurun_out/gate_full.ncu-rep \
        --launches gpurun_out/launches.csv

Writes profiles/<tag>_ncu_full.json (per-kernel key metrics of the --set full
captures), profiles/<tag>_launches.csv (the launch list of the bench command,
cold-cache serialised times) + a per-kernel share table, and updates
profiles/ncu_summary.json (dram bytes per launch, read by bench.py as
roofline.traffic).
"""
from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import os
import shutil
import subprocess

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sectors_srcunit_tex_op_read_evict_first_lookup_miss.sum",
    "lts__t_sectors_srcunit_tex_op_read_evict_normal_lookup_miss.sum",
    "lts__t_sectors_srcunit_tex_op_read_evict_normal_lookup_hit.sum",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
]

SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}


def raw(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        rec = {"kernel": d.get("Kernel Name", "")}
        for k in KEYS:
            if k in d:
                u = units[hdr.index(k)]
                v = d[k].replace(",", "")
                try:
                    val = float(v)
                except ValueError:
                    continue
                if u in SCALE:
                    val *= SCALE[u]
                    u = "byte"
                if u == "ms":
                    val *= 1e6
                    u = "ns"
                elif u == "us":
                    val *= 1e3
                    u = "ns"
                rec[k] = val
                rec[k + ".unit"] = u
        res.append(rec)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--full", nargs="*", default=[])
    ap.add_argument("--launches")
    ap.add_argument("--cmd", default="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-secondary",
                    help="the profiled command, for the summary header")
    args = ap.parse_args()
    os.makedirs("profiles", exist_ok=True)
    full = {}
    for rep in args.full:
        full[os.path.basename(rep)] = raw(rep)
    with open(f"profiles/{args.tag}_ncu_full.json", "w") as f:
        json.dump(full, f, indent=1)
    summ_path = "profiles/ncu_summary.json"
    summ = json.load(open(summ_path)) if os.path.exists(summ_path) else {}
    for name, recs in full.items():
        for rec in recs:
            tot = rec.get("dram__bytes_read.sum", 0) + rec.get("dram__bytes_write.sum", 0)
            if "spmv" in rec["kernel"]:
                summ["spmv_dram_bytes_per_launch"] = tot
                summ["spmv_source"] = f"profiles/{args.tag}_ncu_full.json ({name})"
            elif any(k in rec["kernel"] for k in ("gate_kernel", "tile_pass_kernel", "diaq_jit_pass")):
                summ["gate_dram_bytes_per_launch"] = tot
                summ["gate_source"] = f"profiles/{args.tag}_ncu_full.json ({name})"
    with open(summ_path, "w") as f:
        json.dump(summ, f, indent=1)
    if args.launches:
        shutil.copy(args.launches, f"profiles/{args.tag}_launches.csv")
        lines = open(args.launches).read().splitlines()
        start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
        rows = list(csv.DictReader(lines[start:]))
        agg = collections.OrderedDict()
        for r in rows:
            if r.get("Metric Name") != "gpu__time_duration.sum":
                continue
            k = r["Kernel Name"].split("(")[0][:90]
            ns = float(r["Metric Value"].replace(",", ""))
            a = agg.setdefault(k, [0, 0.0])
            a[0] += 1
            a[1] += ns
        total = sum(v[1] for v in agg.values())
        with open(f"profiles/{args.tag}_launch_shares.md", "w") as f:
            f.write(f"# Launch list summary ({args.tag}): ncu gpu__time_duration.sum, --clock-control none\n\n")
            f.write(f"Cold-cache, serialised per-launch times of `{args.cmd}`; compare shares, not absolutes.\n\n")
            f.write("| kernel | launches | total ms | avg ms | share |\n|---|---|---|---|---|\n")
            for k, (c, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
                f.write(f"| `{k}` | {c} | {ns / 1e6:.3f} | {ns / c / 1e6:.4f} | {100 * ns / total:.1f}% |\n")
    print(json.dumps(summ, indent=1))


if __name__ == "__main__":
    main()
