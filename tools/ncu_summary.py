#!/usr/bin/env python
"""Summarise ncu captures for profiles/: one block per .ncu-rep (key SOL metrics,
tensor-pipe TF32 utilisation, DRAM traffic) and, for a launch list CSV
(--metrics gpu__time_duration.sum), per-kernel-name totals.
    python tools/ncu_summary.py --rep a.ncu-rep [--rep b.ncu-rep] [--launches launches.csv] > profiles/X.md"""
import argparse
import collections
import csv
import io
import subprocess

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("sm__ops_path_tensor_op_utchmma_src_tf32_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_elapsed",
     "tensor pipe TF32 (UTCHMMA) % of peak"),
    ("sm__ops_path_tensor_op_utchmma_src_tf32_dst_fp32_sparsity_off.sum", "TF32 tensor ops executed (all 3 passes)"),
    ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem wavefronts for tensor core % peak"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem wavefronts for LSU % peak"),
    ("lts__t_sectors_srcunit_tex_op_read.sum", "L2 read sectors from SM"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput % peak"),
    ("launch__grid_size", "grid"),
    ("launch__registers_per_thread", "registers/thread"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
]


def rep_block(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    lines = [f"### {path}", ""]
    for vals in rows[2:]:
        ix = {h: i for i, h in enumerate(hdr)}
        lines.append(f"kernel: `{vals[ix['Kernel Name']]}`  grid {vals[ix.get('launch__grid_size', 0)]}")
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        for k, name in KEYS:
            if k in ix:
                lines.append(f"| {name} (`{k}`) | {vals[ix[k]]} | {units[ix[k]]} |")
        lines.append("")
    return "\n".join(lines)


def launches_block(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        name = r[ki].split("(")[0].replace("void ", "")
        tot[name][0] += 1
        tot[name][1] += float(r[vi].replace(",", "")) / 1e3
    lines = [f"### launch list {path} (cold-cache, serialised: compare shares, not absolutes)", "",
             "| kernel | launches | total us | share |", "|---|---|---|---|"]
    s = sum(v[1] for v in tot.values())
    for name, (n, us) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{name}` | {n} | {us:.1f} | {us / s:.3f} |")
    return "\n".join(lines) + "\n"


ap = argparse.ArgumentParser()
ap.add_argument("--rep", action="append", default=[])
ap.add_argument("--launches", default=None)
a = ap.parse_args()
for r in a.rep:
    print(rep_block(r))
if a.launches:
    print(launches_block(a.launches))
