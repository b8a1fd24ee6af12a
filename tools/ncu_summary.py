#!/usr/bin/env python
"""Summarise an ncu report (.ncu-rep) into the per-launch numbers quoted in
DESIGN.md / bench.py: duration, issue / pipe utilisation, DRAM bytes,
registers, occupancy, top stall reasons.  Usage:

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/rNN_name.txt
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_active.avg", "sm_cycles_active"),
    ("smsp__inst_executed.sum", "warp_insts"),
    ("sm__inst_issued.avg.pct_of_peak_sustained_active", "issue_%"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "alu_pipe_%"),
    ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", "fmaheavy_%"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma_%"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu_%"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("lts__t_sectors_srcunit_tex_op_read.sum", "l2_read_sectors"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_%"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2_throughput_%"),
    ("l1tex__t_sector_hit_rate.pct", "l1_hit_%"),
    ("launch__registers_per_thread", "regs"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
    ("launch__grid_size", "grid"),
]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    name_i = hdr.index("Kernel Name")
    print(f"# ncu summary of {path}")
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        print(f"\n## launch {d.get('ID', '?')}: {r[name_i][:90]}")
        for k, label in KEYS:
            if k in d:
                print(f"  {label:18s} {d[k]} {u.get(k, '')}")
        st = sorted(((k, float(v.replace(',', '') or 0)) for k, v in d.items()
                     if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")),
                    key=lambda kv: -kv[1])
        tot = sum(v for _, v in st) or 1
        print("  stall samples      " + ", ".join(f"{k.split('stalled_')[1]} {100 * v / tot:.1f}%"
                                                   for k, v in st[:8]))


if __name__ == "__main__":
    main(sys.argv[1])
