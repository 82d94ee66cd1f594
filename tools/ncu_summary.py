#!/usr/bin/env python3
"""Summarise an .ncu-rep (per kernel): time, DRAM bytes, pipe utilisation, stalls."""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64pipe%"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "fma%"),
    ("sm__inst_executed.avg.per_cycle_active", "ipc"),
    ("smsp__inst_executed.sum", "warp_inst"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
    ("launch__registers_per_thread", "regs"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1%"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2%"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wf"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "gld_sectors"),
    ("l1tex__t_sector_hit_rate.pct", "l1hit%"),
    ("lts__t_sector_hit_rate.pct", "l2hit%"),
    ("lts__t_sectors_srcunit_tex_op_read.sum", "l2rd_sectors"),
    ("l1tex__m_xbar2l1tex_read_bytes.sum", "l2_to_l1_bytes"),
    ("sm__sass_thread_inst_executed_op_dfma_pred_on.sum", "dfma"),
    ("sm__sass_thread_inst_executed_op_dmul_pred_on.sum", "dmul"),
    ("sm__sass_thread_inst_executed_op_dadd_pred_on.sum", "dadd"),
    ("sm__sass_thread_inst_executed_op_ffma_pred_on.sum", "ffma"),
]
STALLS = ["long_scoreboard", "short_scoreboard", "wait", "barrier", "mio_throttle", "math_pipe_throttle",
          "not_selected", "selected", "lg_throttle", "dispatch_stall", "no_instructions", "branch_resolving",
          "drain", "tex_throttle", "membar", "sleeping"]

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
for row in rows[2:]:
    name = row[hdr.index("Kernel Name")][:60]
    print(f"== {name}  grid={row[hdr.index('Grid Size')] if 'Grid Size' in hdr else '?'} block={row[hdr.index('Block Size')] if 'Block Size' in hdr else '?'}")
    for k, short in KEYS:
        if k in hdr:
            print(f"   {short:12s} {row[hdr.index(k)]}")
    tot = 0
    vals = {}
    for s in STALLS:
        k = f"smsp__pcsamp_warps_issue_stalled_{s}"
        if k in hdr and row[hdr.index(k)]:
            vals[s] = float(row[hdr.index(k)].replace(",", ""))
            tot += vals[s]
    if tot:
        print("   stalls: " + ", ".join(f"{s} {100*v/tot:.1f}%" for s, v in sorted(vals.items(), key=lambda x: -x[1]) if v / tot > 0.01))
