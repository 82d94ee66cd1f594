#!/usr/bin/env python3
"""Record a step kernel's DRAM traffic and compute counters from an ncu
--set full capture into profiles/traffic.json (read by bench.py's roofline).

    python tools/traffic_from_ncu.py <rep.ncu-rep> <config/dtype key> [--launches-per-step N]

Per launch: dram__bytes_read.sum + dram__bytes_write.sum; per step (sum over
the step's launches in the capture): warp instructions, the FP pipe's
active percentage (FP64 for f64, FMA for f32) weighted by duration, and the
duration under ncu.
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
rep, key = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, data = rows[0], rows[2:]


def val(r, k):
    return float(r[hdr.index(k)].replace(",", ""))


f32 = key.endswith("f32")
pipe = ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active" if f32 else
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active")
scale = {"Tbyte": 1e12, "Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}


def nbytes(r, k):
    return val(r, k) * scale[rows[1][hdr.index(k)]]


dram = [nbytes(r, "dram__bytes_read.sum") + nbytes(r, "dram__bytes_write.sum") for r in data]
ms = [val(r, "gpu__time_duration.sum") for r in data]
tu = rows[1][hdr.index("gpu__time_duration.sum")]
unit = {"msecond": 1.0, "ms": 1.0, "usecond": 1e-3, "us": 1e-3, "nsecond": 1e-6, "ns": 1e-6, "second": 1e3, "s": 1e3}[tu]
ms = [m * unit for m in ms]
inst = [val(r, "smsp__inst_executed.sum") for r in data]
pct = [val(r, pipe) for r in data]
ipc = [val(r, "sm__inst_executed.avg.per_cycle_active") for r in data]
names = [r[hdr.index("Kernel Name")] for r in data]
tot_ms = sum(ms)
rec = {
    "dram_bytes_per_launch": sum(dram) / len(dram),
    "dram_bytes_per_step": sum(dram),
    "warp_inst_per_step": sum(inst),
    "fp_pipe": "fma" if f32 else "fp64",
    "fp_pipe_active_pct": sum(p * m for p, m in zip(pct, ms)) / tot_ms,
    "ncu_ms_per_step": tot_ms,
    "ipc": sum(i * m for i, m in zip(ipc, ms)) / tot_ms,
    "launches_in_capture": len(data),
    "kernel": "; ".join(n[:110] for n in names),
    "source": f"{Path(rep).name} (ncu --set full; dram__bytes_read+write, smsp__inst_executed, {pipe})",
}
p = ROOT / "profiles" / "traffic.json"
d = json.loads(p.read_text()) if p.exists() else {}
d[key] = rec
p.write_text(json.dumps(d, indent=1) + "\n")
print(json.dumps({key: rec}, indent=1))
