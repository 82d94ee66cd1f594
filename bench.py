#!/usr/bin/env python3
"""Throughput of the B200-native MPDATA step (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c4|c2|c1|c5d|c5s] [--shares a,b,...]

One "step" is one MPDATA time step over the whole grid. The default workload
is BASELINE config 4 (1024x512x128 fp64, IORD=2, nonoscillatory, periodic),
the configuration the metric is quoted on at 1/2/4/8 GPUs; at N>1 (torchrun,
one process per GPU) the grid is split into i-slabs (even, or --shares) and
the step kernel pushes its edge planes into the CUDA-IPC-mapped neighbour
halos over NVLink, ordered by device flag words (--halo ipc, the default;
--halo nccl or a failed mapping uses a per-step NCCL exchange) — strong scaling.

``value`` = interior cell-updates of all ranks / max-over-ranks device time of
K steps (CUDA events inside the library, exchange included). ``e2e`` = the
same metric through the reference-facing host-buffer call
(imb_team_step_host: pinned H2D of x, the step, D2H of x, every step).
``--impl reference`` times the CPU restatement (oracle/, the reference has no
runnable MPDATA of its own) on all host cores over a bounded sample.
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
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "MPDATA 3D Gcell-updates/s per step at 1/2/4/8 B200; % of HBM roofline"
UNIT = "Gcell-updates/s"

# name -> (n, m, l, iord, nonos, fp64, recipe, description)
CONFIGS = {
    "c4": (1024, 512, 128, 2, True, True, 2, "BASELINE config 4: 1024x512x128 fp64 IORD=2 nonos"),
    "c2": (256, 256, 64, 2, True, True, 2, "BASELINE config 2: 256x256x64 fp64 IORD=2 nonos"),
    "c1": (64, 64, 32, 2, False, True, 1, "BASELINE config 1: 64x64x32 fp64 IORD=2"),
    "c5d": (2048, 1024, 128, 3, True, True, 2, "BASELINE config 5: 2048x1024x128 fp64 IORD=3 nonos"),
    "c5s": (2048, 1024, 128, 3, True, False, 2, "BASELINE config 5: 2048x1024x128 fp32 IORD=3 nonos"),
}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (FileNotFoundError, OSError):
            self.proc = None
        time.sleep(0.15)
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[q] for r in self.rows for q in range(4) if r[2 + q] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def spawn_ranks(n: int) -> int:
    """`bench.py --gpus N` outside torchrun: relaunch as N ranks (one process
    per GPU) through torch.distributed.run on 127.0.0.1 and return its code."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1",
           "--nproc-per-node", str(n), "--master-addr", "127.0.0.1", "--master-port", str(port),
           str(ROOT / "bench.py"), *sys.argv[1:]]
    print(f"bench: spawning {n} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_port_gcells(n, m, l, iord, nonos, fp64, recipe, planes, steps, threads, budget_s=0.0):
    """Times the CPU restatement (oracle/) on a slab sample of the workload grid.

    With ``budget_s`` > 0 the step count is raised until the timed region
    covers about that many seconds (a bounded sample of the workload)."""
    import numpy as np

    from oracle import oracle as O
    dt = np.float64 if fp64 else np.float32
    f = O.init_fields(recipe, n, m, l, seed=42, i0=0, ni=planes, dtype=dt)
    t0 = time.perf_counter()
    O.run(*f, iord=iord, nonos=nonos, steps=1, threads=threads)  # warm-up / first touch
    one = time.perf_counter() - t0
    if budget_s > 0:
        steps = max(steps, min(1000, int(budget_s / max(one, 1e-6))))
    t0 = time.perf_counter()
    O.run(*f, iord=iord, nonos=nonos, steps=steps, threads=threads)
    dt_s = time.perf_counter() - t0
    return planes * m * l * steps / dt_s / 1e9, dt_s, steps


def run_reference(args, cfg):
    """The reference arm: the CPU restatement of the path (oracle/, the
    reference ships no runnable MPDATA) on the FULL workload grid with every
    host thread: W untimed steps, then K timed steps in one call (its scratch
    is allocated once per call, as a resident CPU code would)."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import numpy as np

    from oracle import oracle as O
    n, m, l, iord, nonos, fp64, recipe, desc = cfg
    threads = os.cpu_count() or 1
    f = O.init_fields(recipe, n, m, l, seed=42, dtype=np.float64 if fp64 else np.float32)
    x = O.run(*f, iord=iord, nonos=nonos, steps=max(args.warmup, 0), threads=threads)
    t0 = time.perf_counter()
    O.run(x, *f[1:], iord=iord, nonos=nonos, steps=args.steps, threads=threads)
    dt_s = time.perf_counter() - t0
    value = n * m * l * args.steps / dt_s / 1e9
    sample = (f"the full {n}x{m}x{l} grid: {args.warmup} untimed + {args.steps} timed steps "
              f"({dt_s:.1f} s) on {threads} threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": max(world, args.gpus),
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt_s / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64" if fp64 else "f32", "data": "synthetic (seeded BASELINE recipe)",
        "config": {"workload": desc, "grid": [n, m, l], "iord": iord, "nonos": nonos,
                   "boundary": "periodic", "parallelism": "cpu threads"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "the reference ships no MPDATA implementation (SURVEY.md §0); the CPU arm is "
                "the oracle restatement oracle/mpdata_oracle.c, -O3 -ffp-contract=off, pthreads",
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--shares", default="",
                    help="N>1 slab shares: comma-separated planes, or a speed-function CSV "
                         "(cli measure output) to split with the FPM partitioner "
                         "(Algorithm 1 for even N, the exact DP otherwise)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--halo", default="ipc", choices=["nccl", "ipc"],
                    help="N>1 halo exchange: the step kernel pushing its edge planes into "
                         "the CUDA-IPC-mapped neighbour halos over NVLink (default; falls "
                         "back to NCCL if the mapping fails), or NCCL send/recv")
    ap.add_argument("--one-device", action="store_true",
                    help="testing only: every rank on GPU 0 (exercises the N>1 code path "
                         "on a 1-GPU box; the numbers are not a scaling result)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1507_01265_b200 import mpdata

    n, m, l, iord, nonos, fp64, recipe, desc = cfg
    world, rank, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo", rank=rank, world_size=world)
    if args.one_device:
        local = 0
    torch.cuda.set_device(local)
    if args.shares.endswith(".csv"):
        from paper_1507_01265_b200 import fpm
        model = fpm.read_csv(Path(args.shares).read_text())
        pr = fpm.PartitionProblem(n, world, model)
        part = fpm.partition_paired(pr) if world % 2 == 0 else fpm.partition_general(pr)
        shares = list(part.shares)
    elif args.shares:
        shares = [int(s) for s in args.shares.split(",")]
    else:
        shares = [n // world + (1 if r < n % world else 0) for r in range(world)]
    assert len(shares) == world and sum(shares) == n, "shares must cover the grid"
    i0 = sum(shares[:rank])
    opts = mpdata.Options(iord=iord, nonos=nonos, fp64=fp64)
    team = mpdata.Team(n, m, l, opts, device=local, i0=i0, ni=shares[rank])
    team.init_recipe(recipe, 42)
    halo = args.halo
    if world > 1 and halo == "ipc":
        blobs = [None] * world
        dist.all_gather_object(blobs, team.ipc_export())
        err = ""
        try:
            team.connect_ipc(blobs[(rank - 1) % world], blobs[(rank + 1) % world], world, rank)
        except mpdata._lib.ImbError as e:
            err = str(e)
        errs = [None] * world
        dist.all_gather_object(errs, err)
        if any(errs):  # every rank falls back together
            if rank == 0:
                print(f"ipc halo push unavailable ({next(e for e in errs if e)}); using NCCL",
                      file=sys.stderr)
            team.close()
            team = mpdata.Team(n, m, l, opts, device=local, i0=i0, ni=shares[rank])
            team.init_recipe(recipe, 42)
            halo = "nccl"
        dist.barrier()
    if world > 1 and halo == "nccl":
        uid = [mpdata.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        team.connect_nccl(uid[0], world, rank)
    me = {"rank": rank, "device": local, "pci": torch.cuda.get_device_properties(local).pci_bus_id
          if hasattr(torch.cuda.get_device_properties(local), "pci_bus_id") else None,
          "slab": [i0, shares[rank]], "halo": halo if world > 1 else "self-push"}
    ranks = [me]
    if world > 1:
        ranks = [None] * world
        dist.all_gather_object(ranks, me)
        if rank == 0:
            print(f"bench: {world} ranks, halo path {halo}: " +
                  ", ".join(f"rank {r['rank']} -> cuda:{r['device']} slab {r['slab']}"
                            for r in ranks), file=sys.stderr, flush=True)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    team.run(args.warmup)
    barrier()
    launches0 = team.launches
    with ClockSampler(local) as clk:
        comp, wall = team.run(args.steps)
    barrier()
    launches = team.launches - launches0
    wall_max = max_over_ranks(wall)
    comp_max = max_over_ranks(comp)
    cells = n * m * l
    value = cells * args.steps / wall_max / 1e9

    # ---- e2e through the reference-facing host-buffer call -----------------
    dt = np.float64 if fp64 else np.float32
    elem = 8 if fp64 else 4
    xin = torch.empty(team.shape, dtype=torch.float64 if fp64 else torch.float32,
                      pin_memory=True).numpy()
    xout = np.empty_like(xin)
    pin_out = torch.empty(team.shape, dtype=torch.float64 if fp64 else torch.float32,
                          pin_memory=True).numpy()
    xin[...] = team.download("x")
    team.step_host(xin, pin_out)  # warm
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        team.step_host(xin, pin_out)
        xin, pin_out = pin_out, xin
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    barrier()
    del xout, dt
    e2e_value = cells * args.e2e_steps / e2e_s / 1e9

    peak, peak_src = peaks()
    bytes_per_cell = 6 * elem  # psi,u,v,w,h read + psi write
    local_cells = shares[rank] * m * l
    per_step = comp_max / args.steps
    traffic = None  # DRAM bytes per launch from the committed ncu capture
    compute = None  # the secondary (compute) floors, from the same capture
    tfile = ROOT / "profiles" / "traffic.json"
    rec = None
    if tfile.exists():
        rec = json.loads(tfile.read_text()).get(f"{args.config}/{'f64' if fp64 else 'f32'}")
    if rec and world == 1:
        traffic = rec["dram_bytes_per_launch"]
        launches_per_step = max(1, round(launches / args.steps))
        if "warp_inst_per_step" in rec:
            # issue floor: every warp instruction of a step issued at 4 per SM
            # per clock (148 SMs, max SM clock); FP pipe floor: the step's
            # FP64 (fp32: FMA) pipe busy cycles, i.e. its measured utilisation
            # times its ncu duration. frac = floor / this run's step time.
            sm_hz = 1965e6
            issue_ms = rec["warp_inst_per_step"] / (148 * 4 * sm_hz) * 1e3
            pipe_ms = rec["fp_pipe_active_pct"] / 100.0 * rec["ncu_ms_per_step"]
            compute = {"issue_floor_ms": issue_ms, "issue_frac": issue_ms / (per_step * 1e3),
                       "fp_pipe": rec["fp_pipe"], "fp_pipe_floor_ms": pipe_ms,
                       "fp_pipe_frac": pipe_ms / (per_step * 1e3),
                       "warp_inst_per_step": rec["warp_inst_per_step"],
                       "ipc": rec.get("ipc"), "launches_per_step": launches_per_step,
                       "source": rec.get("source")}
    achieved = local_cells * bytes_per_cell / per_step / 1e9 if world == 1 else \
        max(shares) * m * l * bytes_per_cell / per_step / 1e9

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": wall_max / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64" if fp64 else "f32", "data": "synthetic (seeded BASELINE recipe, device-generated)",
        "config": {"workload": desc, "grid": [n, m, l], "iord": iord, "nonos": nonos,
                   "boundary": "periodic", "shares": shares,
                   "parallelism": f"slab{world}" + (f" {halo}-halo" if world > 1 else ""),
                   "ranks": ranks,
                   "l2": f"inputs larger than L2 (5 fields x {cells * elem >> 20} MiB)",
                   # halo planes each GPU sends per step, per direction
                   "halo_bytes_per_gpu_per_step": (2 * mpdata.step_radius(opts) * m * l * elem
                                                   if world > 1 else 0)},
        "e2e": {"value": e2e_value, "unit": UNIT,
                "h2d_bytes_per_step": local_cells * elem, "d2h_bytes_per_step": local_cells * elem,
                "path": "imb_team_step_host (pinned host x in, step incl. halo exchange, x out)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "traffic_note": "bytes per launch: ncu dram__bytes_read+write of the step "
                                     "kernel (profiles/traffic.json); compare with "
                                     "algorithmic_bytes_per_launch; null if not captured",
                     "algorithmic_bytes_per_launch": local_cells * bytes_per_cell,
                     "kernel": ("k_fused (one launch per step; CUDA events on the team compute "
                                "stream)" if iord == 2 and l in (32, 64, 128) else
                                "staged step kernels (per-step compute window)"),
                     "algorithmic_bytes_per_cell": bytes_per_cell, "peak_source": peak_src,
                     "compute": compute},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "compute_ms_per_step": per_step * 1e3,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        planes = min(n, 128)
        v, secs, nst = cpu_port_gcells(n, m, l, iord, nonos, fp64, recipe, planes, 2, threads,
                                       budget_s=15.0)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
                                "sample": f"{nst} steps on a {planes}x{m}x{l} periodic slab of the "
                                          f"{n}x{m}x{l} grid ({secs:.1f} s)"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    team.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
