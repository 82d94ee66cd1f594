"""Command-line front end: measure, check, partition, predict, validate, report.

Mirrors the reference CLI contract: the same
subcommands, global flags ``--seed --out-dir --json``, ``start:stop:step``
ranges (stop included when aligned) and exit codes (errors.hpp:8-9,
SPEC.md:458): 0 success, 1 runtime error or infeasible problem, 2 usage or
parse error. ``check``/``partition``/``predict`` run the C++ model and
partitioner through the C-ABI (no GPU needed); ``measure`` and ``validate``
time the B200 MPDATA step (one team = one GPU).

    python -m paper_1507_01265_b200.cli measure --x 8:64:8 --m 512 --l 128 --out-dir out
    python -m paper_1507_01265_b200.cli check out/speed_avg.csv
    python -m paper_1507_01265_b200.cli partition out/speed_avg.csv --total 1024 --p 8 --paired
    python -m paper_1507_01265_b200.cli validate out/speed_avg.csv --total 1024 --p 8 --offsets 0,8,16
"""
from __future__ import annotations

import argparse
import datetime
import hashlib
import json
import os
import platform
import sys
import threading
from pathlib import Path

from . import __version__, _lib, fpm

EXIT_OK, EXIT_RUNTIME, EXIT_USAGE = 0, 1, 2


class UsageError(Exception):
    pass


def parse_range(text: str) -> list:
    """``start:stop:step`` -> [start, start+step, ...] including stop when aligned."""
    try:
        a, b, c = (int(v) for v in text.split(":"))
    except ValueError:
        raise UsageError(f"range '{text}' is not start:stop:step") from None
    if c <= 0 or a <= 0 or b < a:
        raise UsageError(f"range '{text}' must have 0 < start <= stop and step > 0")
    return list(range(a, b + 1, c))


def parse_list(text: str) -> list:
    try:
        return [int(v) for v in text.split(",") if v.strip()]
    except ValueError:
        raise UsageError(f"'{text}' is not a comma-separated integer list") from None


def manifest(args, inputs=()) -> dict:
    """RunManifest: command, arguments, input hashes, version, machine."""
    hashes = {}
    for p in inputs:
        hashes[str(p)] = hashlib.sha256(Path(p).read_bytes()).hexdigest()
    return {
        "command": args.cmd, "args": {k: v for k, v in vars(args).items() if k != "func"},
        "inputs_sha256": hashes, "tool_version": __version__,
        "timestamp": datetime.datetime.now(datetime.timezone.utc).isoformat(),
        "machine": {"host": platform.node(), "cpus": os.cpu_count(),
                    "thread_cap": os.environ.get("IMBALANCE_THREAD_CAP"),
                    "python": platform.python_version()},
    }


def emit(args, obj: dict, text: str):
    print(json.dumps(obj, indent=1) if args.json else text)


def write_out(args, name: str, content: str) -> Path:
    out = Path(args.out_dir)
    out.mkdir(parents=True, exist_ok=True)
    p = out / name
    p.write_text(content)
    return p


def load_model(path: str) -> fpm.SpeedFunction:
    try:
        text = Path(path).read_text()
    except OSError as e:
        raise UsageError(f"cannot read model file: {e}") from None
    return fpm.read_csv(text)


# ---- check ------------------------------------------------------------------
def cmd_check(args) -> int:
    f = load_model(args.model)
    c = fpm.check_condition(f)
    shape, peak = fpm.classify_shape(f) if len(f.samples) >= 3 else (None, None)
    obj = {"satisfied": c.satisfied, "violations": c.violations,
           "max_gain_pair": c.max_gain_pair, "shape": shape, "peak_x": peak}
    if c.satisfied:
        text = "condition satisfied; balancing optimal"
    else:
        text = (f"condition violated at {len(c.violations)} pair(s): {c.violations}\n"
                f"best imbalancing opportunity: {c.max_gain_pair}")
    if shape is not None:
        text += f"\nshape: {shape}" + (f" (peak at x={peak})" if peak is not None else "")
    emit(args, obj, text)
    return EXIT_OK


# ---- partition / predict ----------------------------------------------------
def balanced_makespan(f, total, p):
    if p < 1 or total % p:
        return None
    try:
        return fpm.predict_makespan(f, [total // p] * p).makespan
    except _lib.ImbError:
        return None


def cmd_partition(args) -> int:
    f = load_model(args.model)
    pr = fpm.PartitionProblem(args.total, args.p, f, args.allow_idle)
    algo = "oracle" if args.oracle else "general" if args.general else "paired"
    if algo == "paired":
        r = fpm.partition_paired(pr)
    elif algo == "general":
        r = fpm.partition_general(pr)
    else:
        r = fpm.brute_force_oracle(pr, args.cap)
    bal = balanced_makespan(f, args.total, args.p)
    obj = {"algorithm": algo, "shares": r.shares, "per_time": r.per_time,
           "makespan": r.makespan, "offset": r.offset, "balanced_makespan": bal,
           "speedup_vs_balanced": (bal / r.makespan) if bal and r.makespan > 0 else None}
    text = (f"{algo}: shares {r.shares} makespan {r.makespan:.6f} s"
            + (f" offset {r.offset}" if r.offset is not None else "")
            + (f"\nbalanced makespan {bal:.6f} s, speedup {bal / r.makespan:.3f}"
               if obj["speedup_vs_balanced"] else ""))
    emit(args, obj, text)
    return EXIT_OK


def cmd_predict(args) -> int:
    f = load_model(args.model)
    shares = parse_list(args.shares)
    r = fpm.predict_makespan(f, shares)
    obj = {"shares": shares, "per_time": r.per_time, "makespan": r.makespan}
    emit(args, obj, f"per-team {['%.6f' % t for t in r.per_time]} makespan {r.makespan:.6f} s")
    return EXIT_OK


# ---- measurement (bench module) ----------------------------
def _opts(args):
    from . import mpdata
    return mpdata.Options(args.iord, args.nonos, not args.fp32)


def measure_simultaneous(ni, m, l, opts, devices, steps, ci, min_reps, max_reps, warmup, seed):
    """One team per device on the same ni x m x l periodic slab, every trial
    started from a shared barrier; each team's time is its own device time for
    `steps` steps (barrier waits excluded). Repeats until every
    team's 95% CI half-width <= ci * mean, or max_reps. -> ([Summary], reps, converged)"""
    from . import mpdata
    nt = len(devices)
    barrier = threading.Barrier(nt)
    times = [[] for _ in range(nt)]
    stop = threading.Event()
    errors = []

    def team(q):
        try:
            with mpdata.Team(ni, m, l, opts, device=devices[q]) as t:
                t.init_recipe(mpdata.RECIPE_ROTCUBE, seed)
                t.run(warmup)
                while True:
                    barrier.wait()
                    if stop.is_set():
                        return
                    _, wall = t.run(steps)
                    times[q].append(wall / steps)
                    barrier.wait()
                    if q == 0:
                        done = len(times[0]) >= max_reps
                        if len(times[0]) >= min_reps and not done:
                            sums = [fpm.summarize(ts) for ts in times]
                            done = all(s.ci_halfwidth <= ci * s.mean for s in sums)
                        if done:
                            stop.set()
                    barrier.wait()
                    if stop.is_set():
                        return
        except BaseException as e:  # surface the first failure, release the others
            errors.append(e)
            stop.set()
            barrier.abort()

    threads = [threading.Thread(target=team, args=(q,)) for q in range(nt)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    if errors:
        raise next((e for e in errors if not isinstance(e, threading.BrokenBarrierError)), errors[0])
    sums = [fpm.summarize(ts) for ts in times]
    conv = all(s.ci_halfwidth <= ci * s.mean for s in sums)
    return sums, len(times[0]), conv


def measure_ring(ni, m, l, opts, devices, steps, ci, min_reps, max_reps, warmup, seed):
    """The production halo path: the listed devices form one ring of slabs of
    ni planes each (an in-process group, the decomposition of a
    len(devices)*ni-plane grid), so every team's time includes its halo push
    into its neighbours (over NVLink between GPUs) and the step
    synchronisation. Each team's time is its own device compute time per step
    (the group's event windows). A device id may repeat: p
    slabs sharing one GPU is the labelled single-GPU stand-in.
    -> ([Summary], reps, converged)"""
    from . import mpdata
    nt = len(devices)
    times = [[] for _ in range(nt)]
    g = mpdata.Group(ni * nt, m, l, [ni] * nt, devices=devices, opts=opts)
    try:
        g.init_recipe(mpdata.RECIPE_ROTCUBE, seed)
        if warmup:
            g.run(warmup)
        while True:
            per, _ = g.run(steps)
            for q in range(nt):
                times[q].append(per[q] / steps)
            n = len(times[0])
            if n >= max_reps:
                break
            if n >= min_reps:
                sums = [fpm.summarize(ts) for ts in times]
                if all(s.ci_halfwidth <= ci * s.mean for s in sums):
                    break
    finally:
        g.close()
    sums = [fpm.summarize(ts) for ts in times]
    conv = all(s.ci_halfwidth <= ci * s.mean for s in sums)
    return sums, len(times[0]), conv


def halo_label(args, devices):
    if args.halo == "self":
        return "halo=self (periodic single slab per GPU)"
    shared = len(set(devices)) < len(devices)
    return (f"halo=ring p={len(devices)} devices={','.join(map(str, devices))}"
            + (" (slabs share a GPU: stand-in)" if shared else ""))


def cmd_measure(args) -> int:
    xs = parse_range(args.x)
    gran = int(args.x.split(":")[2])
    ms = parse_range(args.m_range) if args.m_range else [args.m]
    devices = parse_list(args.devices)
    if not devices:
        raise UsageError("--devices is empty")
    cap = os.environ.get("IMBALANCE_THREAD_CAP")
    if cap and len(devices) > int(cap):
        raise UsageError(f"{len(devices)} teams exceed IMBALANCE_THREAD_CAP={cap}")
    opts = _opts(args)
    from . import mpdata
    R = mpdata.step_radius(opts)
    if xs[0] < R:
        raise UsageError(f"slab thickness {xs[0]} is below the step radius {R}")
    l = args.l
    if args.halo == "self" and len(set(devices)) < len(devices):
        raise UsageError("--halo self needs distinct --devices (repeat a device only with --halo ring)")
    def tname(q):  # gpu<id> for distinct devices, team<q> when slabs share a GPU
        return f"gpu{devices[q]}" if len(set(devices)) == len(devices) else f"team{q}"

    per = {d: {} for d in range(len(devices))}  # team -> {(m, x): SpeedSample}
    unconverged = []
    for m in ms:
        for x in xs:
            how = measure_ring if args.halo == "ring" else measure_simultaneous
            sums, reps, conv = how(x, m, l, opts, devices, args.steps, args.ci, args.min_reps,
                                   args.max_reps, args.warmup, args.seed)
            if not conv:
                unconverged.append([m, x])
            for q, s in enumerate(sums):
                speed = x * m * l / s.mean  # cell-updates per second
                per[q][(m, x)] = fpm.SpeedSample(x, speed, speed * s.ci_halfwidth / s.mean, reps)
            if not args.json:
                print(f"m={m} x={x}: " + "  ".join(
                    f"{tname(q)} {x * m * l / s.mean / 1e9:.3f} Gcell/s" for q, s in enumerate(sums)),
                    flush=True)
    prec = "fp32" if args.fp32 else "fp64"
    what = (f"iord{opts.iord}{' nonos' if opts.nonos else ''} {prec} l={l} cell-updates/s per step "
            f"{halo_label(args, devices)}")
    files = []

    def one_d(q, m, label):
        return fpm.SpeedFunction(m * l, gran, tuple(per[q][(m, x)] for x in xs), label)

    if len(ms) == 1:  # speed functions: x = slab planes, unit = one m x l plane
        m = ms[0]
        fs = [one_d(q, m, f"{tname(q)} m={m} {what}") for q in range(len(devices))]
        for q, f in enumerate(fs):
            files.append(write_out(args, f"speed_{tname(q)}.csv", fpm.write_csv(f)))
        avg = fpm.average(fs)
        files.append(write_out(args, "speed_avg.csv", fpm.write_csv(avg)))
        files.append(write_out(args, "speed_avg.dat", "".join(
            f"{s.x} {s.speed:.17g}\n" for s in avg.samples)))
    else:  # surface keyed by (n = rows m, m = slab planes x); unit = one row of l cells
        for q in range(len(devices)):
            smp = [per[q][(m, x)] for m in ms for x in xs]
            files.append(write_out(args, f"surface_{tname(q)}.csv", fpm.write_surface_csv(
                fpm.SpeedSurface(l, gran, tuple(ms), tuple(xs), tuple(smp), f"{tname(q)} {what}"))))
        avg_smp = []
        for m in ms:
            fs = [fpm.SpeedFunction(l, gran, tuple(per[q][(m, x)] for x in xs))
                  for q in range(len(devices))]
            avg_smp += list(fpm.average(fs).samples)
        files.append(write_out(args, "surface_avg.csv", fpm.write_surface_csv(
            fpm.SpeedSurface(l, gran, tuple(ms), tuple(xs), tuple(avg_smp),
                             f"avg(gpu{','.join(map(str, devices))}) {what}"))))
    man = manifest(args)
    man["outputs"] = [str(p) for p in files]
    man["unconverged"] = unconverged
    man["halo"] = halo_label(args, devices)
    files.append(write_out(args, "measure_manifest.json", json.dumps(man, indent=1) + "\n"))
    emit(args, man, "wrote " + ", ".join(str(p) for p in files)
         + (f"\nunconverged (m, x): {unconverged}" if unconverged else ""))
    return EXIT_OK


# ---- validate (Tables 1-3) ----------------------------------
def run_decomposed(total, m, l, shares, devices, opts, steps, warmup, seed):
    """The real decomposed workload: one slab per device, halos pushed every
    step, lockstep. -> (per-team compute seconds per step, wall per step)."""
    from . import mpdata
    g = mpdata.Group(total, m, l, shares, devices=devices, opts=opts)
    try:
        g.init_recipe(mpdata.RECIPE_ROTCUBE, seed)
        g.run(warmup)
        per, wall = g.run(steps)
    finally:
        g.close()
    return [t / steps for t in per], wall / steps


def cmd_validate(args) -> int:
    f = load_model(args.model)
    offsets = parse_list(args.offsets)
    if not offsets or offsets[0] != 0:
        raise UsageError("--offsets must start with 0 (the balanced baseline row)")
    p, total = args.p, args.total
    if total % p:
        raise UsageError("--total must divide evenly over --p")
    base = total // p
    devices = parse_list(args.devices)
    m = f.unit_cells // args.l if args.m is None else args.m
    if m * args.l != f.unit_cells:
        raise UsageError(f"model unit_cells {f.unit_cells} != m*l = {m * args.l}")
    opts = _opts(args)
    lockstep = len(devices) >= p
    rows, teams = [], []
    for d in offsets:
        lo, hi = base - d, base + d
        if lo < f.min_x or hi > f.max_x:
            raise _lib.RangeError(f"offset {d} leaves the model range [{f.min_x}, {f.max_x}]")
        shares = [lo if q % 2 == 0 else hi for q in range(p)]
        theo = max(fpm.eval_time(f, lo), fpm.eval_time(f, hi))
        if lockstep:  # p GPUs stepping the real decomposition
            per, wall = run_decomposed(total, m, args.l, shares, devices[:p], opts, args.steps,
                                       args.warmup, args.seed)
            if wall < max(per) * (1 - 1e-9):
                raise _lib.ContractError("total time below the slowest team's time")
            exp_ = wall
        else:  # fewer GPUs than teams: time each distinct share on its own
            per_share = {}
            for s in sorted(set(shares)):
                sums, _, _ = measure_simultaneous(s, m, args.l, opts, devices[:1], args.steps,
                                                  args.ci, 3, args.max_reps, args.warmup, args.seed)
                per_share[s] = sums[0].mean
            per = [per_share[s] for s in shares]
            exp_ = max(per)
        rows.append({"offset": d, "shares": [lo, hi], "t_theory_s": theo, "t_exp_s": exp_})
        teams += [{"offset": d, "team": q, "share": shares[q], "t_s": per[q]} for q in range(p)]
    for r in rows:
        r["speedup"] = rows[0]["t_exp_s"] / r["t_exp_s"]  # Table 1: exp(0) / exp(delta)
        r["prediction_error"] = (r["t_theory_s"] - r["t_exp_s"]) / r["t_exp_s"]
    t1 = "offset,t_theory_s,t_exp_s,speedup,prediction_error\n" + "".join(
        f"{r['offset']},{r['t_theory_s']:.9g},{r['t_exp_s']:.9g},{r['speedup']:.6f},"
        f"{r['prediction_error']:.6f}\n" for r in rows)
    t2 = "offset,team,share,t_s\n" + "".join(
        f"{t['offset']},{t['team']},{t['share']},{t['t_s']:.9g}\n" for t in teams)
    files = [write_out(args, "table1.csv", t1), write_out(args, "table2.csv", t2),
             write_out(args, "table1.dat", "".join(f"{r['offset']} {r['t_exp_s']:.9g}\n"
                                                    for r in rows))]
    man = manifest(args, [args.model])
    mode = "per-share timing on one GPU"
    if lockstep:
        mode = ("lockstep decomposition" if len(set(devices[:p])) == p else
                "lockstep decomposition (slabs share a GPU: stand-in)")
    man.update(mode=mode, halo="ring (kernel halo push between slabs)" if lockstep else "self",
               table1=rows, table2=teams, outputs=[str(q) for q in files])
    files.append(write_out(args, "validate_manifest.json", json.dumps(man, indent=1) + "\n"))
    text = f"{'offset':>6} {'t_theory':>10} {'t_exp':>10} {'speedup':>8} {'err':>7}\n" + "".join(
        f"{r['offset']:6d} {r['t_theory_s']:10.6f} {r['t_exp_s']:10.6f} {r['speedup']:8.4f} "
        f"{100 * r['prediction_error']:6.2f}%\n" for r in rows)
    emit(args, man, text.rstrip())
    return EXIT_OK


# ---- report -------------------------------------------------------------------
def cmd_report(args) -> int:
    out = Path(args.out_dir)
    found = sorted(out.glob("*_manifest.json"))
    if not found:
        raise UsageError(f"no *_manifest.json under {out}")
    objs = [json.loads(p.read_text()) for p in found]
    lines = []
    for p, o in zip(found, objs):
        lines.append(f"## {o['command']} ({p.name}, {o['timestamp']})")
        for k in ("outputs", "unconverged", "mode"):
            if k in o:
                lines.append(f"- {k}: {o[k]}")
        for r in o.get("table1", []):
            lines.append(f"  - offset {r['offset']}: theory {r['t_theory_s']:.6f} s, "
                         f"exp {r['t_exp_s']:.6f} s, speedup {r['speedup']:.4f}")
    emit(args, {"manifests": objs}, "\n".join(lines))
    return EXIT_OK


# ---- argument parsing ----------------------------------------------------------
def build_parser() -> argparse.ArgumentParser:
    glob = argparse.ArgumentParser(add_help=False)
    glob.add_argument("--seed", type=int, default=42)
    glob.add_argument("--out-dir", default="imbalance_out")
    glob.add_argument("--json", action="store_true")
    work = argparse.ArgumentParser(add_help=False)
    work.add_argument("--l", type=int, default=128)
    work.add_argument("--iord", type=int, default=2)
    work.add_argument("--nonos", action=argparse.BooleanOptionalAction, default=True)
    work.add_argument("--fp32", action="store_true")
    work.add_argument("--devices", default="0", help="comma-separated GPU ids, one team each")
    work.add_argument("--steps", type=int, default=20, help="time steps per timing trial")
    work.add_argument("--warmup", type=int, default=1)
    work.add_argument("--ci", type=float, default=0.05, help="target CI half-width / mean")
    work.add_argument("--max-reps", type=int, default=20)
    work.add_argument("--halo", choices=["self", "ring"], default="self",
                      help="measure: 'self' = one periodic slab per GPU; 'ring' = the listed "
                           "devices form one slab ring with the production halo push (a "
                           "device may repeat: slabs sharing a GPU, a labelled stand-in)")

    ap = argparse.ArgumentParser(prog="imbalance", description=__doc__.split("\n")[0])
    sub = ap.add_subparsers(dest="cmd", required=True)
    c = sub.add_parser("check", parents=[glob], help="condition (Eq. 1) and shape of a model")
    c.add_argument("model")
    c.set_defaults(func=cmd_check)
    c = sub.add_parser("partition", parents=[glob], help="FPM partition of total over p")
    c.add_argument("model")
    c.add_argument("--total", type=int, required=True)
    c.add_argument("--p", type=int, required=True)
    g = c.add_mutually_exclusive_group()
    g.add_argument("--paired", action="store_true", help="Algorithm 1 (default)")
    g.add_argument("--general", action="store_true", help="exact DP, any p")
    g.add_argument("--oracle", action="store_true", help="brute force (tests)")
    c.add_argument("--allow-idle", action="store_true")
    c.add_argument("--cap", type=int, default=fpm.K_DEFAULT_ORACLE_CAP)
    c.set_defaults(func=cmd_partition)
    c = sub.add_parser("predict", parents=[glob], help="per-team times and makespan of shares")
    c.add_argument("model")
    c.add_argument("--shares", required=True)
    c.set_defaults(func=cmd_predict)
    c = sub.add_parser("measure", parents=[glob, work], help="build speed functions on GPUs")
    c.add_argument("--x", required=True, help="slab thicknesses start:stop:step (i-planes)")
    c.add_argument("--m", type=int, default=512, help="rows per plane")
    c.add_argument("--m-range", default=None, help="rows start:stop:step -> 2-D surface")
    c.add_argument("--min-reps", type=int, default=3)
    c.set_defaults(func=cmd_measure)
    c = sub.add_parser("validate", parents=[glob, work], help="Table 1-3 validation runs")
    c.add_argument("model")
    c.add_argument("--total", type=int, required=True)
    c.add_argument("--p", type=int, required=True)
    c.add_argument("--offsets", default="0")
    c.add_argument("--m", type=int, default=None, help="rows (default: unit_cells / l)")
    c.set_defaults(func=cmd_validate)
    c = sub.add_parser("report", parents=[glob], help="summarise the manifests in --out-dir")
    c.set_defaults(func=cmd_report)
    return ap


def main(argv=None) -> int:
    ap = build_parser()
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:  # argparse: usage errors exit 2, --help exits 0
        return int(e.code or 0)
    try:
        if getattr(args, "min_reps", 3) < 3:
            raise UsageError("--min-reps must be >= 3")
        return args.func(args)
    except (UsageError, _lib.ParseError, _lib.ContractError) as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_USAGE
    except (_lib.ImbError, RuntimeError, OSError) as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_RUNTIME


if __name__ == "__main__":
    sys.exit(main())
