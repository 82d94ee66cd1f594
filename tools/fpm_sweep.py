#!/usr/bin/env python3
"""FPM loop on the GPU (BASELINE configs 3 and 5).

1. Speed-function sweep: time MPDATA steps on slabs of n x m x l for a list of
   slab thicknesses n (the FPM workload unit x is one i-plane, a "frame" of m*l
   cells), repeating each point until the 95% Student-t CI half-width is below
   `--ci` of the mean (stats via the product's t-quantile). The slab runs as a
   periodic team, so its per-step time includes its own halo exchange.
2. Writes the speed function as the SPEC CSV.
3. Partitions `--total` planes over `--p` GPUs with Algorithm 1
   (partition_paired) and with partition_general, predicts even vs FPM
   makespans, and validates by timing the distinct shares of both splits
   (the per-step makespan of p GPUs stepping in lockstep is the slowest
   GPU's step time; each share is measured on its own here, as on one GPU).

    python tools/fpm_sweep.py --config c3 --out profiles/r01_fpm_c3
    python tools/fpm_sweep.py --config c5 --p 8 --out profiles/r01_fpm_c5
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1507_01265_b200 import fpm, mpdata  # noqa: E402


def measure(n, m, l, opts, steps, ci_target, min_reps, max_reps, warm=2):
    with mpdata.Team(n, m, l, opts) as t:
        t.init_recipe(mpdata.RECIPE_ROTCUBE, 42)
        t.run(warm)
        times = []
        while True:
            _, wall = t.run(steps)
            times.append(wall / steps)
            if len(times) >= min_reps:
                s = fpm.summarize(times)
                if s.ci_halfwidth <= ci_target * s.mean or len(times) >= max_reps:
                    return s, len(times)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3", choices=["c3", "c5"])
    ap.add_argument("--fp32", action="store_true")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--ci", type=float, default=0.02)
    ap.add_argument("--p", type=int, default=8)
    ap.add_argument("--gran", type=int, default=8)
    ap.add_argument("--out", default="gpurun_out/fpm")
    ap.add_argument("--validate-steps", type=int, default=100)
    ap.add_argument("--table-max", type=int, default=48, help="largest Delta of the table")
    a = ap.parse_args()
    if a.config == "c3":  # n x 512 x 128 fp64 nonos IORD2, n in powers of two
        m, l, total = 512, 128, 1024
        opts = mpdata.Options(2, True, not a.fp32)
        xs = [8, 16, 32, 64, 128, 256, 512, 1024, 2048]
        base = total // a.p
        dense = list(range(max(a.gran, base - 64), base + 64 + 1, a.gran))
        xs = sorted(set(xs) | set(dense))
    else:  # config 5: slabs of n x 1024 x 128, IORD3 nonos, around n/p of 2048
        m, l, total = 1024, 128, 2048
        opts = mpdata.Options(3, True, not a.fp32)
        base = total // a.p
        xs = sorted(set([64, 128, 512, 1024]) |
                    set(range(base - 128, base + 128 + 1, a.gran)))
    R = mpdata.step_radius(opts)
    xs = [x for x in xs if x >= R]
    samples, rows = [], []
    for x in xs:
        s, reps = measure(x, m, l, opts, a.steps, a.ci, 3, 12)
        speed = x * m * l / s.mean  # cell-updates per second
        ci = speed * s.ci_halfwidth / s.mean
        samples.append(fpm.SpeedSample(x, speed, ci, reps))
        rows.append(dict(x=x, step_s=s.mean, ci_s=s.ci_halfwidth, reps=reps, gcells=speed / 1e9))
        print(f"x={x:5d} step {s.mean*1e3:8.3f} ms +- {s.ci_halfwidth*1e3:.3f}  "
              f"{speed/1e9:7.2f} Gcell/s", flush=True)
    label = f"{a.config} {'fp32' if a.fp32 else 'fp64'} iord{opts.iord} nonos m={m} l={l} cell-updates/s"
    f = fpm.SpeedFunction(m * l, a.gran, tuple(samples), label)
    out = Path(a.out)
    out.parent.mkdir(parents=True, exist_ok=True)
    out.with_suffix(".csv").write_text(fpm.write_csv(f))

    report = {"config": a.config, "grid_total_planes": total, "m": m, "l": l, "p": a.p,
              "opts": dict(iord=opts.iord, nonos=opts.nonos, fp64=opts.fp64), "sweep": rows}
    cond = fpm.check_condition(f)
    report["condition_satisfied"] = cond.satisfied
    report["max_gain_pair"] = cond.max_gain_pair
    report["shape"] = fpm.classify_shape(f)[0] if len(samples) >= 3 else None
    even = [total // a.p] * a.p
    pe = fpm.predict_makespan(f, even)
    report["even"] = dict(shares=even, predicted_makespan_s=pe.makespan)
    try:
        pp = fpm.partition_paired(fpm.PartitionProblem(total, a.p, f))
        report["paired"] = dict(shares=pp.shares, offset=pp.offset, predicted_makespan_s=pp.makespan)
    except mpdata._lib.ImbError as e:
        report["paired"] = dict(error=str(e))
    pg = fpm.partition_general(fpm.PartitionProblem(total, a.p, f))
    report["general"] = dict(shares=pg.shares, predicted_makespan_s=pg.makespan)
    imp = fpm.improvement_search(f, total // a.p) if (total // a.p) in xs else None
    report["improvement"] = None if imp is None else dict(pair=imp.violating_pair,
                                                          delta=imp.delta, gain_s=imp.gain_s)

    # Validation: measured per-step makespan = slowest share of each split.
    def measured_makespan(shares):
        per = {}
        for s_ in sorted(set(shares)):
            st, _ = measure(s_, m, l, opts, a.validate_steps, a.ci, 3, 8)
            per[s_] = st.mean
        return max(per[s_] for s_ in shares), per

    me, per_e = measured_makespan(even)
    report["even"]["measured_step_s"] = me
    for key in ("paired", "general"):
        if "shares" in report[key]:
            mk, per = measured_makespan(report[key]["shares"])
            report[key]["measured_step_s"] = mk
            report[key]["per_share_step_s"] = {str(k): v for k, v in per.items()}
            report[key]["measured_speedup_vs_even"] = me / mk
            report[key]["predicted_speedup_vs_even"] = (
                pe.makespan / report[key]["predicted_makespan_s"])
    # Validation table in the paper's Table 1-3 format (PAPER.md:368-472,
    # SPEC.md:369-377): symmetric offsets Delta around n/p (even processors at
    # n/p - Delta, odd at n/p + Delta), theoretical (model) vs experimental
    # (measured) step makespan, per-share times, speedup vs Delta = 0, and the
    # model's prediction error.
    table = []
    cache = dict(per_e)
    for d in range(0, a.table_max + 1, a.gran):
        lo_, hi_ = base - d, base + d
        if lo_ < min(xs) or hi_ > max(xs):
            break
        for s_ in (lo_, hi_):
            if s_ not in cache:
                cache[s_] = measure(s_, m, l, opts, a.validate_steps, a.ci, 3, 8)[0].mean
        theo = max(fpm.eval_time(f, lo_), fpm.eval_time(f, hi_))
        exp_ = max(cache[lo_], cache[hi_])
        table.append(dict(delta=d, shares=[lo_, hi_], t_theory_s=theo, t_exp_s=exp_,
                          t_even_share_s=cache[lo_], t_odd_share_s=cache[hi_],
                          speedup_theory=pe.makespan / theo, speedup_exp=me / exp_,
                          prediction_error=(theo - exp_) / exp_))
    report["validation_table"] = table
    out.with_suffix(".json").write_text(json.dumps(report, indent=1) + "\n")
    print(json.dumps({k: report[k] for k in ("even", "paired", "general", "condition_satisfied",
                                             "shape")}, indent=1))
    print(f"{'Delta':>6} {'shares':>12} {'t_theory[ms]':>13} {'t_exp[ms]':>10} "
          f"{'speedup':>8} {'err':>7}")
    for row in table:
        print(f"{row['delta']:6d} {str(row['shares']):>12} {row['t_theory_s']*1e3:13.4f} "
              f"{row['t_exp_s']*1e3:10.4f} {row['speedup_exp']:8.4f} "
              f"{100*row['prediction_error']:6.2f}%")


if __name__ == "__main__":
    main()
