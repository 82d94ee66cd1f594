"""Speed-function model, stats and CSV — product vs the compiled reference
(oracle/_ref) and the SPEC known-answer examples. CPU only."""
import math
import random

import pytest

from paper_1507_01265_b200 import _lib, fpm
from oracle import oracle as O

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def test_eval_known_answers():
    # SPEC.md:61-73 / SURVEY Appendix B.
    f = fpm.SpeedFunction(15360, 8, ((112, 1436742.0), (128, 1418579.0)))
    assert fpm.eval_speed(f, 112) == 1436742.0
    assert fpm.eval_speed(f, 128) == 1418579.0
    assert fpm.eval_speed(f, 120) == 1427660.5
    assert abs(fpm.eval_time(f, 128) - 1.385950) < 1e-6
    assert abs(fpm.eval_time(f, 112) - 1.197376) < 1e-6
    assert fpm.eval_time(f, 0) == 0.0
    with pytest.raises(_lib.RangeError):
        fpm.eval_speed(f, 130)
    with pytest.raises(_lib.RangeError):
        fpm.eval_time(f, 129)
    with pytest.raises(_lib.RangeError):
        fpm.eval_time(f, 100)  # below range: RangeError from eval_speed
    with pytest.raises(_lib.DomainError):
        fpm.eval_speed(f, 0)


def test_constructor_contracts():
    for bad in [((0, 1.0),), ((1, 0.0),), ((2, 1.0), (2, 1.0)), ((1, 1.0), (2, 1.0))]:
        with pytest.raises(_lib.ContractError):
            fpm.SpeedFunction(1, 2 if bad == ((1, 1.0), (2, 1.0)) else 1, bad)
    with pytest.raises(_lib.ContractError):
        fpm.SpeedFunction(0, 1, ((1, 1.0),))
    with pytest.raises(_lib.ContractError):
        fpm.SpeedFunction(1, 1, ())


@needs_ref
def test_eval_bit_parity_random():
    rng = random.Random(3)
    for _ in range(200):
        g = rng.choice([1, 2, 4])
        xs = sorted({rng.randint(1, 40) * g for _ in range(rng.randint(1, 8))})
        sm = [(x, rng.uniform(1e3, 1e9)) for x in xs]
        unit = rng.choice([1, 65536, 131072])
        f = fpm.SpeedFunction(unit, g, tuple(sm))
        for _ in range(10):
            x = rng.uniform(0, xs[-1] + 5)
            for kind, fn in (("speed", fpm.eval_speed), ("time", fpm.eval_time)):
                st, want = O.ref_eval(kind, unit, g, sm, x)
                try:
                    got, gst = fn(f, x), 0
                except _lib.ImbError as e:
                    got, gst = None, e.code
                assert (gst, got) == (st, want)


@needs_ref
def test_condition_shape_improvement_average_parity():
    rng = random.Random(4)
    for _ in range(300):
        xs = list(range(2, 2 + 2 * rng.randint(3, 9), 2))
        sm = [(x, float(rng.randint(1, 30))) for x in xs]
        f = fpm.SpeedFunction(5, 2, tuple(sm))
        st, rep = O.ref_check_condition(5, 2, sm)
        c = fpm.check_condition(f)
        assert (c.satisfied, c.violations, c.max_gain_pair) == rep
        st, cls = O.ref_classify(5, 2, sm)
        mine = fpm.classify_shape(f)
        assert (fpm.SHAPES.index(mine[0]), mine[1]) == cls
        bal = xs[len(xs) // 2]
        st, imp = O.ref_improvement(5, 2, sm, bal)
        got = fpm.improvement_search(f, bal)
        assert (None if got is None else (got.violating_pair, got.delta, got.gain_s)) == imp
        f2 = [(x, s * rng.uniform(0.5, 2)) for x, s in sm]
        st, avg = O.ref_average(5, 2, [sm, f2])
        a = fpm.average([f, fpm.SpeedFunction(5, 2, tuple(f2))])
        assert [(s.x, s.speed, s.ci_halfwidth, s.repetitions) for s in a.samples] == avg


def test_condition_and_shape_spec_examples():
    f = fpm.SpeedFunction(1, 1, ((120, 1240377.0), (128, 1418579.0)))
    c = fpm.check_condition(f)
    assert not c.satisfied and c.violations == [(120, 128)] and c.max_gain_pair == (120, 128)
    assert fpm.check_condition(fpm.SpeedFunction(1, 10, ((10, 100.0), (20, 90.0), (30, 80.0)))).satisfied
    assert fpm.classify_shape(fpm.SpeedFunction(1, 10, ((10, 100.0), (20, 90.0), (30, 80.0))))[0] == \
        "monotonically-decreasing"
    assert fpm.classify_shape(fpm.SpeedFunction(
        1, 10, ((10, 100.0), (20, 180.0), (30, 200.0), (40, 150.0)))) == \
        ("increasing-concave-then-decreasing", 30)
    assert fpm.classify_shape(fpm.SpeedFunction(
        1, 10, ((10, 100.0), (20, 300.0), (30, 100.0), (40, 300.0))))[0] == "other"
    with pytest.raises(_lib.InsufficientDataError):
        fpm.classify_shape(fpm.SpeedFunction(1, 1, ((1, 1.0), (2, 1.0))))


def test_improvement_search_paper():
    f = fpm.SpeedFunction(15360, 8, ((112, 1436742.0), (120, 1240377.0), (128, 1418579.0)))
    imp = fpm.improvement_search(f, 120)
    assert imp.delta == 8 and imp.violating_pair == (120, 128)
    assert abs(imp.gain_s - 0.100050) < 1e-6
    with pytest.raises(_lib.DomainError):
        fpm.improvement_search(f, 121)


def test_average_contracts():
    a = fpm.SpeedFunction(1, 1, ((10, 100.0),), "a")
    b = fpm.SpeedFunction(1, 1, ((10, 200.0),), "b")
    m = fpm.average([a, b])
    assert m.samples[0].speed == 150.0 and m.label == "avg(a,b)" and m.samples[0].repetitions == 2
    with pytest.raises(_lib.IncompatibleModelError):
        fpm.average([a, fpm.SpeedFunction(2, 1, ((10, 1.0),))])
    with pytest.raises(_lib.IncompatibleModelError):
        fpm.average([a, fpm.SpeedFunction(1, 1, ((11, 1.0),))])


def test_csv_round_trip_bit_exact():
    rng = random.Random(8)
    f = fpm.SpeedFunction(65536, 8, tuple(fpm.SpeedSample(8 * (q + 1), rng.uniform(1e9, 9e10),
                                                          rng.random(), q + 3) for q in range(9)),
                          "gpu0 cells/s")
    g = fpm.read_csv(fpm.write_csv(f))
    assert g == f
    with pytest.raises(_lib.ParseError):
        fpm.read_csv("# unit_cells=1 granularity=1 label=x\nx,speed,ci_halfwidth,repetitions\n1,2\n")


def test_t_quantile_and_summary():
    # Textbook 0.975 points of Student's t (stats.hpp:20-23).
    table = {1: 12.7062047361747, 2: 4.30265272974946, 3: 3.18244630528371,
             10: 2.22813885198627, 30: 2.04227245630124, 120: 1.97993040508242}
    for df, want in table.items():
        assert abs(fpm.t_quantile_975(df) - want) <= 1e-12 * want
    prev = math.inf
    for df in range(1, 300):
        q = fpm.t_quantile_975(df)
        assert q < prev
        prev = q
    assert abs(fpm.t_quantile_975(10 ** 7) - 1.959963984540054) < 1e-6
    with pytest.raises(_lib.InsufficientDataError):
        fpm.t_quantile_975(0)
    xs = [1.0, 2.0, 4.0, 7.0]
    s = fpm.summarize(xs)
    mu = sum(xs) / 4
    sd = math.sqrt(sum((v - mu) ** 2 for v in xs) / 3)
    assert abs(s.mean - mu) <= 1e-12 * mu and abs(s.stddev - sd) <= 1e-12 * sd
    assert abs(s.ci_halfwidth - fpm.t_quantile_975(3) * sd / 2.0) <= 1e-12 * s.ci_halfwidth
    with pytest.raises(_lib.InsufficientDataError):
        fpm.summarize([1.0])


@needs_ref
def test_slice_surface_parity():
    # fpm.cpp:192-222: validation errors and slicing, product vs reference.
    rng = random.Random(12)
    for _ in range(100):
        nv = sorted(rng.sample(range(100, 140, 4), rng.randint(1, 4)))
        mv = list(range(8, 8 + 4 * rng.randint(1, 6), 4))
        smp = [(mv[j], rng.uniform(1e5, 2e6), rng.random(), rng.randint(1, 5))
               for _ in nv for j in range(len(mv))]
        if rng.random() < 0.2:  # corrupt one x to hit the grid check
            q = rng.randrange(len(smp))
            smp[q] = (smp[q][0] + 1,) + smp[q][1:]
        fixed = rng.choice(nv + [nv[0] + 1])
        st, want = O.ref_slice_surface(15360, 4, nv, mv, smp, fixed)
        srf = fpm.SpeedSurface(15360, 4, tuple(nv), tuple(mv), tuple(smp), "s")
        try:
            f = fpm.slice_surface(srf, fixed)
            got, gst = (f.unit_cells, [(s.x, s.speed, s.ci_halfwidth, s.repetitions)
                                       for s in f.samples]), 0
        except _lib.ImbError as e:
            got, gst = None, e.code
        assert (gst, got) == (st, want)
