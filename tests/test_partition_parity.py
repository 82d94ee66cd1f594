"""Product partitioner (libimb_b200.so via the C-ABI) vs the reference.

The reference partitioner compiles here unmodified (oracle/_ref, SURVEY.md
§8c); its outputs on the paper example, the SURVEY Appendix B cases and 300
seeded random tables are committed in tests/golden/partition_ref.json. Parity
means: identical status, integer-identical shares (order included) and
offset, bit-identical per-processor times and makespan. CPU only.
"""
import json
import random
from pathlib import Path

import pytest

from paper_1507_01265_b200 import _lib, fpm

ROWS = json.loads((Path(__file__).parent / "golden" / "partition_ref.json").read_text())
FN = {"paired": fpm.partition_paired, "general": fpm.partition_general,
      "brute": fpm.brute_force_oracle}


def product(kind, unit, g, samples, total, p, allow_idle=False):
    try:
        model = fpm.SpeedFunction(unit, g, tuple(fpm.SpeedSample(int(x), float(s))
                                                 for x, s in samples))
        r = FN[kind](fpm.PartitionProblem(total, p, model, allow_idle))
    except _lib.ImbError as e:
        return e.code, None
    return 0, r


def test_fixture_covers_all_kinds():
    kinds = {r["kind"] for r in ROWS}
    assert kinds == {"paired", "general", "brute"}
    assert sum(r["status"] == 0 for r in ROWS) > 300
    assert {r["status"] for r in ROWS} >= {0, 3, 6, 9}


@pytest.mark.parametrize("row", ROWS, ids=lambda r: f"{r['kind']}-n{r['total']}-p{r['p']}")
def test_matches_reference_fixture(row):
    st, r = product(row["kind"], row["unit"], row["g"], row["samples"], row["total"], row["p"],
                    row["allow_idle"])
    assert st == row["status"]
    if st == 0:
        assert r.shares == row["shares"]
        assert r.per_time == row["per_time"]  # bit-identical
        assert r.makespan == row["makespan"]
        assert r.offset == row["offset"]


def test_paper_worked_example():
    # shares (112,128,112,128), offset 8, 1.386 s.
    model = fpm.SpeedFunction(15360, 8, ((112, 1436742.0), (120, 1240377.0), (128, 1418579.0)))
    r = fpm.partition_paired(fpm.PartitionProblem(480, 4, model))
    assert r.shares == [112, 128, 112, 128] and r.offset == 8
    assert abs(r.makespan - 1.385950) < 1e-6
    assert abs(fpm.predict_makespan(model, [120] * 4).makespan - 1.486) < 1e-3
    g = fpm.partition_general(fpm.PartitionProblem(480, 4, model))
    assert g.shares == [112, 112, 128, 128]  # ascending, as the reference emits
    b = fpm.brute_force_oracle(fpm.PartitionProblem(480, 4, model))
    assert b.shares == [128, 128, 112, 112]  # descending


@pytest.mark.skipif(not __import__("oracle.oracle", fromlist=["x"]).ref_available(),
                    reason="oracle/_ref not built (reference sources absent)")
def test_live_random_parity_against_compiled_reference():
    from oracle import oracle as O
    rng = random.Random(77)
    for _ in range(1500):
        g = rng.choice([1, 2, 3, 4])
        x = rng.randint(1, 4) * g
        samples = []
        for _ in range(rng.randint(1, 10)):
            # integer speeds make ties (and equal makespans) common
            samples.append((x, rng.choice([rng.uniform(1, 9), float(rng.randint(1, 4))])))
            x += rng.randint(1, 3) * g
        total = rng.randint(1, 40) * g
        p = rng.randint(1, 6)
        idle = rng.random() < 0.3
        unit = rng.choice([1, 7, 15360])
        for kind in ("paired", "general", "brute"):
            st, sh, pt, ms, off = O.ref_partition(kind, unit, g, samples, total, p, idle)
            mst, r = product(kind, unit, g, samples, total, p, idle)
            assert mst == st, (kind, samples, total, p, idle)
            if st == 0:
                assert (r.shares, r.per_time, r.makespan, r.offset) == (sh, pt, ms, off)


def test_theorem1_balanced_is_optimal_when_condition_holds():
    # s(x)/x non-increasing => the even split is optimal.
    rng = random.Random(5)
    for _ in range(100):
        xs = list(range(1, 13))
        sp, s = [], rng.uniform(1, 5)
        for x in xs:
            sp.append(s)
            s *= rng.uniform(0.9, 1.0 + 1.0 / x)  # keeps s(x)/x decreasing
        model = fpm.SpeedFunction(1, 1, tuple(zip(xs, sp)))
        if not fpm.check_condition(model).satisfied:
            continue
        for p in (2, 3, 4):
            total = p * rng.randint(1, 3)
            r = fpm.partition_general(fpm.PartitionProblem(total, p, model))
            even = fpm.predict_makespan(model, [total // p] * p)
            assert r.makespan == even.makespan


def test_scale_invariance():
    # PAPER.md:163 / SPEC.md:223: scaling s by a constant keeps the shares.
    rng = random.Random(9)
    for _ in range(50):
        xs = [2 * q for q in range(1, 9)]
        model = fpm.SpeedFunction(3, 2, tuple((x, rng.uniform(1, 10)) for x in xs))
        pr = fpm.PartitionProblem(16, 4, model)
        base = fpm.partition_general(pr).shares
        basep = fpm.partition_paired(pr).shares
        for f in (0.5, 3.0, 1e3, 1e-3, 7.25):
            m2 = fpm.scaled(model, f)
            assert fpm.partition_general(fpm.PartitionProblem(16, 4, m2)).shares == base
            assert fpm.partition_paired(fpm.PartitionProblem(16, 4, m2)).shares == basep


def test_general_never_worse_than_paired():
    rng = random.Random(13)
    for _ in range(100):
        xs = list(range(1, 21))
        model = fpm.SpeedFunction(1, 1, tuple((x, rng.uniform(1, 10)) for x in xs))
        for p in (2, 4):
            pr = fpm.PartitionProblem(20, p, model)
            assert fpm.partition_general(pr).makespan <= fpm.partition_paired(pr).makespan
