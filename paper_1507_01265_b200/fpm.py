"""Python mirror of the FPM model + partitioner API.

Names, argument meaning and error behaviour follow the reference headers
/root/reference/proj/include/imbalance/fpm.hpp:13-127 and partition.hpp:17-72;
every call goes through the C-ABI (include/imb_mpdata.h) into the C++
implementation in csrc/host/, so Python adds no arithmetic of its own.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Iterable, Optional, Sequence

from . import _lib
from ._lib import check, load, samples_array


@dataclass(frozen=True)
class SpeedSample:  # fpm.hpp:13-18
    x: int
    speed: float
    ci_halfwidth: float = 0.0
    repetitions: int = 1


@dataclass(frozen=True)
class SpeedFunction:  # fpm.hpp:28-49
    unit_cells: int
    granularity: int
    samples: tuple
    label: str = ""

    def __post_init__(self):
        object.__setattr__(self, "samples",
                           tuple(s if isinstance(s, SpeedSample) else SpeedSample(*s)
                                 for s in self.samples))
        arr = samples_array(self.samples)
        check(load().imb_speed_validate(self.unit_cells, self.granularity, arr, len(self.samples)))

    @property
    def min_x(self) -> int:
        return self.samples[0].x

    @property
    def max_x(self) -> int:
        return self.samples[-1].x

    def in_range(self, x: float) -> bool:
        return self.min_x <= x <= self.max_x

    def _c(self):
        return (self.unit_cells, self.granularity, samples_array(self.samples), len(self.samples))


def eval_speed(f: SpeedFunction, x: float) -> float:  # fpm.hpp:93-96
    out = C.c_double()
    check(load().imb_eval_speed(*f._c(), float(x), C.byref(out)))
    return out.value


def eval_time(f: SpeedFunction, x: float) -> float:  # fpm.hpp:98-101
    out = C.c_double()
    check(load().imb_eval_time(*f._c(), float(x), C.byref(out)))
    return out.value


@dataclass
class ConditionReport:  # fpm.hpp:51-63
    satisfied: bool
    violations: list
    max_gain_pair: Optional[tuple]


def check_condition(f: SpeedFunction) -> ConditionReport:
    n = len(f.samples)
    cap = max(n * (n - 1) // 2, 1)
    viol = (C.c_int64 * (2 * cap))()
    sat, nv = C.c_int(), C.c_int()
    mg = (C.c_int64 * 2)()
    check(load().imb_check_condition(*f._c(), C.byref(sat), viol, cap, C.byref(nv), mg))
    pairs = [(viol[2 * q], viol[2 * q + 1]) for q in range(nv.value)]
    return ConditionReport(bool(sat.value), pairs, None if mg[0] < 0 else (mg[0], mg[1]))


SHAPES = ("monotonically-decreasing", "increasing-concave-then-decreasing", "other")


def classify_shape(f: SpeedFunction):  # fpm.hpp:107 -> (classification, peak_x|None)
    cls, peak = C.c_int(), C.c_int64()
    check(load().imb_classify_shape(*f._c(), C.byref(cls), C.byref(peak)))
    return SHAPES[cls.value], (None if peak.value < 0 else peak.value)


def average(fs: Sequence[SpeedFunction]) -> SpeedFunction:  # fpm.hpp:113
    if not fs:
        raise _lib.ContractError("average needs at least one speed function")
    head = fs[0]
    ns = len(head.samples)
    if any(len(f.samples) != ns for f in fs):
        raise _lib.IncompatibleModelError("speed functions sampled on different grids")
    flat = samples_array([s for f in fs for s in f.samples])
    # units/granularity mismatch is detected by the C++ side per function
    for f in fs:
        if (f.unit_cells, f.granularity) != (head.unit_cells, head.granularity):
            raise _lib.IncompatibleModelError("speed functions disagree on units or granularity")
    out = (_lib.imb_speed_sample * max(ns, 1))()
    check(load().imb_average(head.unit_cells, head.granularity, flat, len(fs), ns, out))
    label = "avg(" + ",".join(f.label for f in fs) + ")"
    return SpeedFunction(head.unit_cells, head.granularity,
                         tuple(SpeedSample(o.x, o.speed, o.ci_halfwidth, o.repetitions)
                               for o in out[:ns]), label)


def scaled(f: SpeedFunction, factor: float) -> SpeedFunction:  # fpm.hpp:118
    ns = len(f.samples)
    out = (_lib.imb_speed_sample * max(ns, 1))()
    check(load().imb_scaled(*f._c(), float(factor), out))
    return SpeedFunction(f.unit_cells, f.granularity,
                         tuple(SpeedSample(o.x, o.speed, o.ci_halfwidth, o.repetitions)
                               for o in out[:ns]), f.label)


@dataclass(frozen=True)
class SpeedSurface:  # fpm.hpp:81-91 — rectangular (n, m) grid, row-major in n
    unit_cells: int
    granularity: int
    n_values: tuple
    m_values: tuple
    samples: tuple  # len(n_values) * len(m_values) SpeedSample, x == m_values[j]
    label: str = ""


def slice_surface(g: SpeedSurface, fixed_n: int) -> SpeedFunction:  # fpm.hpp:123
    nn, nm = len(g.n_values), len(g.m_values)
    smp = tuple(s if isinstance(s, SpeedSample) else SpeedSample(*s) for s in g.samples)
    out = (_lib.imb_speed_sample * max(nm, 1))()
    uc = C.c_int64()
    check(load().imb_slice_surface(g.unit_cells, g.granularity,
                                   (C.c_int64 * max(nn, 1))(*g.n_values), nn,
                                   (C.c_int64 * max(nm, 1))(*g.m_values), nm,
                                   samples_array(smp), int(fixed_n), out, C.byref(uc)))
    return SpeedFunction(uc.value, g.granularity,
                         tuple(SpeedSample(o.x, o.speed, o.ci_halfwidth, o.repetitions)
                               for o in out[:nm]), f"{g.label}@n={fixed_n}")


# ---- partitioner (partition.hpp:17-72) -------------------------------------
@dataclass
class PartitionProblem:
    total: int
    processors: int
    model: SpeedFunction
    allow_idle: bool = False


@dataclass
class Partition:
    shares: list
    per_time: list
    makespan: float
    offset: Optional[int] = None


K_DEFAULT_ORACLE_CAP = 10_000_000


def _partition(fn, pr: PartitionProblem, *extra) -> Partition:
    p = max(pr.processors, 1)
    shares = (C.c_int64 * p)()
    per = (C.c_double * p)()
    ms, off = C.c_double(), C.c_int64()
    check(fn(*pr.model._c(), int(pr.total), int(pr.processors), int(bool(pr.allow_idle)), *extra,
             shares, per, C.byref(ms), C.byref(off)))
    return Partition(list(shares), list(per), ms.value, None if off.value < 0 else off.value)


def partition_paired(pr: PartitionProblem) -> Partition:  # Algorithm 1
    return _partition(load().imb_partition_paired, pr)


def partition_general(pr: PartitionProblem) -> Partition:
    return _partition(load().imb_partition_general, pr)


def brute_force_oracle(pr: PartitionProblem, max_compositions: int = K_DEFAULT_ORACLE_CAP):
    return _partition(load().imb_brute_force_oracle, pr, int(max_compositions))


def predict_makespan(model: SpeedFunction, shares: Sequence[int]) -> Partition:
    p = len(shares)
    arr = (C.c_int64 * max(p, 1))(*shares)
    per = (C.c_double * max(p, 1))()
    ms = C.c_double()
    check(load().imb_predict_makespan(*model._c(), arr, p, per, C.byref(ms)))
    return Partition(list(shares), list(per[:p]), ms.value, None)


@dataclass
class Improvement:
    violating_pair: tuple
    delta: int
    gain_s: float


def improvement_search(model: SpeedFunction, balanced_share: int) -> Optional[Improvement]:
    found, delta, gain = C.c_int(), C.c_int64(), C.c_double()
    pair = (C.c_int64 * 2)()
    check(load().imb_improvement_search(*model._c(), int(balanced_share), C.byref(found),
                                        C.byref(delta), C.byref(gain), pair))
    if not found.value:
        return None
    return Improvement((pair[0], pair[1]), delta.value, gain.value)


# ---- stats (stats.hpp) ------------------------------------------------------
def t_quantile_975(df: int) -> float:
    v = load().imb_t_quantile_975(int(df))
    if v < 0:
        raise _lib.InsufficientDataError("t quantile needs df >= 1")
    return v


@dataclass
class Summary:
    count: int
    mean: float
    stddev: float
    ci_halfwidth: float


def summarize(xs: Iterable[float]) -> Summary:
    xs = [float(v) for v in xs]
    arr = (C.c_double * max(len(xs), 1))(*xs)
    m, s, ci = C.c_double(), C.c_double(), C.c_double()
    check(load().imb_summarize(arr, len(xs), C.byref(m), C.byref(s), C.byref(ci)))
    return Summary(len(xs), m.value, s.value, ci.value)


# ---- speed-function CSV ----------------------------------
# One parser/writer of the format: the C++ one (csrc/host/fpm.cpp) behind the
# C-ABI; these wrappers only move the text across.
def write_csv(f: SpeedFunction) -> str:
    arr = samples_array(f.samples)
    n = C.c_size_t()
    lab = f.label.encode()
    rc = load().imb_speed_csv_format(f.unit_cells, f.granularity, arr, len(f.samples), lab, None, 0,
                                     C.byref(n))
    if rc not in (0, _lib.RangeError.code):
        check(rc)
    buf = C.create_string_buffer(n.value + 1)
    check(load().imb_speed_csv_format(f.unit_cells, f.granularity, arr, len(f.samples), lab, buf,
                                      n.value + 1, C.byref(n)))
    return buf.value.decode()


def read_csv(text: str) -> SpeedFunction:
    raw = text.encode()
    unit, gran, ns, line = C.c_int64(), C.c_int64(), C.c_int(), C.c_int()
    lab = C.create_string_buffer(len(raw) + 1)
    cap = raw.count(b"\n") + 1
    out = (_lib.imb_speed_sample * cap)()
    rc = load().imb_speed_csv_parse(raw, len(raw), C.byref(unit), C.byref(gran), out, cap,
                                    C.byref(ns), lab, len(raw) + 1, C.byref(line))
    check(rc)
    samples = tuple(SpeedSample(o.x, o.speed, o.ci_halfwidth, o.repetitions) for o in out[:ns.value])
    return SpeedFunction(unit.value, gran.value, samples, lab.value.decode())


# ---- 2-D speed-surface CSV: row-major in n, then m ------------
def write_surface_csv(g: SpeedSurface) -> str:
    rows = [f"# unit_cells={g.unit_cells} granularity={g.granularity} label={g.label}",
            "n,m,speed,ci_halfwidth,repetitions"]
    nm = len(g.m_values)
    for q, s in enumerate(g.samples):
        s = s if isinstance(s, SpeedSample) else SpeedSample(*s)
        rows.append(f"{g.n_values[q // nm]},{s.x},{s.speed:.17g},{s.ci_halfwidth:.17g},"
                    f"{s.repetitions}")
    return "\n".join(rows) + "\n"


def read_surface_csv(text: str) -> SpeedSurface:
    lines = text.splitlines()
    if not lines or not lines[0].startswith("# "):
        raise _lib.ParseError("missing '# ' header (line 1)")
    head, _, label = lines[0][2:].partition(" label=")
    kv = dict(tok.split("=", 1) for tok in head.split() if "=" in tok)
    try:
        unit, gran = int(kv["unit_cells"]), int(kv["granularity"])
    except (KeyError, ValueError) as e:
        raise _lib.ParseError(f"bad header ({e}) (line 1)") from None
    if len(lines) < 2 or lines[1].strip() != "n,m,speed,ci_halfwidth,repetitions":
        raise _lib.ParseError("expected column header (line 2)")
    ns, ms, samples = [], [], []
    for no, line in enumerate(lines[2:], start=3):
        if not line.strip():
            continue
        cols = line.split(",")
        if len(cols) != 5:
            raise _lib.ParseError(f"expected 5 columns (line {no})")
        try:
            n, m = int(cols[0]), int(cols[1])
            samples.append(SpeedSample(m, float(cols[2]), float(cols[3]), int(cols[4])))
        except ValueError as e:
            raise _lib.ParseError(f"{e} (line {no})") from None
        if not ns or ns[-1] != n:
            if n in ns:
                raise _lib.ParseError(f"rows not grouped by n (line {no})")
            ns.append(n)
        if len(ns) == 1:
            ms.append(m)
        else:
            col = len(samples) - 1 - (len(ns) - 1) * len(ms)
            if col >= len(ms) or m != ms[col]:
                raise _lib.ParseError(f"m grid differs between n rows (line {no})")
    if not samples or len(samples) != len(ns) * len(ms):
        raise _lib.ParseError("surface is not a full n x m grid")
    return SpeedSurface(unit, gran, tuple(ns), tuple(ms), tuple(samples), label)
