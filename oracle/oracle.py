"""TEST INFRASTRUCTURE ONLY — ctypes front-end of the two checkers.

* ``liborc_mpdata.so``: the C restatement of MPDATA (mpdata_oracle.c).
  PARITY UNPINNED BY THE REFERENCE — the reference ships no MPDATA; see
  mpdata_oracle.h. Pinned by analytic properties and self-generated golden
  checksums (tests/golden/).
* ``_ref/libimb_ref.so``: the unmodified reference partitioner
  (/root/reference/proj/src/{fpm,partition}.cpp) behind ref_shim.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this module. It is never part of the product path.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORC_PATH = HERE / "liborc_mpdata.so"
REF_PATH = HERE / "_ref" / "libimb_ref.so"

_orc = None
_ref = None


def build() -> None:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def orc():
    global _orc
    if _orc is None:
        if not ORC_PATH.exists():
            build()
        lib = C.CDLL(str(ORC_PATH))
        i64, P64, P32 = C.c_int64, C.POINTER(C.c_double), C.POINTER(C.c_float)
        lib.orc_init_f64.argtypes = [C.c_int, i64, i64, i64, C.c_uint64, i64, i64] + [P64] * 5
        lib.orc_init_f32.argtypes = [C.c_int, i64, i64, i64, C.c_uint64, i64, i64] + [P32] * 5
        lib.orc_run_f64.argtypes = [C.c_int, C.c_int, i64, i64, i64, P64, P64, P64, P64, P64,
                                    C.c_int, C.c_int]
        lib.orc_run_f32.argtypes = [C.c_int, C.c_int, i64, i64, i64, P32, P32, P32, P32, P32,
                                    C.c_int, C.c_int]
        lib.orc_checksum_f64.argtypes = [P64, C.c_size_t]
        lib.orc_checksum_f64.restype = C.c_uint64
        lib.orc_checksum_f32.argtypes = [P32, C.c_size_t]
        lib.orc_checksum_f32.restype = C.c_uint64
        for nm in ("orc_stage_max7", "orc_stage_min7"):
            getattr(lib, nm).argtypes = [P64, P64, i64, i64, i64, i64]
        lib.orc_fill_halo_clamped.argtypes = [P64, i64, i64, i64, i64]
        lib.orc_eps.restype = C.c_double
        _orc = lib
    return _orc


def _ptr(a: np.ndarray):
    t = C.c_double if a.dtype == np.float64 else C.c_float
    return a.ctypes.data_as(C.POINTER(t))


def init_fields(recipe: int, n: int, m: int, l: int, seed: int = 42, i0: int = 0,
                ni: int | None = None, dtype=np.float64):
    """Seeded (x, u, v, w, h) for planes [i0, i0+ni) of the global n x m x l grid."""
    ni = n if ni is None else ni
    arrs = [np.empty((ni, m, l), dtype=dtype) for _ in range(5)]
    fn = orc().orc_init_f64 if dtype == np.float64 else orc().orc_init_f32
    rc = fn(recipe, n, m, l, C.c_uint64(seed), i0, ni, *[_ptr(a) for a in arrs])
    assert rc == 0, "orc_init failed"
    return arrs


def run(x, u, v, w, h, *, iord: int, nonos: bool, steps: int, threads: int = 1) -> np.ndarray:
    """`steps` MPDATA steps on copies of the inputs; returns the new x."""
    x = np.array(x, copy=True, order="C")
    arrs = [np.ascontiguousarray(a, dtype=x.dtype) for a in (u, v, w, h)]
    n, m, l = x.shape
    fn = orc().orc_run_f64 if x.dtype == np.float64 else orc().orc_run_f32
    rc = fn(int(iord), int(bool(nonos)), n, m, l, _ptr(x), *[_ptr(a) for a in arrs], int(steps),
            int(threads))
    assert rc == 0, "orc_run failed"
    return x


def checksum(x: np.ndarray) -> int:
    a = np.ascontiguousarray(x)
    if a.dtype == np.float64:
        return orc().orc_checksum_f64(_ptr(a), a.size)
    return orc().orc_checksum_f32(_ptr(a), a.size)


def stage7(padded: np.ndarray, n, m, l, halo, is_max=True) -> np.ndarray:
    out = np.zeros_like(padded)
    fn = orc().orc_stage_max7 if is_max else orc().orc_stage_min7
    fn(_ptr(padded), _ptr(out), n, m, l, halo)
    return out


def fill_halo_clamped(padded: np.ndarray, n, m, l, halo) -> np.ndarray:
    a = np.array(padded, copy=True)
    orc().orc_fill_halo_clamped(_ptr(a), n, m, l, halo)
    return a


# ---- the reference partitioner --------------------------------------------
class RefSample(C.Structure):
    _fields_ = [("x", C.c_int64), ("speed", C.c_double), ("ci_halfwidth", C.c_double),
                ("repetitions", C.c_int64)]


def ref_available() -> bool:
    return REF_PATH.exists()


def ref():
    global _ref
    if _ref is None:
        if not REF_PATH.exists():
            build()
        if not REF_PATH.exists():
            raise FileNotFoundError(f"{REF_PATH} not built (reference sources absent?)")
        lib = C.CDLL(str(REF_PATH))
        i64, SS, f64 = C.c_int64, C.POINTER(RefSample), C.c_double
        P = C.POINTER
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_eval_speed.argtypes = [i64, i64, SS, C.c_int, f64, P(f64)]
        lib.ref_eval_time.argtypes = [i64, i64, SS, C.c_int, f64, P(f64)]
        lib.ref_partition.argtypes = [C.c_int, i64, i64, SS, C.c_int, i64, C.c_int, C.c_int, i64,
                                      P(i64), P(f64), P(f64), P(i64)]
        lib.ref_predict_makespan.argtypes = [i64, i64, SS, C.c_int, P(i64), C.c_int, P(f64), P(f64)]
        lib.ref_check_condition.argtypes = [i64, i64, SS, C.c_int, P(C.c_int), P(i64), C.c_int,
                                            P(C.c_int), P(i64)]
        lib.ref_classify_shape.argtypes = [i64, i64, SS, C.c_int, P(C.c_int), P(i64)]
        lib.ref_improvement_search.argtypes = [i64, i64, SS, C.c_int, i64, P(C.c_int), P(i64),
                                               P(f64), P(i64)]
        lib.ref_average.argtypes = [i64, i64, SS, C.c_int, C.c_int, SS]
        lib.ref_slice_surface.argtypes = [i64, i64, P(i64), C.c_int, P(i64), C.c_int, SS, i64,
                                          SS, P(i64)]
        _ref = lib
    return _ref


def _samples(samples):
    arr = (RefSample * max(len(samples), 1))()
    for q, s in enumerate(samples):
        vals = list(s) + [0.0, 1][len(s) - 2:]
        arr[q] = RefSample(int(vals[0]), float(vals[1]), float(vals[2]), int(vals[3]))
    return arr


def ref_partition(kind: str, unit, g, samples, total, p, allow_idle=False, cap=10_000_000):
    """Returns (status, shares, per_time, makespan, offset|None)."""
    k = {"paired": 0, "general": 1, "brute": 2}[kind]
    pp = max(p, 1)
    sh, pt = (C.c_int64 * pp)(), (C.c_double * pp)()
    ms, off = C.c_double(), C.c_int64()
    st = ref().ref_partition(k, unit, g, _samples(samples), len(samples), total, p,
                             int(allow_idle), cap, sh, pt, C.byref(ms), C.byref(off))
    if st:
        return st, None, None, None, None
    return 0, list(sh[:p]), list(pt[:p]), ms.value, (None if off.value < 0 else off.value)


def ref_eval(kind: str, unit, g, samples, x):
    out = C.c_double()
    fn = ref().ref_eval_speed if kind == "speed" else ref().ref_eval_time
    st = fn(unit, g, _samples(samples), len(samples), float(x), C.byref(out))
    return st, (out.value if st == 0 else None)


def ref_predict(unit, g, samples, shares):
    p = len(shares)
    pt, ms = (C.c_double * max(p, 1))(), C.c_double()
    st = ref().ref_predict_makespan(unit, g, _samples(samples), len(samples),
                                    (C.c_int64 * max(p, 1))(*shares), p, pt, C.byref(ms))
    return st, (list(pt[:p]) if st == 0 else None), (ms.value if st == 0 else None)


def ref_check_condition(unit, g, samples):
    n = len(samples)
    cap = max(n * (n - 1) // 2, 1)
    viol = (C.c_int64 * (2 * cap))()
    sat, nv, mg = C.c_int(), C.c_int(), (C.c_int64 * 2)()
    st = ref().ref_check_condition(unit, g, _samples(samples), n, C.byref(sat), viol, cap,
                                   C.byref(nv), mg)
    if st:
        return st, None
    pairs = [(viol[2 * q], viol[2 * q + 1]) for q in range(nv.value)]
    return 0, (bool(sat.value), pairs, None if mg[0] < 0 else (mg[0], mg[1]))


def ref_classify(unit, g, samples):
    cls, peak = C.c_int(), C.c_int64()
    st = ref().ref_classify_shape(unit, g, _samples(samples), len(samples), C.byref(cls),
                                  C.byref(peak))
    return st, (None if st else (cls.value, None if peak.value < 0 else peak.value))


def ref_improvement(unit, g, samples, balanced):
    found, delta, gain, pair = C.c_int(), C.c_int64(), C.c_double(), (C.c_int64 * 2)()
    st = ref().ref_improvement_search(unit, g, _samples(samples), len(samples), balanced,
                                      C.byref(found), C.byref(delta), C.byref(gain), pair)
    if st:
        return st, None
    return 0, (None if not found.value else ((pair[0], pair[1]), delta.value, gain.value))


def ref_average(unit, g, funcs):
    nf, ns = len(funcs), len(funcs[0])
    flat = _samples([s for f in funcs for s in f])
    out = (RefSample * max(ns, 1))()
    st = ref().ref_average(unit, g, flat, nf, ns, out)
    return st, (None if st else [(o.x, o.speed, o.ci_halfwidth, o.repetitions) for o in out[:ns]])


def ref_slice_surface(unit, g, n_values, m_values, samples, fixed_n):
    nn, nm = len(n_values), len(m_values)
    out = (RefSample * max(nm, 1))()
    uc = C.c_int64()
    st = ref().ref_slice_surface(unit, g, (C.c_int64 * max(nn, 1))(*n_values), nn,
                                 (C.c_int64 * max(nm, 1))(*m_values), nm, _samples(samples),
                                 fixed_n, out, C.byref(uc))
    if st:
        return st, None
    return 0, (uc.value, [(o.x, o.speed, o.ci_halfwidth, o.repetitions) for o in out[:nm]])
