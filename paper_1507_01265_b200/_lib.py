"""ctypes binding of the C-ABI boundary ``include/imb_mpdata.h``.

The shared library ``libimb_b200.so`` (sm_100a kernels + C++ runtime) is
built in-tree by ``__graft_entry__.build()`` / ``make -C
paper_1507_01265_b200/csrc``. There is no fallback: if the library is missing
every entry point raises, so a GPU run can never silently take a CPU path.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "libimb_b200.so"

# Status codes: include/imb_mpdata.h (errors.hpp:15-64 one-to-one).
IMB_OK = 0
STATUS_NAMES = {
    1: "RangeError", 2: "DomainError", 3: "AlignmentError", 4: "IncompatibleModelError",
    5: "InsufficientDataError", 6: "InfeasibleError", 7: "TooLargeError", 8: "ConfigError",
    9: "ContractError", 10: "ParseError", 20: "CudaError", 21: "NcclError", 22: "NoMemError",
    99: "InternalError",
}


class ImbError(RuntimeError):
    """Base of the Python mirror of imb::Error (errors.hpp:10)."""

    code = 99


def _mk(name: str, code: int):
    return type(name, (ImbError,), {"code": code})


RangeError = _mk("RangeError", 1)
DomainError = _mk("DomainError", 2)
AlignmentError = _mk("AlignmentError", 3)
IncompatibleModelError = _mk("IncompatibleModelError", 4)
InsufficientDataError = _mk("InsufficientDataError", 5)
InfeasibleError = _mk("InfeasibleError", 6)
TooLargeError = _mk("TooLargeError", 7)
ConfigError = _mk("ConfigError", 8)
ContractError = _mk("ContractError", 9)
ParseError = _mk("ParseError", 10)
CudaError = _mk("CudaError", 20)
NcclError = _mk("NcclError", 21)
NoMemError = _mk("NoMemError", 22)
InternalError = _mk("InternalError", 99)
_BY_CODE = {c.code: c for c in (RangeError, DomainError, AlignmentError, IncompatibleModelError,
                                InsufficientDataError, InfeasibleError, TooLargeError,
                                ConfigError, ContractError, ParseError, CudaError, NcclError,
                                NoMemError, InternalError)}


class imb_domain(C.Structure):
    _fields_ = [("n", C.c_int64), ("m", C.c_int64), ("l", C.c_int64), ("halo", C.c_int64)]


class imb_opts(C.Structure):
    _fields_ = [("iord", C.c_int), ("nonos", C.c_int), ("precision", C.c_int)]


class imb_speed_sample(C.Structure):
    _fields_ = [("x", C.c_int64), ("speed", C.c_double), ("ci_halfwidth", C.c_double),
                ("repetitions", C.c_int64)]


P = C.POINTER
i64, i32, f64, vp, sz = C.c_int64, C.c_int, C.c_double, C.c_void_p, C.c_size_t
SS = P(imb_speed_sample)

# name -> (restype, argtypes); must match include/imb_mpdata.h exactly.
SIGNATURES = {
    "imb_last_error": (C.c_char_p, []),
    "imb_version": (C.c_char_p, []),
    "imb_step_radius": (i32, [P(imb_opts)]),
    "imb_team_create": (i32, [P(imb_domain), P(imb_opts), i32, i64, i64, P(vp)]),
    "imb_team_destroy": (i32, [vp]),
    "imb_team_init_recipe": (i32, [vp, i32, C.c_uint64]),
    "imb_team_upload": (i32, [vp, i32, vp, sz]),
    "imb_team_download": (i32, [vp, i32, vp, sz]),
    "imb_team_reset": (i32, [vp]),
    "imb_team_run": (i32, [vp, i32, P(f64), P(f64)]),
    "imb_team_step_host": (i32, [vp, vp, vp]),
    "imb_team_checksum": (i32, [vp, P(C.c_uint64)]),
    "imb_team_launch_count": (i64, [vp]),
    "imb_nccl_unique_id": (i32, [C.c_char_p]),
    "imb_team_connect_nccl": (i32, [vp, C.c_char_p, i32, i32]),
    "imb_team_ipc_export": (i32, [vp, C.c_char_p]),
    "imb_team_connect_ipc": (i32, [vp, C.c_char_p, C.c_char_p, i32, i32]),
    "imb_ring_plan": (i32, [i32, i32, i64, i64, P(i32), P(i32), P(i64), P(i64)]),
    "imb_slab_offsets": (i32, [P(i64), i32, P(i64)]),
    "imb_group_create": (i32, [P(imb_domain), P(imb_opts), i32, P(i32), P(i64), P(vp)]),
    "imb_group_destroy": (i32, [vp]),
    "imb_group_team": (i32, [vp, i32, P(vp)]),
    "imb_group_init_recipe": (i32, [vp, i32, C.c_uint64]),
    "imb_group_set_sync": (i32, [vp, i32]),
    "imb_group_run": (i32, [vp, i32, P(f64), P(f64)]),
    "imb_fill_halo_clamped": (i32, [P(imb_domain), P(f64)]),
    "imb_stage_max7": (i32, [P(imb_domain), P(f64), P(f64)]),
    "imb_stage_min7": (i32, [P(imb_domain), P(f64), P(f64)]),
    "imb_checksum_padded": (i32, [P(imb_domain), P(f64), P(C.c_uint64)]),
    "imb_speed_validate": (i32, [i64, i64, SS, i32]),
    "imb_eval_speed": (i32, [i64, i64, SS, i32, f64, P(f64)]),
    "imb_eval_time": (i32, [i64, i64, SS, i32, f64, P(f64)]),
    "imb_check_condition": (i32, [i64, i64, SS, i32, P(i32), P(i64), i32, P(i32), P(i64)]),
    "imb_classify_shape": (i32, [i64, i64, SS, i32, P(i32), P(i64)]),
    "imb_average": (i32, [i64, i64, SS, i32, i32, SS]),
    "imb_scaled": (i32, [i64, i64, SS, i32, f64, SS]),
    "imb_speed_csv_parse": (i32, [C.c_char_p, C.c_size_t, P(i64), P(i64), SS, i32, P(i32), C.c_char_p,
                                  C.c_size_t, P(i32)]),
    "imb_speed_csv_format": (i32, [i64, i64, SS, i32, C.c_char_p, C.c_char_p, C.c_size_t,
                                   P(C.c_size_t)]),
    "imb_slice_surface": (i32, [i64, i64, P(i64), i32, P(i64), i32, SS, i64, SS, P(i64)]),
    "imb_predict_makespan": (i32, [i64, i64, SS, i32, P(i64), i32, P(f64), P(f64)]),
    "imb_partition_paired": (i32, [i64, i64, SS, i32, i64, i32, i32, P(i64), P(f64), P(f64), P(i64)]),
    "imb_partition_general": (i32, [i64, i64, SS, i32, i64, i32, i32, P(i64), P(f64), P(f64), P(i64)]),
    "imb_brute_force_oracle": (i32, [i64, i64, SS, i32, i64, i32, i32, i64, P(i64), P(f64), P(f64), P(i64)]),
    "imb_improvement_search": (i32, [i64, i64, SS, i32, i64, P(i32), P(i64), P(f64), P(i64)]),
    "imb_t_quantile_975": (f64, [i32]),
    "imb_summarize": (i32, [P(f64), i32, P(f64), P(f64), P(f64)]),
}

_lib: C.CDLL | None = None


def load() -> C.CDLL:
    """Load libimb_b200.so once; raises (never falls back) when it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    path = Path(os.environ.get("IMB_LIB", LIB_PATH))
    if not path.exists():
        raise ImportError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "or `make -C paper_1507_01265_b200/csrc` (there is no CPU fallback)")
    lib = C.CDLL(str(path))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status: int) -> None:
    if status != IMB_OK:
        msg = load().imb_last_error().decode(errors="replace")
        raise _BY_CODE.get(status, InternalError)(f"[{STATUS_NAMES.get(status, status)}] {msg}")


def samples_array(samples):
    """Sequence of (x, speed[, ci, reps]) or objects with those attributes -> ctypes array."""
    arr = (imb_speed_sample * max(len(samples), 1))()
    for q, s in enumerate(samples):
        if isinstance(s, imb_speed_sample):
            arr[q] = s
            continue
        if hasattr(s, "x"):
            vals = (s.x, s.speed, getattr(s, "ci_halfwidth", 0.0), getattr(s, "repetitions", 1))
        else:
            vals = list(s) + [0.0, 1][len(s) - 2:]
        arr[q] = imb_speed_sample(int(vals[0]), float(vals[1]), float(vals[2]), int(vals[3]))
    return arr
