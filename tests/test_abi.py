"""The C-ABI library loads and exports every symbol include/imb_mpdata.h
declares; the status mapping follows errors.hpp. No compute calls need a GPU
here (CPU only)."""
import ctypes as C
import re
import subprocess
from pathlib import Path

import pytest

from paper_1507_01265_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]
HEADER = (ROOT / "include" / "imb_mpdata.h").read_text()
DECLARED = sorted(set(re.findall(r"\b(imb_[a-z0-9_]+)\s*\(", HEADER)))


def test_header_declares_the_boundary():
    for name in ("imb_team_create", "imb_team_run", "imb_partition_paired",
                 "imb_partition_general", "imb_eval_time", "imb_group_run",
                 "imb_team_connect_nccl", "imb_stage_max7"):
        assert name in DECLARED


def test_every_declared_symbol_is_exported():
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (imb_\w+)", out))
    missing = [d for d in DECLARED if d not in exported]
    assert not missing, missing
    lib = _lib.load()
    for d in DECLARED:
        assert getattr(lib, d) is not None


def test_python_binding_covers_header():
    assert sorted(_lib.SIGNATURES) == DECLARED


def test_library_is_sm100a():
    # The fatbin carries sm_100a SASS (cross-compiled here, no GPU needed).
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_status_codes_without_gpu():
    lib = _lib.load()
    assert lib.imb_version().decode().startswith("0.1.0")
    # A team needs a device: on a GPU-less host the CUDA/config error surfaces,
    # never a silent CPU path.
    if not Path("/dev/nvidia0").exists():
        h = C.c_void_p()
        st = lib.imb_team_create(C.byref(_lib.imb_domain(8, 8, 8, 1)),
                                 C.byref(_lib.imb_opts(2, 1, 0)), 0, 0, 8, C.byref(h))
        assert st in (_lib.CudaError.code, _lib.ConfigError.code)
        assert lib.imb_last_error()
    # Contract violations map to 9, alignment to 3, as errors.hpp says.
    s = _lib.samples_array([(8, 1.0), (16, 2.0)])
    sh = (C.c_int64 * 3)()
    pt = (C.c_double * 3)()
    ms, off = C.c_double(), C.c_int64()
    assert lib.imb_partition_paired(1, 8, s, 2, 48, 3, 0, sh, pt, C.byref(ms), C.byref(off)) == 9
    assert lib.imb_partition_paired(1, 8, s, 2, 40, 2, 0, sh, pt, C.byref(ms), C.byref(off)) == 3
    assert b"granules" in lib.imb_last_error()
    with pytest.raises(_lib.ContractError):
        _lib.check(9)


def test_step_radius():
    from paper_1507_01265_b200 import mpdata
    assert mpdata.step_radius(mpdata.Options(1, False)) == 1
    assert mpdata.step_radius(mpdata.Options(2, False)) == 2
    assert mpdata.step_radius(mpdata.Options(2, True)) == 3
    assert mpdata.step_radius(mpdata.Options(3, True)) == 5
    bad = _lib.imb_opts(2, 1, 7)  # unknown precision
    assert _lib.load().imb_step_radius(C.byref(bad)) == -_lib.ConfigError.code
    h = C.c_void_p()
    assert _lib.load().imb_team_create(None, None, 0, 0, 0, C.byref(h)) == _lib.ContractError.code


def _demo():
    subprocess.run(["make", "-s", "-C", str(ROOT / "paper_1507_01265_b200" / "csrc"), "demo"],
                   check=True)
    return ROOT / "tests" / "cpp" / "api_demo"


def test_cpp_caller_links_reference_named_api():
    # A C++ program written against include/imbalance/*.hpp (the reference's
    # names) builds and links against libimb_b200.so; its FPM part runs here.
    out = subprocess.run([str(_demo()), "cpu"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "cpu part: ok" in out.stdout


@pytest.mark.gpu
def test_cpp_caller_runs_workload_on_gpu():
    out = subprocess.run([str(_demo()), "gpu"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "gpu part: ok" in out.stdout
