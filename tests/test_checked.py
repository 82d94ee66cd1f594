"""Checked build (-DIMB_CHECKED device bounds asserts) over small runs of every
kernel family — the stand-in for compute-sanitizer,
which this GPU pool does not allow. A failed assert traps the kernel, so the
subprocess fails with the IMB_CHECKED message on stdout."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
CHECKED = ROOT / "paper_1507_01265_b200" / "libimb_b200_checked.so"
sys.path.insert(0, str(ROOT / "tools"))
from sanitize_cases import CASES  # noqa: E402


def test_cases_cover_every_kernel_family():
    names = set(CASES)
    assert {"fused_f64", "fused_f32", "fused_plain", "fused_iord3", "fused_l64", "fused_l32",
            "staged", "group", "group_flags"} <= names


@pytest.mark.gpu
@pytest.mark.parametrize("case", sorted(CASES))
def test_checked_build_case(case):
    if not CHECKED.exists():
        subprocess.run(["bash", str(ROOT / "tools" / "checked_build.sh")], check=True)
    env = dict(os.environ, IMB_LIB=str(CHECKED))
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "sanitize_cases.py"), case],
                       env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and f"{case} ok" in r.stdout, r.stdout + r.stderr
    assert "IMB_CHECKED" not in r.stdout
