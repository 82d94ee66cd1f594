import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on the GPU box)")


def _ensure_built():
    lib = ROOT / "paper_1507_01265_b200" / "libimb_b200.so"
    if not lib.exists():
        import subprocess
        subprocess.run(["make", "-s", "-j8", "-C", str(ROOT / "paper_1507_01265_b200" / "csrc")],
                       check=True)


_ensure_built()


@pytest.fixture(scope="session")
def imb():
    import paper_1507_01265_b200 as pkg
    return pkg


@pytest.fixture(scope="session")
def orc():
    from oracle import oracle as o
    o.orc()
    return o
