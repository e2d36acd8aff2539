"""Shared test setup.

Markers: ``gpu`` -- needs a CUDA device (B200); the CPU suite runs with
``-m "not gpu"``.  The reference package is imported from
/root/reference/pkg/src when it exists (this container only); tests that need
it are skipped elsewhere and fall back to the committed golden fixtures.
"""

import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
REF_SRC = Path("/root/reference/pkg/src")
# the unmodified reference installed by bench.py's reference arm recipe
# (pip install --target baseline/_ref); travels to the GPU box
REF_INSTALLED = ROOT / "baseline" / "_ref"
GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")


def _reference_dir():
    for d in (REF_SRC, REF_INSTALLED):
        if (d / "dwmconv" / "__init__.py").exists():
            return d
    return None


def reference_available() -> bool:
    return _reference_dir() is not None


def import_reference():
    d = _reference_dir()
    if d is None:
        pytest.skip("reference package not present; golden fixtures cover this")
    if str(d) not in sys.path:
        sys.path.append(str(d))
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    sys.dont_write_bytecode = True
    import dwmconv
    return dwmconv


@pytest.fixture(scope="session")
def ref():
    return import_reference()


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2002_00552_b200 import _native
    _native.load()
    return torch.device("cuda", 0)
