"""Test configuration.

Markers:
  gpu  -- needs a B200 (run by the driver with `pytest -m gpu` on a GPU box).
Everything unmarked runs on CPU: the oracle against the reference and the
golden fixtures, the host graph builder, the C-ABI surface and the
multi-process (gloo) host logic.
"""
from __future__ import annotations

import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: test needs a CUDA B200 device")
    config.addinivalue_line("markers", "slow: long-running CPU test")
    # The native library and the oracle are built in-tree; build them if a
    # fresh checkout runs the suite directly.
    lib = ROOT / "paper_2410_01657_b200" / "lib" / "libhgnn_b200.so"
    orc = ROOT / "oracle" / "_build" / "liboracle.so"
    if not lib.exists() or not orc.exists():
        import importlib.util
        spec = importlib.util.spec_from_file_location("hgnn_b200_build", ROOT / "paper_2410_01657_b200" / "build.py")
        B = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(B)
        if not lib.exists():
            B.build_library()
        if not orc.exists():
            B.build_oracle()


def gpu_count() -> int:
    from paper_2410_01657_b200 import _native as N
    return N.LIB.hgnn_device_count()


@pytest.fixture(scope="session")
def gpus():
    n = gpu_count()
    if n == 0:
        pytest.skip("no CUDA device visible")
    return n


@pytest.fixture(scope="session")
def golden_dir():
    return GOLDEN
