"""C-ABI surface (include/hgnn_b200.h): the library loads without a GPU,
exports every declared symbol, and device entry points fail loudly (typed
errors, no silent CPU fallback) when no B200 is present."""
from __future__ import annotations

import ctypes as C
import re
from pathlib import Path

import pytest

import paper_2410_01657_b200 as P
from paper_2410_01657_b200 import _native as N

HEADER = Path(__file__).resolve().parents[1] / "include" / "hgnn_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hgnn_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(P.lib_path())
    syms = declared_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) <= set(N.EXPORTED)


def test_library_is_sm100a_only():
    data = Path(P.lib_path()).read_bytes()
    assert b"sm_100a" in data


def test_config_errors_map_to_reference_exceptions():
    with pytest.raises(P.ConfigError):
        P.build_rank_graph(0, 2, 1, 0)
    with pytest.raises(P.PartitionError):
        P.build_rank_graph(2, 2, 2, 5)


def test_no_gpu_means_loud_failure():
    from conftest import gpu_count
    if gpu_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(P.DeviceError):
        P.Engine(0)
