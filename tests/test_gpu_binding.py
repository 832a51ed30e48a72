"""The drop-in, end to end on a B200: the reference's own gnn_forward /
gnn_backward (compiled in place into oracle/_ref) against the same step with
its MP-layer loops routed through the reference-side C++ binding
(integration/hgnn_b200_backend.hpp), wired as INTEGRATION.md §2 shows.
Tolerances (in integration/binding_gpu_check.cpp): output and a_sync traces
5e-5, every gradient tensor 2e-4, per tensor normalised by max |reference|.

The binary is built in the container that has the reference headers
(oracle/Makefile, via __graft_entry__.build()); it travels prebuilt, so this
test never reads /root/reference."""
from __future__ import annotations

import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

EXE = Path(__file__).resolve().parents[1] / "oracle" / "_ref" / "binding_gpu_check"


@pytest.mark.skipif(not EXE.exists(), reason="oracle/_ref/binding_gpu_check not built (needs the reference headers)")
def test_reference_training_step_through_the_binding(gpus):
    out = subprocess.run([str(EXE)], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "binding_gpu_check: OK" in out.stdout, out.stdout + out.stderr
