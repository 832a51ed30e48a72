"""The reference-side C++ binding (integration/hgnn_b200_backend.hpp) compiles
against the reference's own headers, builds hgnn_graph_desc from the
REFERENCE's ReducedGraph/HaloMap identically to our builder, maps status codes
to hgnn::Error subclasses and refuses to run without a GPU. CPU-only; needs the
reference headers and oracle/_ref (this container), skipped elsewhere."""
from __future__ import annotations

import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF_INC = Path("/root/reference/proj/include")
REF_LIB = ROOT / "oracle" / "_ref" / "libhgnn_ref.so"
OUR_LIB = ROOT / "paper_2410_01657_b200" / "lib" / "libhgnn_b200.so"


@pytest.mark.skipif(not (REF_INC.exists() and REF_LIB.exists() and OUR_LIB.exists() and shutil.which("g++")),
                    reason="needs the reference headers, oracle/_ref and the built library")
def test_reference_side_binding(tmp_path):
    exe = tmp_path / "binding_check"
    cmd = ["g++", "-std=c++20", "-O1", f"-I{REF_INC}", f"-I{ROOT / 'include'}", f"-I{ROOT / 'integration'}",
           str(ROOT / "integration" / "binding_check.cpp"), "-o", str(exe), f"-L{REF_LIB.parent}", "-lhgnn_ref",
           f"-L{OUR_LIB.parent}", "-lhgnn_b200", f"-Wl,-rpath,{REF_LIB.parent}", f"-Wl,-rpath,{OUR_LIB.parent}",
           "-fopenmp"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "binding_check: OK" in out.stdout
