"""In-tree build of the native library (sm_100a) and of the test oracle.

    python paper_2410_01657_b200/build.py            # product .so
    python paper_2410_01657_b200/build.py --oracle   # + oracle/_build and oracle/_ref
(run by path: importing the package would first load the native library)

The product library `paper_2410_01657_b200/lib/libhgnn_b200.so` is compiled
directly with nvcc for `-gencode arch=compute_100a,code=sm_100a` (no JIT, no
torch extension cache) so it travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "lib"
OBJ_DIR = PKG / "build"
LIB = LIB_DIR / "libhgnn_b200.so"
DEBUG_LIB = LIB_DIR / "libhgnn_b200_debug.so"  # tcgen05 self-tests / microbenchmarks (scripts/dbg_*.py only)

NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CXXFLAGS = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-lineinfo", "-Xcompiler", "-Wall"]

SOURCES = ["engine.cu", "model.cu", "host_graph.cpp", "host_params.cpp"]
DEBUG_SOURCES = ["selftest.cu"]
HEADERS = ["common.hpp", "engine_ctx.hpp", "local_group.hpp", "mlp_generic.cuh", "model_kernels.cuh", "graph_kernels.cuh", "mlp_simt.cuh", "mlp_tc.cuh", "mlp_tc_bwd.cuh", "tc_ptx.cuh", "edge_fact.cuh", "encoder_tc.cuh"]


def _newer(src: list[Path], out: Path) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    return any(s.stat().st_mtime > t for s in src)


def _compile(src: Path, obj: Path, deps: list[Path], verbose: bool) -> None:
    if not _newer([src] + deps, obj):
        return
    cmd = [NVCC, *ARCH, *CXXFLAGS, "-c", str(src), "-o", str(obj)]
    if src.suffix == ".cu":
        cmd.insert(1, "-Xptxas=-v" if verbose else "-Xptxas=-warn-spills")
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{res.stdout}\n{res.stderr}")
    if verbose and res.stderr:
        sys.stderr.write(res.stderr)


def build_library(verbose: bool = False, force: bool = False) -> Path:
    OBJ_DIR.mkdir(exist_ok=True)
    LIB_DIR.mkdir(exist_ok=True)
    deps = [CSRC / h for h in HEADERS] + [ROOT / "include" / "hgnn_b200.h"]
    objs = []
    jobs = []
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        for s in SOURCES:
            src = CSRC / s
            obj = OBJ_DIR / (s + ".o")
            if force and obj.exists():
                obj.unlink()
            objs.append(obj)
            jobs.append(ex.submit(_compile, src, obj, deps, verbose))
        for j in jobs:
            j.result()
    if _newer(objs, LIB) or force:
        cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lnccl", "-Xlinker", "-z,defs",
               "-lcudart_static", "-lpthread", "-ldl", "-lrt"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stdout}\n{res.stderr}")
    # debug aids live outside the product ABI, in their own library on top of it
    dobjs = []
    for s in DEBUG_SOURCES:
        obj = OBJ_DIR / (s + ".o")
        _compile(CSRC / s, obj, deps, verbose)
        dobjs.append(obj)
    if _newer(dobjs + [LIB], DEBUG_LIB) or force:
        cmd = [NVCC, *ARCH, "-shared", "-o", str(DEBUG_LIB), *map(str, dobjs), "-L", str(LIB_DIR), "-lhgnn_b200",
               "-Xlinker", "-rpath,$ORIGIN", "-lcudart_static", "-lpthread", "-ldl", "-lrt"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"debug library link failed:\n{res.stdout}\n{res.stderr}")
    return LIB


def build_oracle() -> None:
    """Test infrastructure: oracle/_build (C restatement) and, when the
    reference tree is present in this container, oracle/_ref."""
    res = subprocess.run(["make", "-C", str(ROOT / "oracle"), "-s"], capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{res.stdout}\n{res.stderr}")


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--oracle", action="store_true")
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args()
    print(build_library(verbose=a.verbose, force=a.force))
    if a.oracle:
        build_oracle()


if __name__ == "__main__":
    main()
