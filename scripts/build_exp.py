"""Timing-experiment builds (debug only): lib/exp/libhgnn_b200_exp<N>.so compiled
with -DHGNN_EXP=N, where the bits of N drop parts of the tcgen05 backward kernel
(mlp_tc_bwd.cuh: 1 dW staging + MMAs, 2 scratch loads, 4 bias column sums,
8 recompute LayerNorm, 16 input gathers). Results are wrong by construction;
only the kernel times mean something. Select one with HGNN_B200_LIB=<path>."""
import subprocess, sys, concurrent.futures as cf
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
PKG = ROOT / "paper_2410_01657_b200"
sys.path.insert(0, str(PKG))
import build as B  # noqa: E402
out = PKG / "lib" / "exp"
out.mkdir(parents=True, exist_ok=True)
def one(spec):
    """spec: N (HGNN_EXP bits) or name=FLAG1,FLAG2 (extra -D flags, e.g. trunc=HGNN_TF32_RNA=0)"""
    n, flags = (spec.split("=", 1)[0], ["-D" + f for f in spec.split("=", 1)[1].split(",")]) if "=" in spec \
        else (spec, [f"-DHGNN_EXP={spec}"])
    objs = []
    for s in B.SOURCES:
        obj = out / f"{s}.exp{n}.o"
        cmd = [B.NVCC, *B.ARCH, *B.CXXFLAGS, *flags, "-c", str(B.CSRC / s), "-o", str(obj)]
        subprocess.run(cmd, check=True, capture_output=True)
        objs.append(str(obj))
    lib = out / f"libhgnn_b200_exp{n}.so"
    subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", str(lib), *objs, "-lnccl", "-lcudart_static", "-lpthread", "-ldl",
                    "-lrt"], check=True, capture_output=True)
    return lib
with cf.ThreadPoolExecutor(8) as ex:
    for lib in ex.map(one, sys.argv[1:]):
        print(lib)
