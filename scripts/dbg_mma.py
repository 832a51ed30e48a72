import sys, numpy as np, ctypes as C
sys.path.insert(0, "/root/repo")
from paper_2410_01657_b200 import _native as N
rng = np.random.default_rng(0)
A = rng.integers(-3, 4, (128, 32)).astype(np.float32)
B = rng.integers(-3, 4, (32, 128)).astype(np.float32)
ref = A.astype(np.float64) @ B.astype(np.float64)
for mode in (0, 2, 6, 7, 8):
    D = np.zeros((128, 128), np.float32)
    st = N.debug_lib().hgnn_selftest_mma(mode, A.ctypes.data, B.ctypes.data, D.ctypes.data)
    err = np.abs(D - ref).max()
    print("mode", mode, "status", st, "max err", err, "nonzero", np.count_nonzero(D), "D[0,:4]", D[0,:4], "ref", ref[0,:4])
    if err > 0:
        # find structure
        for name, cand in [("A^T B?", None)]:
            pass

# also try swapped lbo/sbo interpretation for the swizzled case by checking structure of mode 6 output
