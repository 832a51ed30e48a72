import sys, numpy as np
sys.path.insert(0, "/root/repo")
from paper_2410_01657_b200 import _native as N
rng = np.random.default_rng(0)
A = rng.integers(-3, 4, (128, 32)).astype(np.float32)
B = rng.integers(-3, 4, (32, 128)).astype(np.float32)
ref = A[:64].astype(np.float64) @ B[:, :64].astype(np.float64)  # 64 x 64
for mode in (9, 10):
    D = np.zeros((128, 128), np.float32)
    st = N.debug_lib().hgnn_selftest_mma(mode, A.ctypes.data, B.ctypes.data, D.ctypes.data)
    print("mode", mode, "status", st, "nonzero lanes", np.nonzero(np.abs(D).sum(1))[0][[0, -1]] if np.count_nonzero(D) else None,
          "nonzero cols", np.nonzero(np.abs(D).sum(0))[0][[0, -1]] if np.count_nonzero(D) else None)
    # locate each reference row
    where = []
    for i in range(64):
        hit = [l for l in range(128) if np.array_equal(D[l, :64], ref[i])]
        where.append(hit[0] if hit else -1)
    print("  row -> lane:", where[:8], "...", where[56:], "all found:", all(w >= 0 for w in where))
    if not all(w >= 0 for w in where):
        print("  D[0,:8]", D[0, :8], "ref[0,:8]", ref[0, :8], "D[32,:8]", D[32, :8])
