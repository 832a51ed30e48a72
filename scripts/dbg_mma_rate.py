import sys, numpy as np
sys.path.insert(0, "/root/repo")
from paper_2410_01657_b200 import _native as N
blocks = 148
for n, ts, nd in ((64, 1, 1), (64, 1, 2), (128, 1, 1), (128, 1, 2), (256, 1, 1), (64, 0, 1), (128, 0, 1), (256, 0, 1)):
    out = np.zeros(blocks, np.uint64)
    iters = 400
    N.check(N.debug_lib().hgnn_bench_mma(iters, n, ts, nd, blocks, out.ctypes.data))
    cyc = out.astype(np.float64).mean() / (iters * 24)
    flops = 2 * 128 * n * 8
    print(f"N {n:3d} {'TS' if ts else 'SS'} accumulators {nd}: {cyc:7.2f} cycles/MMA, "
          f"{flops / cyc:7.0f} flop/cycle/SM = {flops / cyc * 1.9e9 * 148 / 1e12:6.0f} TF at 1.9 GHz")
for kind, name in ((0, "ex2"), (1, "ffma"), (2, "rsqrt")):
    for threads in (128, 512, 1024):
        out = np.zeros(148, np.uint64)
        iters = 2000
        N.check(N.debug_lib().hgnn_bench_alu(kind, iters, threads, 148, out.ctypes.data))
        cyc = out.astype(np.float64).mean()
        ops = threads * 8 * iters
        print(f"{name:6s} threads/SM {threads:5d}: {ops / cyc:7.1f} ops/cycle/SM")
