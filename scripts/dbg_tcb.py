import sys, numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import oracle as O
from paper_2410_01657_b200 import Engine, GnnConfig, build_rank_graph, init_params, mp_params, mp_layer_slices
from test_gpu_parity import random_inputs, rel
for (E, p, k, M) in [(3, 3, 5, 1), (2, 4, 0, 1)]:
    H = 64
    cfg = GnnConfig("tcb", H, M, k, mode="na2a")
    g = build_rank_graph(E, p, 1, 0, "verify")
    mp = mp_params(cfg, init_params(cfg, 21))
    x0, e0, dx, de = random_inputs(g, H, 9)
    eng = Engine(0)
    eng.upload_graph(g); eng.configure(cfg); eng.upload_params(mp)
    eng.nmp_forward(x0, e0)
    dx0, de0, grads = eng.nmp_backward(dx, de)
    ref = O.oracle_mp_run([g], H, M, k, "na2a", mp, [x0], [e0], [dx], [de])
    print("E p k M", E, p, k, M, "dx0", rel(dx0, ref["dx_in"][0][0]), "de0", rel(de0, ref["de_in"][0][0]))
    for name, a, b in mp_layer_slices(cfg):
        r = ref["grads"][0][a:b]; t = grads[a:b]
        e = rel(t, r)
        if e > 1e-4:
            nz = np.count_nonzero(t)
            # row-wise check for weights
            print(f"  {name:28s} rel={e:.3e} nonzero={nz}/{b-a}")
            if name.endswith("w0") or ".w" in name:
                rows = (b - a) // H
                tt = t.reshape(rows, H); rr = r.reshape(rows, H)
                bad = [i for i in range(rows) if np.abs(tt[i]-rr[i]).max() > 1e-4*np.abs(rr).max()]
                print("     bad rows:", bad[:20], "...", len(bad))
        else:
            print(f"  {name:28s} ok {e:.2e}")
    eng.close()
