"""Per-tensor gradient deviations of the backward implementations vs the oracle."""
import sys
import numpy as np
sys.path.insert(0, "/root/repo")
import oracle as O
from paper_2410_01657_b200 import Engine, GnnConfig, build_rank_graph, init_params, mp_params, mp_layer_slices

E, p, H, M, k = [int(v) for v in (sys.argv[1:] or [3, 5, 64, 2, 5])]
cfg = GnnConfig("t", H, M, k, mode="na2a")
g = build_rank_graph(E, p, 1, 0, "verify")
mp = mp_params(cfg, init_params(cfg, E + H))
rng = np.random.default_rng(3)
x0 = rng.uniform(-1, 1, (g.rows, H)); e0 = rng.uniform(-1, 1, (g.num_edges, H))
dx = rng.uniform(-1, 1, (g.rows, H)); dx[g.num_local:] = 0; de = rng.uniform(-1, 1, (g.num_edges, H))
ref = O.oracle_mp_run([g], H, M, k, "na2a", mp, [x0], [e0], [dx], [de])["grads"][0]
eng = Engine(0)
for impl in (0, 1):
    eng.upload_graph(g); eng.configure(cfg); eng.upload_params(mp)
    eng.set_option("mlp_backward_impl", impl)
    eng.nmp_forward(x0, e0)
    _, _, gr = eng.nmp_backward(dx, de)
    bad = []
    for name, a, b in mp_layer_slices(cfg):
        mag = np.abs(ref[a:b]).max() or 1.0
        r = np.abs(gr[a:b] - ref[a:b]).max() / mag
        if r > 1e-4:
            bad.append((name, b - a, f"{r:.2e}"))
    print("impl", impl, "edges", g.num_edges, "bad tensors:", bad[:40])
