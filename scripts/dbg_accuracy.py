"""Per-tensor gradient deviations vs the reference at the bench shape
(H64 k5 M4, 6^3/P5) for the tcgen05 and SIMT paths (debug: which numerics
limit the full-size gradient tolerance)."""
import sys
sys.path.insert(0, "/root/repo")
sys.path.insert(0, "/root/repo/tests")
import numpy as np
import oracle as O
from paper_2410_01657_b200 import Engine, GnnConfig, build_rank_graph, init_params, mp_layer_slices, mp_params
from rank_worker import gid_inputs
E, p, H, M, k = [int(v) for v in (sys.argv[1:6] if len(sys.argv) > 5 else (6, 5, 64, 4, 5))]
cfg = GnnConfig("a", H, M, k, mode="na2a")
mp = mp_params(cfg, init_params(cfg, 0))
g = build_rank_graph(E, p, 1, 0, "verify")
x0, e0, dx = gid_inputs(g, H)
ref = O.ref_mp_run(O.RefGraph(E, p, 1, "verify", features=False), H, M, k, "na2a", mp, [x0], [e0], [dx])
rg = ref.get(0, "mp_grads")
def rel(a, b):
    m = np.abs(b).max()
    return float(np.abs(a - b).max() / (m if m > 0 else 1))
eng = Engine(0)
for name, opts in (("tc", {}), ("simt", {"mlp_forward_impl": 0, "mlp_backward_impl": 0}),
                   ("tc_fwd_simt_bwd", {"mlp_backward_impl": 0}), ("simt_fwd_tc_bwd", {"mlp_forward_impl": 0})):
    eng.upload_graph(g); eng.configure(cfg); eng.upload_params(mp)
    for kk in ("mlp_forward_impl", "mlp_backward_impl"):
        eng.set_option(kk, opts.get(kk, 1))
    xo = eng.nmp_forward(x0, e0)
    dx0, de0, gr = eng.nmp_backward(dx)
    worst = sorted(((rel(gr[a:b], rg[a:b]), n) for n, a, b in mp_layer_slices(cfg)), reverse=True)[:4]
    print(name, "x_out", f"{rel(xo, ref.get(0, 'x_out', M - 1)):.2e}", "dx0", f"{rel(dx0, ref.get(0, 'dx_in', 0)):.2e}",
          "worst grads", [(f"{v:.2e}", n) for v, n in worst], flush=True)
