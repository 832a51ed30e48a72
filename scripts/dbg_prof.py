import sys, numpy as np, time
sys.path.insert(0, "/root/repo")
from paper_2410_01657_b200 import Engine, GnnConfig, build_rank_graph, init_params, mp_params, _native as N
H, M, k = 64, 1, 5
for E in ((int(sys.argv[1]),) if len(sys.argv) > 1 else (8,)):
    cfg = GnnConfig("p", H, M, k, mode="na2a")
    g = build_rank_graph(E, 5, 1, 0)
    eng = Engine(0); eng.upload_graph(g); eng.configure(cfg); eng.upload_params(mp_params(cfg, init_params(cfg, 0)))
    if len(sys.argv) > 2:
        eng.set_option("edge_factorized", int(sys.argv[2]))
    eng.synthetic_inputs(1)
    eng.step_device(); eng.step_device()
    eng.set_option("bwd_profile", 1)
    eng.kernel_timing(True)
    eng.step_device()
    kt = eng.kernel_times()
    out = np.zeros(64, np.uint64)
    N.check(N.LIB.hgnn_debug_profile(eng._h, out.ctypes.data))
    names = ["total", "w_full", "a_full", "st_full", "dw_empty", "fwd_phase", "dw_job", "mma3_bwd"]
    print("E", E, "edges", g.num_edges, {kk: round(v[0], 3) for kk, v in kt.items()})
    for w, base in (("edge", 0), ("node", 16)):
        tot = out[base] or 1
        print(w, {names[i]: f"{out[base+i]/tot:.3f}" for i in range(8)}, "total Mcyc/CTA", out[base] / 148 / 1e6)
    en = ["epi_total", "recompute", "flush", "stage", "write_db", "wait_dx", "ln_bwd", "input_phase"]
    for w, base in (("edge", 0), ("node", 16)):
        tot = out[base + 8] or 1
        print(w, "epilogue", {en[i]: f"{out[base+8+i]/tot:.3f}" for i in range(8)}, "Mcyc/CTA", out[base + 8] / 148 / 1e6)
    fn = ["iss_total", "iss_wait_a", "iss_wait_w", "iss_mma", "epi_total", "epi_wait_d", "epi_wait_aempty", "epi_signal", "epi_ld", "epi_math", "epi_store_a"]
    for w, base in (("fwd edge", 32), ("fwd node", 48)):
        print(w, {fn[i]: f"{out[base+i]/max(out[base + (0 if i < 4 else 4)],1):.3f}" for i in range(11)},
              "iss Mcyc/CTA", out[base] / 148 / 1e6, "epi Mcyc/CTA", out[base + 4] / 148 / 1e6)
    eng.set_option("bwd_profile", 0)
    for impl in (0, 1):
        eng.set_option("mlp_backward_impl", impl)
        eng.step_device()
        eng.step_device()
        kt = eng.kernel_times()
        print("bwd_impl", impl, {kk: round(v[0], 3) for kk, v in kt.items()})
