import sys, numpy as np
sys.path.insert(0, "/root/repo")
from paper_2410_01657_b200 import Engine, GnnConfig, build_rank_graph, init_params, mp_params, _native as N
H, M, k = 64, 1, 5
for E in (8,):
    cfg = GnnConfig("p", H, M, k, mode="na2a")
    g = build_rank_graph(E, 5, 1, 0)
    eng = Engine(0); eng.upload_graph(g); eng.configure(cfg); eng.upload_params(mp_params(cfg, init_params(cfg, 0)))
    eng.synthetic_inputs(1)
    for impl in (1,):
        eng.set_option("mlp_forward_impl", impl)
        eng.step_device()
        eng.kernel_timing(True)
        k0 = eng.kernel_times()
        for _ in range(3):
            eng.step_device()
        k1 = eng.kernel_times()
        kt = {n: (k1[n][0] - k0[n][0], 0) for n in k1}
        eng.kernel_timing(False)
        eng.set_option("bwd_profile", 1)
        eng.step_device()
        out = np.zeros(64, np.uint64)
        N.check(N.LIB.hgnn_debug_profile(eng._h, out.ctypes.data))
        eng.set_option("bwd_profile", 0)
        fn = ["iss_total", "iss_wait_a", "iss_wait_w", "iss_mma", "epi_total", "epi_wait_d", "epi_wait_aempty", "epi_signal", "epi_ld", "epi_math", "epi_store_a", "epi_input_phase", "epi_output_phase"]
        base = 32
        print("E", E, "impl", impl, "edge_fwd ms", round(kt["edge_fwd"][0] / 3, 3), "node_fwd", round(kt["node_fwd"][0] / 3, 3),
              {fn[i]: f"{out[base+i]/max(out[base + (0 if i < 4 else 4)],1):.3f}" for i in range(13)})
    eng.close()
