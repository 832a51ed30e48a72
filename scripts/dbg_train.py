import sys, numpy as np
sys.path.insert(0, "/root/repo")
from paper_2410_01657_b200 import Engine, GnnConfig, build_rank_graph, init_params
E = int(sys.argv[1]) if len(sys.argv) > 1 else 16
cfg = GnnConfig("t", 64, 4, 5)
g = build_rank_graph(E, 5, 1, 0)
eng = Engine(0); eng.upload_graph(g); eng.configure(cfg); eng.model_configure(3, 7, 3)
eng.model_params_upload(init_params(cfg, 0))
rng = np.random.default_rng(0)
eng.model_set_data(np.sin(g.global_ids[:, None] * 0.1 + np.arange(3)), rng.uniform(-1, 1, (g.num_edges, 7)), None)
eng.train_step()
eng.kernel_timing(True)
eng.train_step()
print({k: round(v[0], 3) for k, v in eng.kernel_times().items()})
