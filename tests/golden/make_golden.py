"""Regenerates tests/golden/*.npz|json from the REFERENCE implementation.

Runs the reference compiled in place (oracle/_ref/libhgnn_ref.so, built by
`make -C oracle ref` from /root/reference/proj). Only needed when the fixtures
change; the committed fixtures let the test-suite pin the oracle and the graph
builder on machines that have no copy of the reference.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import oracle as O  # noqa: E402

OUT = Path(__file__).resolve().parent

GRAPH_CASES = [  # (E, p, R, strategy, factors)
    (2, 2, 1, "verify", None), (2, 2, 4, "verify", None), (2, 1, 2, "slab", None), (2, 5, 2, "slab", None),
    (4, 2, 8, "verify", None), (4, 3, 8, "verify", None), (6, 2, 6, "block", None), (4, 2, 8, "block", (2, 2, 2)),
    (3, 2, 3, "slab", None), (4, 3, 2, "block", (1, 2, 1)),
    (16, 3, 1, "verify", None), (16, 3, 2, "verify", None),  # BASELINE configs[0] (C1) and configs[1] (C2)
]
GRAPH_FIELDS = ["global_ids", "positions", "edge_src", "edge_dst", "node_degree", "edge_degree", "node_inv_degree",
                "edge_inv_degree", "in_offsets", "in_edges", "out_offsets", "out_edges", "neighbors", "send_offsets",
                "send_rows", "recv_offsets", "recv_rows", "halo_to_local", "sync_local", "sync_offsets", "sync_slots"]

# MP-stack fixtures: (name, E, p, R, H, M, k, mode, seed)
MP_CASES = [
    ("mp_e2p2_r1_h8", 2, 2, 1, 8, 2, 2, "na2a", 11),
    ("mp_e2p2_r4_h8", 2, 2, 4, 8, 2, 2, "na2a", 12),
    ("mp_e2p2_r4_h8_a2a", 2, 2, 4, 8, 1, 1, "a2a", 13),
    ("mp_e2p3_r2_h32", 2, 3, 2, 32, 2, 5, "na2a", 14),
]


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def binary_shas(ref, R) -> list[str]:
    """sha256 of the reference's own save_graph_binary file (io.cpp:200-231) per rank."""
    import tempfile
    out = []
    with tempfile.TemporaryDirectory() as d:
        for r in range(R):
            f = Path(d) / f"r{r}.bin"
            ref.save_binary(r, f)
            out.append(hashlib.sha256(f.read_bytes()).hexdigest())
    return out


def mp_inputs(graph_ranks, H, seed):
    rng = np.random.default_rng(seed)
    x0 = [rng.uniform(-1, 1, (g.num_local + g.num_halo, H)) for g in graph_ranks]
    e0 = [rng.uniform(-1, 1, (g.num_edges, H)) for g in graph_ranks]
    dx = [rng.uniform(-1, 1, (g.num_local + g.num_halo, H)) for g in graph_ranks]
    for r, g in enumerate(graph_ranks):
        dx[r][g.num_local:] = 0.0  # halo rows of the output adjoint are zero (model.cpp:403-409)
    de = [rng.uniform(-1, 1, (g.num_edges, H)) for g in graph_ranks]
    return x0, e0, dx, de


def main() -> None:
    graphs = {}
    for E, p, R, strat, fac in GRAPH_CASES:
        ref = O.RefGraph(E, p, R, strat, fac, features=False)
        key = f"E{E}_p{p}_R{R}_{strat}" + (f"_{fac[0]}{fac[1]}{fac[2]}" if fac else "")
        graphs[key] = {"E": E, "p": p, "R": R, "strategy": strat, "factors": fac,
                       "ranks": [{**{f: sha(getattr(g, f)) for f in GRAPH_FIELDS},
                                  "num_local": g.num_local, "num_halo": g.num_halo, "num_edges": g.num_edges,
                                  "max_buffer_rows": g.max_buffer_rows,
                                  "binary_sha256": b} for g, b in zip(ref.ranks, binary_shas(ref, R))]}
    params = {}
    for H, M, k in [(8, 4, 2), (32, 4, 5), (64, 4, 5)]:
        for seed in (0, 3):
            p = O.ref_init_params(H, M, k, seed)
            params[f"H{H}_M{M}_k{k}_s{seed}"] = {"count": int(p.size), "sha256": sha(p)}
    losses = {}
    for E, p, R in [(2, 2, 1), (2, 2, 2), (2, 2, 4), (2, 2, 8), (4, 3, 2)]:
        ref = O.RefGraph(E, p, R, "verify", features=True)
        for mode in ("na2a", "none"):
            run = O.ref_run(ref, 8, 4, 2, mode, seed=0)
            losses[f"small_E{E}_p{p}_R{R}_{mode}"] = run.loss
    json.dump({"graphs": graphs, "params": params, "losses": losses,
               "c1_large_loss_seed0": 1670973.5417324416},
              open(OUT / "reference_hashes.json", "w"), indent=1, sort_keys=True)

    if "--hashes-only" in sys.argv:
        return
    for name, E, p, R, H, M, k, mode, seed in MP_CASES:
        ref = O.RefGraph(E, p, R, "verify", features=False)
        n_mp = O.ref_lib().ref_mp_param_count(H, M, k)
        rng = np.random.default_rng(seed + 1000)
        mp = rng.uniform(-0.4, 0.4, n_mp)
        x0, e0, dx, de = mp_inputs(ref.ranks, H, seed)
        run = O.ref_mp_run(ref, H, M, k, mode, mp, x0, e0, dx, de)
        arrs = {"mp_params": mp, "meta": np.array([E, p, R, H, M, k, O.MODES[mode], seed])}
        for r in range(R):
            arrs[f"r{r}_x0"], arrs[f"r{r}_e0"], arrs[f"r{r}_dx"], arrs[f"r{r}_de"] = x0[r], e0[r], dx[r], de[r]
            arrs[f"r{r}_x_out"] = run.get(r, "x_out", M - 1)
            arrs[f"r{r}_e_out"] = run.get(r, "e_out", M - 1)
            arrs[f"r{r}_a_sync0"] = run.get(r, "a_sync", 0)
            arrs[f"r{r}_dx0"] = run.get(r, "dx_in", 0)
            arrs[f"r{r}_de0"] = run.get(r, "de_in", 0)
            arrs[f"r{r}_grads"] = run.get(r, "mp_grads")
        np.savez_compressed(OUT / f"{name}.npz", **arrs)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
