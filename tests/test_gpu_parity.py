"""GPU parity: the CUDA MP stack (through the C-ABI) against the oracle and
the reference's golden fixtures, on the same inputs.

Tolerances (fp32 device arithmetic vs the fp64 reference), per tensor,
normalised by that tensor's max |reference| (the reference's own metric,
fixtures.hpp:56-70 / harness.cpp:201-212):
  FWD_TOL  layer outputs, aggregates         (stated in DESIGN.md)
  BWD_TOL  input adjoints and weight gradients
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle as O
from paper_2410_01657_b200 import (Engine, GnnConfig, UninitializedError, build_distributed_graph,
                                   build_rank_graph, init_params, load_graph_binary, mp_params,
                                   save_graph_binary)

pytestmark = pytest.mark.gpu

FWD_TOL = 5e-5
BWD_TOL = 2e-4


def rel(test, ref):
    mag = np.abs(ref).max()
    return float(np.abs(test - ref).max() / (mag if mag > 0 else 1.0))


def grad_rel(test, ref, cfg):
    """max over tensors of per-tensor normalised deviation (harness.cpp:201-212)."""
    from paper_2410_01657_b200 import mp_layer_slices
    return max(rel(test[a:b], ref[a:b]) for _, a, b in mp_layer_slices(cfg))


def random_inputs(g, H, seed):
    rng = np.random.default_rng(seed)
    x0 = rng.uniform(-1, 1, (g.rows, H))
    e0 = rng.uniform(-1, 1, (g.num_edges, H))
    dx = rng.uniform(-1, 1, (g.rows, H))
    dx[g.num_local:] = 0.0
    de = rng.uniform(-1, 1, (g.num_edges, H))
    return x0, e0, dx, de


@pytest.fixture(scope="module")
def engine(gpus):
    eng = Engine(0)
    yield eng
    eng.close()


def run_engine(eng, g, cfg, mp, x0, e0, dx, de):
    eng.upload_graph(g)
    eng.configure(cfg)
    eng.upload_params(mp)
    x_out, e_out = eng.nmp_forward(x0, e0, want_e=True)
    traces = {m: {w: eng.trace(m, w) for w in ("a_sync", "x_out", "e_out")} for m in range(cfg.num_mp_layers)}
    dx0, de0, grads = eng.nmp_backward(dx, de)
    return x_out, e_out, traces, dx0, de0, grads


@pytest.mark.parametrize("name", ["mp_e2p2_r1_h8"])
def test_engine_matches_reference_golden(engine, golden_dir, name):
    z = np.load(golden_dir / f"{name}.npz")
    E, p, R, H, M, k, mode, seed = [int(v) for v in z["meta"]]
    cfg = GnnConfig("g", H, M, k, mode={0: "none", 1: "a2a", 2: "na2a"}[mode])
    g = build_rank_graph(E, p, 1, 0, "verify")
    x_out, e_out, _, dx0, de0, grads = run_engine(engine, g, cfg, z["mp_params"], z["r0_x0"], z["r0_e0"],
                                                  z["r0_dx"], z["r0_de"])
    assert rel(x_out, z["r0_x_out"]) < FWD_TOL
    assert rel(e_out, z["r0_e_out"]) < FWD_TOL
    assert rel(dx0, z["r0_dx0"]) < BWD_TOL
    assert rel(de0, z["r0_de0"]) < BWD_TOL
    assert grad_rel(grads, z["r0_grads"], cfg) < BWD_TOL


def test_graph_loaded_from_hgnngrb1_file_runs_identically(engine, golden_dir, tmp_path):
    """A graph read back from an HGNNGRB1 file (num_ranks unknown = 0) drives the
    device path to bitwise the same results as the built graph."""
    z = np.load(golden_dir / "mp_e2p2_r1_h8.npz")
    E, p, R, H, M, k, mode, seed = [int(v) for v in z["meta"]]
    cfg = GnnConfig("g", H, M, k, mode={0: "none", 1: "a2a", 2: "na2a"}[mode])
    g = build_rank_graph(E, p, 1, 0, "verify")
    save_graph_binary(g, tmp_path / "r0.bin")
    h = load_graph_binary(tmp_path / "r0.bin")
    assert h.num_ranks == 0
    args = (cfg, z["mp_params"], z["r0_x0"], z["r0_e0"], z["r0_dx"], z["r0_de"])
    a = run_engine(engine, g, *args)
    b = run_engine(engine, h, *args)
    for u, v in zip((a[0], a[1], a[3], a[4], a[5]), (b[0], b[1], b[3], b[4], b[5])):
        assert u.tobytes() == v.tobytes()


CASES = [  # E, p, H, M, k
    (2, 2, 8, 2, 2), (3, 2, 16, 2, 1), (4, 3, 32, 4, 5), (3, 5, 64, 2, 5), (2, 4, 64, 1, 0), (3, 3, 32, 2, 8),
]


@pytest.mark.parametrize("E,p,H,M,k", CASES)
def test_engine_matches_oracle(engine, E, p, H, M, k):
    cfg = GnnConfig("t", H, M, k, mode="na2a")
    g = build_rank_graph(E, p, 1, 0, "verify")
    rng = np.random.default_rng(E * 1000 + H)
    full = init_params(cfg, E + H)
    mp = mp_params(cfg, full)
    x0, e0, dx, de = random_inputs(g, H, E + 7 * H)
    x_out, e_out, traces, dx0, de0, grads = run_engine(engine, g, cfg, mp, x0, e0, dx, de)
    ref = O.oracle_mp_run([g], H, M, k, "na2a", mp, [x0], [e0], [dx], [de])
    for m in range(M):
        assert rel(traces[m]["a_sync"], ref["a_sync"][0][m]) < FWD_TOL, ("a_sync", m)
        assert rel(traces[m]["x_out"], ref["x_out"][0][m]) < FWD_TOL, ("x_out", m)
        assert rel(traces[m]["e_out"], ref["e_out"][0][m]) < FWD_TOL, ("e_out", m)
    assert rel(x_out, ref["x_out"][0][M - 1]) < FWD_TOL
    assert rel(dx0, ref["dx_in"][0][0]) < BWD_TOL
    assert rel(de0, ref["de_in"][0][0]) < BWD_TOL
    assert grad_rel(grads, ref["grads"][0], cfg) < BWD_TOL


def test_engine_is_deterministic(engine):
    cfg = GnnConfig("t", 32, 2, 5)
    g = build_rank_graph(4, 3, 1, 0)
    mp = mp_params(cfg, init_params(cfg, 5))
    x0, e0, dx, de = random_inputs(g, 32, 3)
    a = run_engine(engine, g, cfg, mp, x0, e0, dx, de)
    b = run_engine(engine, g, cfg, mp, x0, e0, dx, de)
    for u, v in zip((a[0], a[1], a[3], a[4], a[5]), (b[0], b[1], b[3], b[4], b[5])):
        assert u.tobytes() == v.tobytes()


def test_edges_keep_reference_order_at_the_boundary(engine):
    """Device slots are receiver-sorted; host tensors stay in edge-id order."""
    cfg = GnnConfig("t", 8, 1, 0)
    g = build_rank_graph(2, 2, 1, 0)
    mp = np.zeros(mp_params(cfg, init_params(cfg, 0)).size)
    n_e = 3 * 8 * 8 + 8
    # identity-like edge MLP: e' = bias only -> zero weights, bias = 0; x_out = 0
    x0, e0, dx, de = random_inputs(g, 8, 1)
    engine.upload_graph(g)
    engine.configure(cfg)
    engine.upload_params(mp)
    engine.nmp_forward(x0, e0)
    assert engine.trace(0, "e_in").tobytes() == e0.astype(np.float32).astype(np.float64).tobytes()
    assert n_e > 0


def test_device_step_runs_and_is_finite(engine):
    cfg = GnnConfig("t", 64, 2, 5)
    g = build_rank_graph(4, 5, 1, 0)
    engine.upload_graph(g)
    engine.configure(cfg)
    engine.upload_params(mp_params(cfg, init_params(cfg, 0)))
    engine.synthetic_inputs(7)
    engine.step_device()
    gr = engine.grads()
    assert np.isfinite(gr).all() and np.abs(gr).max() > 0
    engine.step_device()
    assert engine.grads().tobytes() == gr.tobytes()


def test_backward_before_forward_is_uninitialized(gpus):
    eng = Engine(0)
    cfg = GnnConfig("t", 8, 1, 1)
    g = build_rank_graph(2, 2, 1, 0)
    eng.upload_graph(g)
    eng.configure(cfg)
    eng.upload_params(mp_params(cfg, init_params(cfg, 0)))
    with pytest.raises(UninitializedError):
        eng.nmp_backward(np.zeros((g.rows, 8)))
    eng.close()


def test_option_values_are_validated(engine):
    """hgnn_set_option: unknown keys and out-of-range values raise ConfigError
    (the engine's state is unchanged)."""
    from paper_2410_01657_b200 import ConfigError
    for key, bad in [("edge_factorized", 2), ("memory_lean", 3), ("encoder_impl", -1), ("tma_gather", 5),
                     ("mlp_backward_split", 0), ("adjoint_presum", 2), ("mlp_backward_impl", 7), ("halo_sm_reserve", 99),
                     ("collective_timeout_ms", 0), ("no_such_option", 1)]:
        with pytest.raises(ConfigError):
            engine.set_option(key, bad)


@pytest.mark.parametrize("H,k", [(32, 5), (64, 5), (64, 0), (32, 2)])
def test_tensor_core_forward_matches_simt_and_oracle(engine, H, k):
    """tcgen05 3xTF32 MLP forward vs the SIMT fp32 kernels vs the fp64 oracle."""
    M = 2
    cfg = GnnConfig("tc", H, M, k, mode="na2a")
    g = build_rank_graph(3, 3, 1, 0, "verify")
    mp = mp_params(cfg, init_params(cfg, 11))
    x0, e0, dx, de = random_inputs(g, H, 5)
    outs = {}
    impls = (0, 1)
    for impl in impls:
        engine.upload_graph(g)
        engine.configure(cfg)
        engine.upload_params(mp)
        engine.set_option("mlp_forward_impl", impl)
        outs[impl] = engine.nmp_forward(x0, e0, want_e=True)
    engine.set_option("mlp_forward_impl", 1)
    ref = O.oracle_mp_run([g], H, M, k, "na2a", mp, [x0], [e0], [dx], [de])
    for impl in impls:
        assert rel(outs[impl][0], ref["x_out"][0][M - 1]) < FWD_TOL, impl
        assert rel(outs[impl][1], ref["e_out"][0][M - 1]) < FWD_TOL, impl


@pytest.mark.parametrize("E,p,k,M,H", [(3, 3, 5, 2, 64), (3, 5, 2, 1, 64), (2, 4, 0, 1, 64), (4, 5, 5, 2, 64),
                                       (3, 3, 5, 2, 32), (4, 3, 3, 2, 32), (3, 4, 0, 1, 32), (5, 3, 5, 4, 32)])
def test_tensor_core_backward_matches_simt_and_oracle(engine, E, p, k, M, H):
    """tcgen05 3xTF32 MLP backward (dX chain + stacked dW MMAs) vs SIMT vs fp64
    oracle; H = 32 runs zero-padded on the 64-wide kernel (mlp_tc_bwd.cuh HL)."""
    cfg = GnnConfig("tcb", H, M, k, mode="na2a")
    g = build_rank_graph(E, p, 1, 0, "verify")
    mp = mp_params(cfg, init_params(cfg, 21))
    x0, e0, dx, de = random_inputs(g, H, 9)
    res = {}
    for impl in (0, 1):
        engine.upload_graph(g)
        engine.configure(cfg)
        engine.upload_params(mp)
        engine.set_option("mlp_backward_impl", impl)
        engine.nmp_forward(x0, e0)
        res[impl] = engine.nmp_backward(dx, de)
    engine.set_option("mlp_backward_impl", 1)
    ref = O.oracle_mp_run([g], H, M, k, "na2a", mp, [x0], [e0], [dx], [de])
    for impl in (0, 1):
        dx0, de0, grads = res[impl]
        assert rel(dx0, ref["dx_in"][0][0]) < BWD_TOL, (impl, rel(dx0, ref["dx_in"][0][0]))
        assert rel(de0, ref["de_in"][0][0]) < BWD_TOL, (impl, rel(de0, ref["de_in"][0][0]))
        assert grad_rel(grads, ref["grads"][0], cfg) < BWD_TOL, (impl, grad_rel(grads, ref["grads"][0], cfg))


@pytest.mark.parametrize("E,p,H,M,k", [(3, 5, 64, 2, 5), (4, 3, 32, 2, 3), (3, 4, 64, 1, 0)])
def test_factorized_edge_path_matches_three_segment_path(engine, E, p, H, M, k):
    """Default edge path (node projections P = x [W0_s | W0_d], one fused
    gather -> MLP -> e' + segmented 1/d aggregate kernel; node-level input
    adjoints) against the 3-segment edge kernels + aggregate + dx gather
    (option edge_factorized = 0), both against the fp64 oracle."""
    cfg = GnnConfig("f", H, M, k, mode="na2a")
    g = build_rank_graph(E, p, 1, 0, "verify")
    mp = mp_params(cfg, init_params(cfg, 31))
    x0, e0, dx, de = random_inputs(g, H, 17)
    res = {}
    for fact in (1, 0):
        engine.upload_graph(g)
        engine.configure(cfg)
        engine.upload_params(mp)
        engine.set_option("edge_factorized", fact)
        x_out, e_out = engine.nmp_forward(x0, e0, want_e=True)
        a0 = engine.trace(0, "a_sync")
        res[fact] = (x_out, e_out, a0) + engine.nmp_backward(dx, de)
    engine.set_option("edge_factorized", 1)
    ref = O.oracle_mp_run([g], H, M, k, "na2a", mp, [x0], [e0], [dx], [de])
    for fact in (1, 0):
        x_out, e_out, a0, dx0, de0, grads = res[fact]
        assert rel(a0, ref["a_sync"][0][0]) < FWD_TOL, fact
        assert rel(x_out, ref["x_out"][0][M - 1]) < FWD_TOL, fact
        assert rel(e_out, ref["e_out"][0][M - 1]) < FWD_TOL, fact
        assert rel(dx0, ref["dx_in"][0][0]) < BWD_TOL, fact
        assert rel(de0, ref["de_in"][0][0]) < BWD_TOL, fact
        assert grad_rel(grads, ref["grads"][0], cfg) < BWD_TOL, fact


def test_memory_lean_plan_matches_standard(engine):
    """The memory-lean plan (no stored last-layer e', de_m written over e_m,
    one recomputed node-projection buffer, dx_node in place of dx, x_M in the
    idle dY buffer — the plan that fits configs[3]'s 2-way split in 180 GB)
    computes bitwise what the standard plan computes."""
    from paper_2410_01657_b200 import SizeError
    H, M, k = 64, 3, 2
    cfg = GnnConfig("lean", H, M, k, mode="na2a")
    g = build_rank_graph(3, 4, 1, 0, "verify")
    mp = mp_params(cfg, init_params(cfg, 41))
    x0, e0, dx, _ = random_inputs(g, H, 23)
    res = {}
    for lean in (0, 1):
        engine.upload_graph(g)
        engine.configure(cfg)
        engine.upload_params(mp)
        engine.set_option("edge_factorized", 1)
        engine.set_option("memory_lean", lean)
        x_out = engine.nmp_forward(x0, e0)
        a1 = engine.trace(1, "a_sync")
        if lean:
            with pytest.raises(SizeError):
                engine.trace(M - 1, "e_out")
        res[lean] = (x_out, a1) + engine.nmp_backward(dx)
        if lean:
            with pytest.raises(UninitializedError):  # the backward consumed the trace storage
                engine.trace(0, "e_in")
    engine.set_option("memory_lean", -1)
    engine.set_option("edge_factorized", 1)  # the default
    for u, v in zip(res[0], res[1]):
        assert u.tobytes() == v.tobytes()
    ref = O.oracle_mp_run([g], H, M, k, "na2a", mp, [x0], [e0], [dx])
    assert rel(res[1][0], ref["x_out"][0][M - 1]) < FWD_TOL
    assert rel(res[1][3], ref["de_in"][0][0]) < BWD_TOL
    assert grad_rel(res[1][4], ref["grads"][0], cfg) < BWD_TOL


@pytest.mark.parametrize("E,p,M,k,fact", [(3, 5, 2, 5, 0), (4, 3, 2, 2, 1), (2, 4, 1, 0, 0)])
def test_tma_gathered_forward_is_bitwise_equal(engine, E, p, M, k, fact):
    """Fused edge forward with TMA tile::gather4 input rows (option tma_gather 1)
    against per-thread 256-bit row loads (0, default): the same arithmetic on the
    same operands, so outputs, aggregates and the backward are bitwise equal."""
    H = 64
    cfg = GnnConfig("tma", H, M, k, mode="na2a")
    g = build_rank_graph(E, p, 1, 0, "verify")
    mp = mp_params(cfg, init_params(cfg, 41))
    x0, e0, dx, de = random_inputs(g, H, 23)
    res = {}
    for tma in (1, 0):
        engine.upload_graph(g)
        engine.configure(cfg)
        engine.upload_params(mp)
        engine.set_option("edge_factorized", fact)
        engine.set_option("tma_gather", tma)
        x_out, e_out = engine.nmp_forward(x0, e0, want_e=True)
        a0 = engine.trace(0, "a_sync")
        res[tma] = (x_out, e_out, a0) + tuple(engine.nmp_backward(dx, de))
    engine.set_option("tma_gather", 0)
    engine.set_option("edge_factorized", 1)  # the default
    for u, v in zip(res[1], res[0]):
        assert np.asarray(u).tobytes() == np.asarray(v).tobytes()
    ref = O.oracle_mp_run([g], H, M, k, "na2a", mp, [x0], [e0], [dx], [de])
    assert rel(res[1][0], ref["x_out"][0][M - 1]) < FWD_TOL


def test_presummed_node_adjoint_is_bitwise_equal(engine):
    """Node-level input adjoint of the factorised path with the segment sums
    precomputed at full occupancy (adjoint_presum 1) against the in-kernel
    gather (0, default): same sums in the same slot order, bitwise equal
    adjoints and gradients; a repeated backward recomputes the node projection
    whose buffer held the sums."""
    H, M, k = 64, 2, 3
    cfg = GnnConfig("ps", H, M, k, mode="na2a")
    g = build_rank_graph(4, 3, 1, 0, "verify")
    mp = mp_params(cfg, init_params(cfg, 51))
    x0, e0, dx, de = random_inputs(g, H, 29)
    res = {}
    for ps in (1, 0):
        engine.upload_graph(g)
        engine.configure(cfg)
        engine.upload_params(mp)
        engine.set_option("edge_factorized", 1)
        engine.set_option("adjoint_presum", ps)
        engine.nmp_forward(x0, e0)
        res[ps] = tuple(engine.nmp_backward(dx, de))
        if ps:
            again = tuple(engine.nmp_backward(dx, de))
            for u, v in zip(res[ps], again):
                assert u.tobytes() == v.tobytes()
    engine.set_option("adjoint_presum", 0)
    for u, v in zip(res[1], res[0]):
        assert u.tobytes() == v.tobytes()
