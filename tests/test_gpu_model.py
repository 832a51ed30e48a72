"""Model level on the GPU: encoders + MP stack + decoder,
consistent loss, gradient averaging and Adam against the reference itself
(oracle/_ref: compute_gradients via ref_run, train via ref_train), on the
reference's own TGV features and init_params weights.

Tolerances (fp32 device vs fp64 reference): loss and decoder output 5e-5
relative; gradients per tensor normalised by the tensor's max |ref| 2e-4 (the
same metric and bounds as tests/test_gpu_parity.py); Adam trajectories: losses
1e-4 relative per step, parameter updates (p_T - p_0) per tensor 1e-2 of the
tensor's largest update (Adam's normalised step amplifies fp32 noise in
gradients that are ~0).
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle as O
from paper_2410_01657_b200 import Engine, GnnConfig, build_rank_graph, model_slices

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not O.ref_available(), reason="needs the reference compiled in place (oracle/_ref)")]

LOSS_TOL = 5e-5
BWD_TOL = 2e-4


def rel(a, b):
    m = np.abs(b).max()
    return float(np.abs(a - b).max() / (m if m > 0 else 1.0))


def setup(eng, E, p, H, M, k, seed):
    cfg = GnnConfig("model", H, M, k, mode="na2a")
    ref_g = O.RefGraph(E, p, 1, "verify")
    g = build_rank_graph(E, p, 1, 0, "verify")
    eng.upload_graph(g)
    eng.configure(cfg)
    n = eng.model_configure(3, 7, 3)
    params = O.ref_init_params(H, M, k, seed)
    assert n == params.size
    eng.model_params_upload(params)
    r0 = ref_g.ranks[0]
    eng.model_set_data(r0.node_features, r0.edge_features, None)
    return cfg, ref_g, params


@pytest.fixture(scope="module")
def engine(gpus):
    eng = Engine(0)
    yield eng
    eng.close()


@pytest.mark.parametrize("E,p,M,k", [(2, 3, 2, 2), (3, 2, 1, 5), (6, 3, 2, 5)])
def test_compute_gradients_matches_reference(engine, E, p, M, k):
    H, seed = 64, 3
    cfg, ref_g, _ = setup(engine, E, p, H, M, k, seed)
    loss, grads, y = engine.compute_gradients()
    ref = O.ref_run(ref_g, H, M, k, "na2a", seed=seed)
    assert abs(loss - ref.loss) / abs(ref.loss) < LOSS_TOL, (loss, ref.loss)
    assert rel(y, ref.get(0, "y")) < LOSS_TOL
    ref_grads = ref.get(0, "all_grads")
    worst = max((rel(grads[a:b], ref_grads[a:b]), name) for name, a, b in model_slices(cfg))
    assert worst[0] < BWD_TOL, worst


@pytest.mark.parametrize("E,p,M,k", [(3, 2, 1, 5), (6, 3, 2, 3)])
def test_tensor_core_encoders_match_simt(gpus, E, p, M, k):
    """encoder_impl 1 (tcgen05 encoders and decoder, encoder_tc.cuh) against 0 (fp32
    SIMT, mlp_generic.cuh) on the same inputs: loss, output and every
    gradient tensor (incl. W_skip and the encoders' LayerNorm gamma, beta)."""
    out = {}
    for impl in (0, 1):
        eng = Engine(0)
        eng.set_option("encoder_impl", impl)
        cfg, _, _ = setup(eng, E, p, 64, M, k, 11)
        out[impl] = eng.compute_gradients()
        eng.close()
    (l0, g0, y0), (l1, g1, y1) = out[0], out[1]
    assert abs(l1 - l0) / abs(l0) < LOSS_TOL, (l0, l1)
    assert rel(y1, y0) < LOSS_TOL
    worst = max((rel(g1[a:b], g0[a:b]), name) for name, a, b in model_slices(cfg))
    assert worst[0] < BWD_TOL, worst


def test_train_steps_match_reference(engine):
    E, p, H, M, k, seed, steps, lr = 2, 3, 64, 2, 2, 5, 4, 1e-3
    cfg, ref_g, p0 = setup(engine, E, p, H, M, k, seed)
    losses = [engine.train_step(lr=lr) for _ in range(steps)]
    ref_losses, ref_p = O.ref_train(ref_g, H, M, k, "na2a", seed, steps, lr=lr)
    for a, b in zip(losses, ref_losses):
        assert abs(a - b) / abs(b) < 1e-4, (losses, list(ref_losses))
    ours = engine.model_params()
    for name, a, b in model_slices(cfg):
        d_ref, d_ours = ref_p[a:b] - p0[a:b], ours[a:b] - p0[a:b]
        assert rel(d_ours, d_ref) < 1e-2, name


def test_training_reduces_loss_and_is_deterministic(gpus):
    def run():
        eng = Engine(0)
        setup(eng, 2, 3, 64, 1, 1, 7)
        out = [eng.train_step(lr=1e-3) for _ in range(5)]
        p = eng.model_params()
        eng.close()
        return out, p
    l1, p1 = run()
    l2, p2 = run()
    assert l1 == l2 and p1.tobytes() == p2.tobytes()
    assert l1[-1] < l1[0]
