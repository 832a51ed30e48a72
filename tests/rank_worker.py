"""One rank of a multi-GPU parity run (launched by test_gpu_multirank.py).

Inputs are functions of global ids only, so coincident nodes / duplicated
edges carry identical values on every rank, as in the reference harness.
"""
from __future__ import annotations

import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2410_01657_b200 import Engine, GnnConfig, build_rank_graph, init_params, mp_params  # noqa: E402


def gid_inputs(g, H):
    cols = np.arange(H)[None, :]
    x0 = np.sin(0.37 * g.global_ids[:, None] + 0.5 * cols)
    key = (g.global_ids[g.edge_src] * 7919 + g.global_ids[g.edge_dst]).astype(np.float64)
    e0 = np.cos(1e-3 * key[:, None] + 0.3 * cols)
    dx = 1e-2 * np.cos(0.21 * g.global_ids[:, None] - 0.7 * cols)
    # consistent output adjoint: coincident copies carry 1/d of the seed
    # (consistent_loss_backward, model.cpp:493-499)
    dx[:g.num_local] *= g.node_inv_degree[:, None]
    dx[g.num_local:] = 0.0
    return x0, e0, dx


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rank", type=int)
    ap.add_argument("--R", type=int)
    ap.add_argument("--uid")
    ap.add_argument("--E", type=int)
    ap.add_argument("--p", type=int)
    ap.add_argument("--H", type=int)
    ap.add_argument("--M", type=int)
    ap.add_argument("--k", type=int)
    ap.add_argument("--mode")
    ap.add_argument("--out")
    ap.add_argument("--model", action="store_true", help="full model (encoders, loss, Adam) on TGV features")
    ap.add_argument("--mismatch", action="store_true",
                    help="collective_check on; rank 1 runs another exchange mode: both ranks must raise")
    a = ap.parse_args()
    if a.model:
        return model_main(a)
    if a.mismatch:
        return mismatch_main(a)
    cfg = GnnConfig("w", a.H, a.M, a.k, mode=a.mode)
    g = build_rank_graph(a.E, a.p, a.R, a.rank, "verify")
    eng = Engine(a.rank, a.rank, a.R, bytes.fromhex(a.uid))
    eng.upload_graph(g)
    eng.configure(cfg)
    eng.upload_params(mp_params(cfg, init_params(cfg, 0)))
    x0, e0, dx = gid_inputs(g, a.H)
    x_out, e_out = eng.nmp_forward(x0, e0, want_e=True)
    a_sync0 = eng.trace(0, "a_sync")
    dx0, de0, grads = eng.nmp_backward(dx)
    x_out2 = eng.nmp_forward(x0, e0)
    eng.set_option("halo_overlap", 0)  # the serial schedule (exchange between aggregation and node update)
    x_ser, e_ser = eng.nmp_forward(x0, e0, want_e=True)
    dx0_s, de0_s, grads_s = eng.nmp_backward(dx)
    np.savez(a.out, x_out=x_out, e_out=e_out, a_sync0=a_sync0, dx0=dx0, de0=de0, grads=grads, x_out2=x_out2,
             x_serial=x_ser, e_serial=e_ser, dx0_serial=dx0_s, de0_serial=de0_s, grads_serial=grads_s,
             halo_bytes=eng.halo_bytes())
    eng.close()


def mismatch_main(a):
    """A mismatched collective sequence over NCCL raises CollectiveError on every
    rank (debug option collective_check) instead of deadlocking."""
    from paper_2410_01657_b200 import CollectiveError
    mode = a.mode if a.rank == 0 else ("a2a" if a.mode == "na2a" else "na2a")
    cfg = GnnConfig("w", a.H, a.M, a.k, mode=mode)
    g = build_rank_graph(a.E, a.p, a.R, a.rank, "verify")
    eng = Engine(a.rank, a.rank, a.R, bytes.fromhex(a.uid))
    eng.upload_graph(g)
    eng.configure(cfg)
    eng.upload_params(mp_params(cfg, init_params(cfg, 0)))
    eng.set_option("collective_check", 1)
    eng.set_option("collective_timeout_ms", 20000)
    x0, e0, _ = gid_inputs(g, a.H)
    msg = ""
    try:
        eng.nmp_forward(x0, e0)
    except CollectiveError as ex:
        msg = str(ex)
    np.savez(a.out, raised=np.array(bool(msg)), msg=np.array(msg))
    eng.close()


def model_main(a):
    """compute_gradients + 3 train steps on the reference's TGV features of this rank."""
    import oracle as O
    cfg = GnnConfig("w", a.H, a.M, a.k, mode=a.mode)
    g = build_rank_graph(a.E, a.p, a.R, a.rank, "verify")
    rg = O.RefGraph(a.E, a.p, a.R, "verify").ranks[a.rank]
    eng = Engine(a.rank, a.rank, a.R, bytes.fromhex(a.uid))
    eng.upload_graph(g)
    eng.configure(cfg)
    eng.model_configure(3, 7, 3)
    eng.model_params_upload(O.ref_init_params(a.H, a.M, a.k, 11))
    eng.model_set_data(rg.node_features, rg.edge_features, None)
    loss, grads, y = eng.compute_gradients()
    steps = [eng.train_step(lr=1e-3) for _ in range(3)]
    np.savez(a.out, loss=loss, grads=grads, steps=np.array(steps), params=eng.model_params())
    eng.close()


if __name__ == "__main__":
    main()
