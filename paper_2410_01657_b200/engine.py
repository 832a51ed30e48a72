"""Per-rank device engine: the B200 drop-in for the reference's MP stack.

Mirrors the reference interface of the hot path (model.hpp:98-116):
  Engine.nmp_forward   ~ gnn_forward's layer loop (M x nmp_layer_forward)
  Engine.nmp_backward  ~ gnn_backward's layer loop (M x nmp_layer_backward)
  Engine.trace         ~ NmpLayerTrace (x_in, e_in, a_sync) plus layer outputs
One Engine per rank / GPU (one process per GPU under torchrun); ranks share an
NCCL communicator whose unique id is broadcast by the caller.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .graph import RankGraph
from .params import GnnConfig


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    N.check(N.LIB.hgnn_nccl_unique_id(buf))
    return bytes(buf)


def _f64(a: np.ndarray | None, shape=None):
    if a is None:
        return None, None
    a = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None and a.shape != shape and a.size != int(np.prod(shape)):
        raise N.ShapeError(f"expected shape {shape}, got {a.shape}")
    return a, a.ctypes.data_as(N.f64p)


def _out(a: np.ndarray, shape) -> np.ndarray:
    """Caller-provided output buffer: must be fp64, C-contiguous, right size."""
    if a.dtype != np.float64 or not a.flags.c_contiguous or a.size != int(np.prod(shape)):
        raise N.ShapeError(f"output buffer must be C-contiguous float64 of shape {shape}, got {a.dtype} {a.shape}")
    return a.reshape(shape)


class LocalGroup:
    """In-process rank group (the reference's RankRuntime, comm.cpp:35-93): R
    Engines, one per rank, driven by R host threads of this process (one GPU or
    several). Every collective rendezvous checks that all ranks post the same
    collective in the same order (CollectiveError otherwise, comm.cpp:168-208)
    and times out instead of hanging."""

    def __init__(self, num_ranks: int, timeout_ms: int | None = None):
        self._h = C.c_void_p()
        N.check(N.LIB.hgnn_local_group_create(num_ranks, C.byref(self._h)))
        self.num_ranks = num_ranks
        if timeout_ms is not None:
            N.check(N.LIB.hgnn_local_group_set_timeout(self._h, int(timeout_ms)))

    def engine(self, rank: int, device: int = 0) -> "Engine":
        return Engine(device, rank, self.num_ranks, group=self)

    def run(self, body, engines):
        """Runs body(engine) on one thread per rank (RankRuntime::run); returns
        the per-rank results and re-raises the first failure after all joined."""
        import threading
        out, err = [None] * len(engines), [None] * len(engines)

        def work(r):
            try:
                out[r] = body(engines[r])
            except BaseException as e:  # noqa: BLE001
                err[r] = e
        ts = [threading.Thread(target=work, args=(r,)) for r in range(len(engines))]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        for e in err:
            if e is not None:
                raise e
        return out

    def close(self) -> None:
        if self._h:
            N.check(N.LIB.hgnn_local_group_destroy(self._h))
            self._h = C.c_void_p()


class Engine:
    def __init__(self, device: int = 0, rank: int = 0, num_ranks: int = 1, uid: bytes | None = None,
                 group: LocalGroup | None = None):
        self._h = C.c_void_p()
        if group is not None:
            N.check(N.LIB.hgnn_ctx_create_local(device, rank, group._h, C.byref(self._h)))
            num_ranks = group.num_ranks
        else:
            uid_buf = (C.c_uint8 * 128).from_buffer_copy(uid) if uid is not None else None
            N.check(N.LIB.hgnn_ctx_create(device, rank, num_ranks, uid_buf, C.byref(self._h)))
        self.rank, self.num_ranks, self.device = rank, num_ranks, device
        self.graph: RankGraph | None = None
        self.cfg: GnnConfig | None = None

    def close(self) -> None:
        if self._h:
            N.check(N.LIB.hgnn_ctx_destroy(self._h))
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream_ptr(self) -> int:
        return N.LIB.hgnn_ctx_stream(self._h) or 0

    # ---- setup -----------------------------------------------------------
    def upload_graph(self, g: RankGraph) -> None:
        d = g.desc()
        N.check(N.LIB.hgnn_graph_upload(self._h, C.byref(d)))
        self.graph = g

    def configure(self, cfg: GnnConfig) -> None:
        N.check(N.LIB.hgnn_configure(self._h, cfg.hidden_dim, cfg.num_mp_layers, cfg.mlp_hidden_layers,
                                     N.MODES[cfg.mode]))
        self.cfg = cfg

    def upload_params(self, mp_params: np.ndarray) -> None:
        a, p = _f64(mp_params)
        N.check(N.LIB.hgnn_params_upload(self._h, p, a.size))

    # ---- MP stack ----------------------------------------------------------
    def nmp_forward(self, x0: np.ndarray, e0: np.ndarray, want_e: bool = False, out=None):
        """Runs the M consistent NMP layers; returns x_M (rows x H) [and e_M].
        out: optional preallocated (x_M, e_M or None) fp64 C-contiguous arrays
        (e.g. pinned host memory), written in place."""
        g, H = self.graph, self.cfg.hidden_dim
        x, xp = _f64(x0, (g.rows, H))
        e, ep = _f64(e0, (g.num_edges, H))
        if out is not None:
            xo, eo = _out(out[0], (g.rows, H)), (_out(out[1], (g.num_edges, H)) if want_e else None)
        else:
            xo = np.empty((g.rows, H))
            eo = np.empty((g.num_edges, H)) if want_e else None
        N.check(N.LIB.hgnn_mp_forward(self._h, xp, ep, xo.ctypes.data_as(N.f64p),
                                      eo.ctypes.data_as(N.f64p) if want_e else None))
        return (xo, eo) if want_e else xo

    def nmp_backward(self, dx: np.ndarray, de: np.ndarray | None = None, out=None):
        """Adjoint of the MP stack; returns (dx0, de0, mp_grads).
        out: optional preallocated (dx0, de0, grads) fp64 arrays, written in place."""
        g, H = self.graph, self.cfg.hidden_dim
        d, dp = _f64(dx, (g.rows, H))
        e, epp = _f64(de, (g.num_edges, H))
        n_par = self.cfg.num_mp_layers * (_mlp(3 * H, H, self.cfg.mlp_hidden_layers)
                                          + _mlp(2 * H, H, self.cfg.mlp_hidden_layers))
        if out is not None:
            dx0, de0, grads = _out(out[0], (g.rows, H)), _out(out[1], (g.num_edges, H)), _out(out[2], (n_par,))
        else:
            dx0 = np.empty((g.rows, H))
            de0 = np.empty((g.num_edges, H))
            grads = np.empty(n_par)
        N.check(N.LIB.hgnn_mp_backward(self._h, dp, epp, dx0.ctypes.data_as(N.f64p), de0.ctypes.data_as(N.f64p),
                                       grads.ctypes.data_as(N.f64p)))
        return dx0, de0, grads

    def trace(self, layer: int, which: str) -> np.ndarray:
        g, H = self.graph, self.cfg.hidden_dim
        sel = {"x_in": N.TRACE_X_IN, "e_in": N.TRACE_E_IN, "a_sync": N.TRACE_A_SYNC, "x_out": N.TRACE_X_OUT,
               "e_out": N.TRACE_E_OUT}[which]
        n = g.num_edges if which.startswith("e") else g.rows
        out = np.empty((n, H))
        N.check(N.LIB.hgnn_get_trace(self._h, layer, sel, out.ctypes.data_as(N.f64p)))
        return out

    # ---- model level: encoders + MP stack + decoder, loss, Adam --
    def model_configure(self, in_node_dim: int = 3, in_edge_dim: int = 7, out_dim: int = 3) -> int:
        N.check(N.LIB.hgnn_model_configure(self._h, in_node_dim, in_edge_dim, out_dim))
        self.model_dims = (in_node_dim, in_edge_dim, out_dim)
        return int(N.LIB.hgnn_model_param_count(self._h))

    def model_params_upload(self, params: np.ndarray) -> None:
        a, p = _f64(params)
        N.check(N.LIB.hgnn_model_params_upload(self._h, p, a.size))

    def model_params(self) -> np.ndarray:
        out = np.empty(int(N.LIB.hgnn_model_param_count(self._h)))
        N.check(N.LIB.hgnn_model_params_download(self._h, out.ctypes.data_as(N.f64p)))
        return out

    def model_set_data(self, node_features: np.ndarray, edge_features: np.ndarray, target=None) -> None:
        g = self.graph
        fx, fe, fy = self.model_dims
        _, xp = _f64(node_features, (g.rows, fx))
        _, ep = _f64(edge_features, (g.num_edges, fe))
        _, tp = _f64(target, (g.num_local, fy))
        N.check(N.LIB.hgnn_model_set_data(self._h, xp, ep, tp))

    def compute_gradients(self):
        """compute_gradients (model.cpp:556-567): (loss, rank-averaged grads, y)."""
        g = self.graph
        loss = C.c_double()
        grads = np.empty(int(N.LIB.hgnn_model_param_count(self._h)))
        y = np.empty((g.num_local, self.model_dims[2]))
        N.check(N.LIB.hgnn_compute_gradients(self._h, C.byref(loss), grads.ctypes.data_as(N.f64p),
                                             y.ctypes.data_as(N.f64p)))
        return loss.value, grads, y

    def train_step(self, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8) -> float:
        """train_step (model.cpp:569-579): loss before the Adam update."""
        loss = C.c_double()
        N.check(N.LIB.hgnn_train_step(self._h, lr, beta1, beta2, eps, C.byref(loss)))
        return loss.value

    # ---- device-resident step (benchmark) ---------------------------------
    def synthetic_inputs(self, seed: int = 0) -> None:
        N.check(N.LIB.hgnn_synthetic_inputs(self._h, seed))

    def set_inputs(self, x0, e0, dx) -> None:
        _, xp = _f64(x0)
        _, ep = _f64(e0)
        _, dp = _f64(dx)
        N.check(N.LIB.hgnn_set_inputs(self._h, xp, ep, dp))

    def step_device(self) -> None:
        N.check(N.LIB.hgnn_mp_step_device(self._h))

    def grads(self) -> np.ndarray:
        H, k = self.cfg.hidden_dim, self.cfg.mlp_hidden_layers
        out = np.empty(self.cfg.num_mp_layers * (_mlp(3 * H, H, k) + _mlp(2 * H, H, k)))
        N.check(N.LIB.hgnn_get_grads(self._h, out.ctypes.data_as(N.f64p)))
        return out

    def set_option(self, key: str, value: int) -> None:
        N.check(N.LIB.hgnn_set_option(self._h, key.encode(), int(value)))

    # ---- instrumentation ---------------------------------------------------
    def kernel_timing(self, enable: bool) -> None:
        N.check(N.LIB.hgnn_kernel_timing(self._h, int(enable)))

    def kernel_times(self) -> dict[str, tuple[float, int]]:
        out = {}
        for i, name in enumerate(N.KERNEL_CLASSES):
            t, n = C.c_double(), C.c_int64()
            N.check(N.LIB.hgnn_kernel_time(self._h, i, C.byref(t), C.byref(n)))
            out[name] = (t.value, n.value)
        return out

    def launch_count(self, reset: bool = False) -> int:
        return N.LIB.hgnn_launch_count(self._h, int(reset))

    def halo_bytes(self, reset: bool = False) -> int:
        return N.LIB.hgnn_halo_bytes(self._h, int(reset))


def _mlp(in_dim: int, H: int, k: int) -> int:
    return in_dim * H + H + k * (H * H + H) + H * H + H
