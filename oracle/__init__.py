"""TEST INFRASTRUCTURE ONLY — Python bindings of the oracle.

  * `liboracle` (oracle/_build/liboracle.so): plain-C fp64 restatement of the
    reference hot path (oracle/hgnn_oracle.c), bitwise equal to the reference.
  * `libhgnn_ref` (oracle/_ref/libhgnn_ref.so): the reference itself, compiled
    in place from /root/reference/proj by oracle/Makefile (optional: absent on
    boxes where it was not built).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this package. The product path never does.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_LIB = HERE / "_build" / "liboracle.so"
REF_LIB = HERE / "_ref" / "libhgnn_ref.so"

i32p = C.POINTER(C.c_int32)
f64p = C.POINTER(C.c_double)
MODES = {"none": 0, "a2a": 1, "na2a": 2}


class OrRankGraph(C.Structure):
    _fields_ = [
        ("num_local", C.c_int64), ("num_halo", C.c_int64), ("num_edges", C.c_int64),
        ("edge_src", i32p), ("edge_dst", i32p), ("edge_inv", f64p),
        ("in_off", i32p), ("in_edges", i32p), ("out_off", i32p), ("out_edges", i32p),
        ("num_nbr", C.c_int32), ("nbr", i32p),
        ("send_off", i32p), ("send_rows", i32p), ("recv_off", i32p), ("recv_rows", i32p),
        ("num_sync", C.c_int64), ("sync_local", i32p), ("sync_off", i32p), ("sync_slots", i32p),
    ]


def _ptr(a, t):
    return a.ctypes.data_as(C.POINTER(t))


# ---------------------------------------------------------------------------
# C restatement
# ---------------------------------------------------------------------------
_olib = None


def oracle_lib() -> C.CDLL:
    global _olib
    if _olib is None:
        if not ORACLE_LIB.exists():
            import subprocess
            subprocess.run(["make", "-C", str(HERE), "-s", "oracle"], check=True)
        lib = C.CDLL(str(ORACLE_LIB))
        pp = C.POINTER(f64p)
        lib.or_mlp_param_count.restype = C.c_int64
        lib.or_mlp_param_count.argtypes = [C.c_int64] * 3
        lib.or_mlp_forward.argtypes = [f64p, C.c_int64, C.c_int64, C.c_int64, C.c_int64, f64p, f64p]
        lib.or_mlp_backward.argtypes = [f64p, C.c_int64, C.c_int64, C.c_int64, C.c_int64, f64p, f64p, f64p, f64p]
        g = C.POINTER(OrRankGraph)
        lib.or_nmp_layer_forward.argtypes = [C.c_int, C.c_int, g, f64p, C.c_int64, C.c_int64, pp, pp, pp, pp, pp, pp]
        lib.or_nmp_layer_backward.argtypes = [C.c_int, C.c_int, g, f64p, C.c_int64, C.c_int64, pp, pp, pp, pp, pp, pp]
        lib.or_exchange_bytes.restype = C.c_int64
        lib.or_exchange_bytes.argtypes = [C.c_int, C.c_int, g, C.c_int, C.c_int64, C.c_int64]
        _olib = lib
    return _olib


def or_graph(rg, keep: list) -> OrRankGraph:
    """or_rank_graph view of a RankGraph-like object (numpy attributes)."""
    def a(x, dt):
        arr = np.ascontiguousarray(x, dtype=dt)
        keep.append(arr)
        return arr
    g = OrRankGraph()
    g.num_local, g.num_halo, g.num_edges = rg.num_local, rg.num_halo, rg.num_edges
    g.edge_src = _ptr(a(rg.edge_src, np.int32), C.c_int32)
    g.edge_dst = _ptr(a(rg.edge_dst, np.int32), C.c_int32)
    g.edge_inv = _ptr(a(rg.edge_inv_degree, np.float64), C.c_double)
    g.in_off = _ptr(a(rg.in_offsets, np.int32), C.c_int32)
    g.in_edges = _ptr(a(rg.in_edges, np.int32), C.c_int32)
    g.out_off = _ptr(a(rg.out_offsets, np.int32), C.c_int32)
    g.out_edges = _ptr(a(rg.out_edges, np.int32), C.c_int32)
    g.num_nbr = len(rg.neighbors)
    g.nbr = _ptr(a(rg.neighbors, np.int32), C.c_int32)
    g.send_off = _ptr(a(rg.send_offsets, np.int32), C.c_int32)
    g.send_rows = _ptr(a(rg.send_rows, np.int32), C.c_int32)
    g.recv_off = _ptr(a(rg.recv_offsets, np.int32), C.c_int32)
    g.recv_rows = _ptr(a(rg.recv_rows, np.int32), C.c_int32)
    g.num_sync = len(rg.sync_local)
    g.sync_local = _ptr(a(rg.sync_local, np.int32), C.c_int32)
    g.sync_off = _ptr(a(rg.sync_offsets, np.int32), C.c_int32)
    g.sync_slots = _ptr(a(rg.sync_slots, np.int32), C.c_int32)
    return g


def _pp(arrs):
    return (f64p * len(arrs))(*[x.ctypes.data_as(f64p) for x in arrs])


def mlp_param_count(in_dim, H, k):
    return in_dim * H + H + k * (H * H + H) + H * H + H


def oracle_mp_run(graphs, H, M, k, mode, mp_params, x0s, e0s, dxms, dems=None):
    """Forward + backward of the MP stack on R in-process ranks (fp64 oracle).

    Returns dict with per-rank lists: x_out[m], e_out[m], a_pre[m], a_sync[m],
    dx_in[m], de_in[m] (adjoints of layer m's inputs) and grads (MP block)."""
    lib = oracle_lib()
    R = len(graphs)
    keep: list = []
    garr = (OrRankGraph * R)(*[or_graph(g, keep) for g in graphs])
    n_layer = mlp_param_count(3 * H, H, k) + mlp_param_count(2 * H, H, k)
    mp_params = np.ascontiguousarray(mp_params, dtype=np.float64)
    res = {key: [[None] * M for _ in range(R)] for key in ("x_in", "e_in", "x_out", "e_out", "a_pre", "a_sync",
                                                          "dx_in", "de_in")}
    x = [np.ascontiguousarray(v, dtype=np.float64) for v in x0s]
    e = [np.ascontiguousarray(v, dtype=np.float64) for v in e0s]
    for m in range(M):
        rows = [g.num_local + g.num_halo for g in graphs]
        xo = [np.zeros((rows[r], H)) for r in range(R)]
        eo = [np.zeros((graphs[r].num_edges, H)) for r in range(R)]
        ap = [np.zeros((rows[r], H)) for r in range(R)]
        asy = [np.zeros((rows[r], H)) for r in range(R)]
        lp = mp_params[m * n_layer:(m + 1) * n_layer]
        lib.or_nmp_layer_forward(R, MODES[mode], garr, lp.ctypes.data_as(f64p), H, k, _pp(x), _pp(e), _pp(xo),
                                 _pp(eo), _pp(ap), _pp(asy))
        for r in range(R):
            res["x_in"][r][m], res["e_in"][r][m] = x[r], e[r]
            res["x_out"][r][m], res["e_out"][r][m] = xo[r], eo[r]
            res["a_pre"][r][m], res["a_sync"][r][m] = ap[r], asy[r]
        x, e = xo, eo
    grads = [np.zeros(M * n_layer) for _ in range(R)]
    dx = [np.array(v, dtype=np.float64) for v in dxms]
    if dems is not None:
        de = [np.array(v, dtype=np.float64) for v in dems]
    else:
        de = [np.zeros((g.num_edges, H)) for g in graphs]
    for m in range(M - 1, -1, -1):
        lp = mp_params[m * n_layer:(m + 1) * n_layer]
        gl = [gr[m * n_layer:(m + 1) * n_layer] for gr in grads]
        gviews = (f64p * R)(*[g.ctypes.data_as(f64p) for g in gl])
        lib.or_nmp_layer_backward(R, MODES[mode], garr, lp.ctypes.data_as(f64p), H, k,
                                  _pp([res["x_in"][r][m] for r in range(R)]),
                                  _pp([res["e_in"][r][m] for r in range(R)]),
                                  _pp([res["a_sync"][r][m] for r in range(R)]), _pp(dx), _pp(de), gviews)
        for r in range(R):
            res["dx_in"][r][m], res["de_in"][r][m] = dx[r].copy(), de[r].copy()
    res["grads"] = grads
    return res


# ---------------------------------------------------------------------------
# reference compiled in place
# ---------------------------------------------------------------------------
_rlib = None


def ref_available() -> bool:
    return REF_LIB.exists()


def ref_has_io() -> bool:
    """True when oracle/_ref was built with the reference's io.cpp."""
    return ref_available() and bool(ref_lib().ref_has_io())


def ref_lib() -> C.CDLL:
    global _rlib
    if _rlib is None:
        lib = C.CDLL(str(REF_LIB))
        vp = C.c_void_p
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_graph_build.restype = vp
        lib.ref_graph_build.argtypes = [C.c_int64] * 3 + [C.c_int] + [C.c_int64] * 3 + [C.c_int]
        lib.ref_graph_build_domain.restype = vp
        lib.ref_graph_build_domain.argtypes = [C.c_int64] * 3 + [C.c_int] + [C.c_int64] * 3 + [C.c_int, f64p, f64p]
        lib.ref_graph_free.argtypes = [vp]
        lib.ref_graph_save_binary.argtypes = [vp, C.c_int, C.c_char_p]
        lib.ref_has_io.restype = C.c_int
        lib.ref_graph_sizes.argtypes = [vp, C.c_int, C.POINTER(C.c_int64)]
        i64p = C.POINTER(C.c_int64)
        lib.ref_graph_export.argtypes = [vp, C.c_int, i64p, f64p, f64p, f64p, i32p, i32p, i32p, i32p, f64p, f64p,
                                         i32p, i32p, i32p, i32p]
        lib.ref_halo_export.argtypes = [vp, C.c_int] + [i32p] * 9
        lib.ref_param_count.restype = C.c_int64
        lib.ref_param_count.argtypes = [C.c_int64] * 3
        lib.ref_mp_param_count.restype = C.c_int64
        lib.ref_mp_param_count.argtypes = [C.c_int64] * 3
        lib.ref_init_params.argtypes = [C.c_int64] * 3 + [C.c_uint64, f64p]
        pp = C.POINTER(f64p)
        lib.ref_mp_run.restype = vp
        lib.ref_mp_run.argtypes = [vp, C.c_int64, C.c_int64, C.c_int64, C.c_int, f64p, pp, pp, pp, pp, C.c_int]
        lib.ref_run.restype = vp
        lib.ref_run.argtypes = [vp, C.c_int64, C.c_int64, C.c_int64, C.c_int, C.c_uint64, f64p, C.c_int]
        lib.ref_run_free.argtypes = [vp]
        lib.ref_run_loss.restype = C.c_double
        lib.ref_run_loss.argtypes = [vp]
        lib.ref_run_times.argtypes = [vp, f64p, f64p]
        lib.ref_run_size.restype = C.c_int64
        lib.ref_run_size.argtypes = [vp, C.c_int, C.c_int, C.c_int]
        lib.ref_run_export.argtypes = [vp, C.c_int, C.c_int, C.c_int, f64p]
        lib.ref_train.restype = C.c_int
        lib.ref_train.argtypes = [vp, C.c_int64, C.c_int64, C.c_int64, C.c_int, C.c_uint64, C.c_int64, C.c_double,
                                  C.c_double, C.c_double, C.c_double, C.c_int, f64p, f64p]
        _rlib = lib
    return _rlib


class RefRankGraph:
    """One rank of the reference's DistributedGraph, as numpy arrays."""


class RefGraph:
    STRAT = {"slab": 0, "block": 1, "verify": 2}

    def __init__(self, E, p, R, strategy="verify", factors=None, features=True, domain=None):
        lib = ref_lib()
        f = factors or (0, 0, 0)
        if domain is None:
            self.h = lib.ref_graph_build(E, p, R, self.STRAT[strategy], f[0], f[1], f[2], int(features))
        else:  # MeshConfig::domain_min / domain_max
            lo, hi = (C.c_double * 3)(*domain[0]), (C.c_double * 3)(*domain[1])
            self.h = lib.ref_graph_build_domain(E, p, R, self.STRAT[strategy], f[0], f[1], f[2], int(features),
                                                C.cast(lo, f64p), C.cast(hi, f64p))
        if not self.h:
            raise RuntimeError(lib.ref_last_error().decode())
        self.R = R
        self.features = features
        self.ranks = [self._export(r) for r in range(R)]

    def _export(self, r):
        lib = ref_lib()
        s = (C.c_int64 * 9)()
        lib.ref_graph_sizes(self.h, r, s)
        nl, nh, ne, nn, ns, nsync, nslots, mbr, _ = list(s)
        rows = nl + nh
        g = RefRankGraph()
        g.rank, g.num_ranks, g.num_local, g.num_halo, g.num_edges, g.max_buffer_rows = r, self.R, nl, nh, ne, mbr
        g.global_ids = np.zeros(rows, np.int64)
        g.positions = np.zeros((rows, 3))
        g.node_features = np.zeros((rows, 3))
        g.edge_features = np.zeros((ne, 7))
        for nm, n in (("edge_src", ne), ("edge_dst", ne), ("node_degree", nl), ("edge_degree", ne),
                      ("in_offsets", rows + 1), ("in_edges", ne), ("out_offsets", rows + 1), ("out_edges", ne)):
            setattr(g, nm, np.zeros(n, np.int32))
        g.node_inv_degree = np.zeros(nl)
        g.edge_inv_degree = np.zeros(ne)
        lib.ref_graph_export(self.h, r, _ptr(g.global_ids, C.c_int64), _ptr(g.positions, C.c_double),
                             _ptr(g.node_features, C.c_double) if self.features else None,
                             _ptr(g.edge_features, C.c_double) if self.features else None,
                             _ptr(g.edge_src, C.c_int32), _ptr(g.edge_dst, C.c_int32),
                             _ptr(g.node_degree, C.c_int32), _ptr(g.edge_degree, C.c_int32),
                             _ptr(g.node_inv_degree, C.c_double), _ptr(g.edge_inv_degree, C.c_double),
                             _ptr(g.in_offsets, C.c_int32), _ptr(g.in_edges, C.c_int32),
                             _ptr(g.out_offsets, C.c_int32), _ptr(g.out_edges, C.c_int32))
        g.neighbors = np.zeros(nn, np.int32)
        g.send_offsets = np.zeros(nn + 1, np.int32)
        g.send_rows = np.zeros(ns, np.int32)
        g.recv_offsets = np.zeros(nn + 1, np.int32)
        g.recv_rows = np.zeros(nh, np.int32)
        g.halo_to_local = np.zeros(nh, np.int32)
        g.sync_local = np.zeros(nsync, np.int32)
        g.sync_offsets = np.zeros(nsync + 1, np.int32)
        g.sync_slots = np.zeros(nslots, np.int32)
        lib.ref_halo_export(self.h, r, *[_ptr(getattr(g, n), C.c_int32) for n in (
            "neighbors", "send_offsets", "send_rows", "recv_offsets", "recv_rows", "halo_to_local", "sync_local",
            "sync_offsets", "sync_slots")])
        return g

    def save_binary(self, rank, path):
        """The reference's own save_graph_binary (io.cpp:200-231) for one rank."""
        rc = ref_lib().ref_graph_save_binary(self.h, rank, str(path).encode())
        if rc == -2:
            raise RuntimeError("io.cpp is not compiled into oracle/_ref (nlohmann/json.hpp not found)")
        if rc != 0:
            raise RuntimeError(ref_lib().ref_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            ref_lib().ref_graph_free(self.h)
            self.h = None


def ref_init_params(H, M, k, seed) -> np.ndarray:
    lib = ref_lib()
    out = np.zeros(lib.ref_param_count(H, M, k))
    lib.ref_init_params(H, M, k, seed, out.ctypes.data_as(f64p))
    return out


class RefRun:
    """Recorded reference run; export(rank, what, layer) returns an fp64 array."""
    WHAT = {"x0": 0, "e0": 1, "x_in": 2, "e_in": 3, "a_sync": 4, "x_out": 5, "e_out": 6, "y": 7, "dy": 8,
            "dx_m": 9, "dx_in": 10, "de_in": 11, "de_m": 12, "mp_grads": 13, "all_grads": 14}

    def __init__(self, handle, H):
        if not handle:
            raise RuntimeError(ref_lib().ref_last_error().decode())
        self.h, self.H = handle, H

    def get(self, rank, what, layer=0):
        lib = ref_lib()
        w = self.WHAT[what]
        n = lib.ref_run_size(self.h, rank, w, layer)
        out = np.zeros(n)
        lib.ref_run_export(self.h, rank, w, layer, out.ctypes.data_as(f64p))
        if what not in ("mp_grads", "all_grads"):
            out = out.reshape(-1, self.H) if what not in ("y", "dy") else out.reshape(-1, 3)
        return out

    @property
    def loss(self):
        return ref_lib().ref_run_loss(self.h)

    def times_ms(self):
        f, b = C.c_double(), C.c_double()
        ref_lib().ref_run_times(self.h, C.byref(f), C.byref(b))
        return f.value, b.value

    def __del__(self):
        if getattr(self, "h", None):
            ref_lib().ref_run_free(self.h)
            self.h = None


def ref_mp_run(graph: RefGraph, H, M, k, mode, mp_params, x0s, e0s, dxms, dems=None, threads_per_rank=0) -> RefRun:
    lib = ref_lib()
    keep = [np.ascontiguousarray(a, dtype=np.float64) for a in list(x0s) + list(e0s) + list(dxms)
            + (list(dems) if dems is not None else [])]
    R = graph.R
    mp = np.ascontiguousarray(mp_params, dtype=np.float64)
    h = lib.ref_mp_run(graph.h, H, M, k, MODES[mode], mp.ctypes.data_as(f64p), _pp(keep[0:R]), _pp(keep[R:2 * R]),
                       _pp(keep[2 * R:3 * R]), _pp(keep[3 * R:4 * R]) if dems is not None else None,
                       threads_per_rank)
    return RefRun(h, H)


def ref_run(graph: RefGraph, H, M, k, mode, seed=0, params=None, threads_per_rank=0) -> RefRun:
    lib = ref_lib()
    p = None
    if params is not None:
        params = np.ascontiguousarray(params, dtype=np.float64)
        p = params.ctypes.data_as(f64p)
    return RefRun(lib.ref_run(graph.h, H, M, k, MODES[mode], seed, p, threads_per_rank), H)


def ref_train(graph: RefGraph, H, M, k, mode, seed, iters, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8,
              threads_per_rank=0):
    """Reference train() (model.cpp:582-640): per-iteration losses and rank 0's final parameters."""
    lib = ref_lib()
    losses = np.zeros(iters)
    params = np.zeros(lib.ref_param_count(H, M, k))
    rc = lib.ref_train(graph.h, H, M, k, MODES[mode], seed, iters, lr, beta1, beta2, eps, threads_per_rank,
                       losses.ctypes.data_as(f64p), params.ctypes.data_as(f64p))
    if rc != 0:
        raise RuntimeError(lib.ref_last_error().decode())
    return losses, params
