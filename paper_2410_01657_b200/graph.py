"""Per-rank graph (ReducedGraph + HaloMap, graph.hpp:16-65) as numpy arrays.

`build_rank_graph` calls the native analytic builder (csrc/host_graph.cpp),
which reproduces build_box_mesh -> partition_mesh -> build_distributed_graph
(mesh.cpp:106-226, graph.cpp:40-265) bit-exactly for one rank.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field, fields

import numpy as np

from . import _native as N

STRATEGIES = {"slab": N.PART_SLAB, "block": N.PART_BLOCK, "verify": N.PART_VERIFY}


@dataclass
class RankGraph:
    rank: int
    num_ranks: int
    num_local: int
    num_halo: int
    num_edges: int
    global_ids: np.ndarray           # int64 [rows]
    positions: np.ndarray            # float64 [rows, 3]
    edge_src: np.ndarray             # int32 [N_e]
    edge_dst: np.ndarray
    node_degree: np.ndarray          # int32 [num_local]
    edge_degree: np.ndarray          # int32 [N_e]
    node_inv_degree: np.ndarray      # float64 [num_local]
    edge_inv_degree: np.ndarray      # float64 [N_e]
    in_offsets: np.ndarray           # int32 [rows+1]
    in_edges: np.ndarray
    out_offsets: np.ndarray
    out_edges: np.ndarray
    neighbors: np.ndarray            # int32 [n_nbr]
    send_offsets: np.ndarray         # int32 [n_nbr+1]
    send_rows: np.ndarray
    recv_offsets: np.ndarray
    recv_rows: np.ndarray
    halo_to_local: np.ndarray
    sync_local: np.ndarray           # int32 [n_sync]
    sync_offsets: np.ndarray         # int32 [n_sync+1]
    sync_slots: np.ndarray
    max_buffer_rows: int
    _keep: list = field(default_factory=list, repr=False)

    @property
    def rows(self) -> int:
        return self.num_local + self.num_halo

    def desc(self) -> N.GraphDesc:
        """hgnn_graph_desc pointing into this object's arrays."""
        d = N.GraphDesc()
        d.rank, d.num_ranks = self.rank, self.num_ranks
        d.num_local, d.num_halo, d.num_edges = self.num_local, self.num_halo, self.num_edges
        self._keep = []

        def ptr(arr, ctype):
            a = np.ascontiguousarray(arr)
            self._keep.append(a)
            return a.ctypes.data_as(C.POINTER(ctype))

        ctypes_of = {np.dtype(np.int64): C.c_int64, np.dtype(np.float64): C.c_double, np.dtype(np.int32): C.c_int32}
        for f in fields(self):
            v = getattr(self, f.name)
            if isinstance(v, np.ndarray):
                setattr(d, f.name, ptr(v, ctypes_of[v.dtype]))
        d.num_neighbors = len(self.neighbors)
        d.num_sync_groups = len(self.sync_local)
        d.max_buffer_rows = self.max_buffer_rows
        return d


def _arr(ptr, n, dtype):
    if n == 0:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)


def build_rank_graph(elements_per_axis: int, poly_order: int, num_ranks: int, rank: int,
                     strategy: str = "verify", factors=None, domain_min=None, domain_max=None) -> RankGraph:
    """One rank's reduced graph and halo map for the GLL box mesh on
    [domain_min, domain_max] (MeshConfig, default the unit cube)."""
    h = C.c_void_p()
    fac = None
    if factors is not None:
        fac = (C.c_int64 * 3)(*factors)
    lo = (C.c_double * 3)(*domain_min) if domain_min is not None else None
    hi = (C.c_double * 3)(*domain_max) if domain_max is not None else None
    N.check(N.LIB.hgnn_graph_build_domain(elements_per_axis, poly_order, num_ranks, STRATEGIES[strategy],
                                          C.cast(fac, N.i64p) if fac is not None else None, rank,
                                          C.cast(lo, N.f64p) if lo is not None else None,
                                          C.cast(hi, N.f64p) if hi is not None else None, C.byref(h)))
    return _take(h)


def load_graph_binary(path) -> RankGraph:
    """load_graph for HGNNGRB1 files (io.cpp:241-309); num_ranks is 0 (not stored)."""
    h = C.c_void_p()
    N.check(N.LIB.hgnn_graph_load_binary(str(path).encode(), C.byref(h)))
    return _take(h)


def save_graph_binary(graph: RankGraph, path) -> None:
    """save_graph_binary (io.cpp:200-231), byte-identical to the reference's."""
    d = graph.desc()
    N.check(N.LIB.hgnn_graph_save_binary(C.byref(d), str(path).encode()))


def _take(h) -> RankGraph:
    """Copy a native hgnn_host_graph into numpy arrays and free it."""
    try:
        d = N.GraphDesc()
        N.check(N.LIB.hgnn_graph_view(h, C.byref(d)))
        nl, nh, ne = d.num_local, d.num_halo, d.num_edges
        rows = nl + nh
        nn = d.num_neighbors
        ns = d.send_offsets[nn] if nn else 0
        nsync = d.num_sync_groups
        nslots = d.sync_offsets[nsync] if nsync else 0
        return RankGraph(
            rank=d.rank, num_ranks=d.num_ranks, num_local=nl, num_halo=nh, num_edges=ne,
            global_ids=_arr(d.global_ids, rows, np.int64),
            positions=_arr(d.positions, rows * 3, np.float64).reshape(rows, 3),
            edge_src=_arr(d.edge_src, ne, np.int32), edge_dst=_arr(d.edge_dst, ne, np.int32),
            node_degree=_arr(d.node_degree, nl, np.int32), edge_degree=_arr(d.edge_degree, ne, np.int32),
            node_inv_degree=_arr(d.node_inv_degree, nl, np.float64),
            edge_inv_degree=_arr(d.edge_inv_degree, ne, np.float64),
            in_offsets=_arr(d.in_offsets, rows + 1, np.int32), in_edges=_arr(d.in_edges, ne, np.int32),
            out_offsets=_arr(d.out_offsets, rows + 1, np.int32), out_edges=_arr(d.out_edges, ne, np.int32),
            neighbors=_arr(d.neighbors, nn, np.int32),
            send_offsets=_arr(d.send_offsets, nn + 1, np.int32), send_rows=_arr(d.send_rows, ns, np.int32),
            recv_offsets=_arr(d.recv_offsets, nn + 1, np.int32),
            recv_rows=_arr(d.recv_rows, d.recv_offsets[nn] if nn else 0, np.int32),
            halo_to_local=_arr(d.halo_to_local, nh, np.int32),
            sync_local=_arr(d.sync_local, nsync, np.int32), sync_offsets=_arr(d.sync_offsets, nsync + 1, np.int32),
            sync_slots=_arr(d.sync_slots, nslots, np.int32),
            max_buffer_rows=d.max_buffer_rows)
    finally:
        N.LIB.hgnn_graph_free(h)


def build_distributed_graph(elements_per_axis: int, poly_order: int, num_ranks: int,
                            strategy: str = "verify", factors=None) -> list[RankGraph]:
    """All ranks (test helper; production ranks build only their own)."""
    return [build_rank_graph(elements_per_axis, poly_order, num_ranks, r, strategy, factors)
            for r in range(num_ranks)]


def balanced_factors(num_ranks: int, elements_per_axis: int) -> tuple[int, int, int]:
    out = (C.c_int64 * 3)()
    N.check(N.LIB.hgnn_balanced_factors(num_ranks, elements_per_axis, out))
    return tuple(out)
