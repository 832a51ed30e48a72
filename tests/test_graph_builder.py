"""The analytic per-rank graph builder (csrc/host_graph.cpp) is bit-exact to
the reference's build_box_mesh -> partition_mesh -> build_distributed_graph
(mesh.cpp:106-226, graph.cpp:40-265): every array of ReducedGraph + HaloMap,
checked against golden hashes from the reference and, when built, against the
reference itself. Structural known answers come from test_graph.cpp /
test_mesh.cpp / acceptance.cpp."""
from __future__ import annotations

import hashlib
import json

import numpy as np
import pytest

import oracle as O
from paper_2410_01657_b200 import (GnnConfig, PartitionError, balanced_factors, build_distributed_graph,
                                   build_rank_graph, init_params, param_count)

FIELDS = ["global_ids", "positions", "edge_src", "edge_dst", "node_degree", "edge_degree", "node_inv_degree",
          "edge_inv_degree", "in_offsets", "in_edges", "out_offsets", "out_edges", "neighbors", "send_offsets",
          "send_rows", "recv_offsets", "recv_rows", "halo_to_local", "sync_local", "sync_offsets", "sync_slots"]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def golden(golden_dir):
    return json.load(open(golden_dir / "reference_hashes.json"))


def test_graphs_match_reference_hashes(golden):
    for key, case in golden["graphs"].items():
        fac = tuple(case["factors"]) if case["factors"] else None
        for r, want in enumerate(case["ranks"]):
            g = build_rank_graph(case["E"], case["p"], case["R"], r, case["strategy"], fac)
            assert (g.num_local, g.num_halo, g.num_edges, g.max_buffer_rows) == (
                want["num_local"], want["num_halo"], want["num_edges"], want["max_buffer_rows"]), key
            for f in FIELDS:
                assert sha(getattr(g, f)) == want[f], (key, r, f)


@pytest.mark.skipif(not O.ref_available(), reason="reference not built in place (oracle/_ref)")
@pytest.mark.parametrize("E,p,R,strat,fac", [(4, 3, 4, "verify", None), (6, 1, 6, "slab", None),
                                             (4, 2, 8, "block", (4, 2, 1)), (6, 2, 12, "verify", None)])
def test_graphs_match_reference_build(E, p, R, strat, fac):
    ref = O.RefGraph(E, p, R, strat, fac, features=False)
    for r in range(R):
        g = build_rank_graph(E, p, R, r, strat, fac)
        for f in FIELDS:
            assert getattr(g, f).tobytes() == getattr(ref.ranks[r], f).tobytes(), (r, f)
        assert g.max_buffer_rows == ref.ranks[r].max_buffer_rows


@pytest.mark.skipif(not O.ref_available(), reason="reference not built in place (oracle/_ref)")
@pytest.mark.parametrize("E,p,R,strat,dom", [(4, 2, 2, "slab", ((-1.0, 0.0, 2.0), (1.0, 0.5, 5.0))),
                                             (4, 3, 4, "verify", ((0.25, -3.0, 0.0), (2.0, 3.0, 0.1)))])
def test_graphs_match_reference_build_on_a_domain(E, p, R, strat, dom):
    """MeshConfig::domain_min / domain_max (mesh.cpp:86-104): positions and every
    other array bit-exact on a non-unit box."""
    ref = O.RefGraph(E, p, R, strat, None, features=False, domain=dom)
    for r in range(R):
        g = build_rank_graph(E, p, R, r, strat, None, dom[0], dom[1])
        for f in FIELDS:
            assert getattr(g, f).tobytes() == getattr(ref.ranks[r], f).tobytes(), (r, f)


def test_domain_must_be_a_box():
    """MeshConfig::validate (mesh.cpp:12-14): ConfigError unless max > min on every axis."""
    from paper_2410_01657_b200 import ConfigError
    with pytest.raises(ConfigError):
        build_rank_graph(2, 2, 1, 0, "slab", None, (0.0, 0.0, 0.0), (1.0, 0.0, 1.0))


def test_params_match_reference_hashes(golden):
    for key, want in golden["params"].items():
        H, M, k, s = [int(t[1:]) for t in key.split("_")]
        p = init_params(GnnConfig("x", H, M, k), s)
        assert p.size == want["count"] and sha(p) == want["sha256"], key


def test_param_counts_table_i():
    """test_nn.cpp:206-219 / PAPER.md Table I: 3,979 and 91,459."""
    assert param_count(GnnConfig.small_model()) == 3979
    assert param_count(GnnConfig.large_model()) == 91459


def test_structured_counts():
    """Acceptance 6: unique nodes (E p + 1)^3, 3 p (p+1)^2 edges per element."""
    for E, p in [(2, 5), (2, 1), (3, 2), (4, 3)]:
        g = build_rank_graph(E, p, 1, 0, "slab")
        assert g.num_local == (E * p + 1) ** 3
        assert g.num_halo == 0 and g.num_edges == 2 * 3 * (E * p) * (E * p + 1) ** 2


def test_table_ii_halo_stats():
    """Acceptance 7 / test_graph.cpp:173-196: E=2, p=5, R=2 slab -> 121 halo, 1 neighbour;
    test_graph.cpp:279-291: E=4, p=2, R=8 block -> 7 neighbours."""
    for r in range(2):
        g = build_rank_graph(2, 5, 2, r, "slab")
        assert g.num_halo == 121 and len(g.neighbors) == 1
    assert all(len(build_rank_graph(4, 2, 8, r, "block").neighbors) == 7 for r in range(8))


def test_partition_of_unity():
    """Acceptance 5: sum over ranks of 1/d is exactly 1 per node and per edge."""
    for E, p, R, strat in [(4, 2, 8, "verify"), (6, 1, 3, "slab"), (4, 3, 4, "verify")]:
        graphs = build_distributed_graph(E, p, R, strat)
        node, edge = {}, {}
        for g in graphs:
            for i in range(g.num_local):
                node[int(g.global_ids[i])] = node.get(int(g.global_ids[i]), 0.0) + g.node_inv_degree[i]
            for e in range(0, g.num_edges, 2):
                a, b = sorted((int(g.global_ids[g.edge_src[e]]), int(g.global_ids[g.edge_dst[e]])))
                edge[(a, b)] = edge.get((a, b), 0.0) + g.edge_inv_degree[e]
        assert all(abs(v - 1.0) <= 1e-14 for v in node.values())
        assert all(abs(v - 1.0) <= 1e-14 for v in edge.values())
        assert len(node) == (E * p + 1) ** 3


def test_halo_pairing_and_isolation():
    """test_graph.cpp:198-277: send/recv masks pair by gid; edges never touch halo rows;
    recv rows are one consecutive block per neighbour."""
    graphs = build_distributed_graph(4, 2, 8, "verify")
    for g in graphs:
        assert g.edge_src.max() < g.num_local and g.edge_dst.max() < g.num_local
        for n, s in enumerate(g.neighbors):
            recv = g.recv_rows[g.recv_offsets[n]:g.recv_offsets[n + 1]]
            assert np.array_equal(recv, np.arange(recv[0], recv[0] + len(recv)))
            other = graphs[s]
            back = list(other.neighbors).index(g.rank)
            sent = other.send_rows[other.send_offsets[back]:other.send_offsets[back + 1]]
            assert np.array_equal(other.global_ids[sent], g.global_ids[recv])
        # twins
        assert np.array_equal(g.edge_src[0::2], g.edge_dst[1::2])


def test_partition_errors():
    with pytest.raises(PartitionError):
        build_rank_graph(3, 2, 2, 0, "slab")
    with pytest.raises(PartitionError):
        build_rank_graph(4, 2, 8, 0, "block", (3, 1, 1))
    assert balanced_factors(8, 4) == (2, 2, 2)
    assert balanced_factors(4, 50) == (2, 2, 1)


def test_model_slices_cover_the_full_parameter_vector():
    """model_slices (encoders, MP layers, decoder; nn.cpp:38-46 names) tile
    the full ModelParams::for_each vector exactly (model.cpp:124-135)."""
    from paper_2410_01657_b200 import GnnConfig, model_slices, param_count
    for H, M, k in ((64, 4, 5), (64, 2, 2), (32, 3, 1)):
        cfg = GnnConfig("s", H, M, k)
        sl = model_slices(cfg)
        assert sl[0][1] == 0 and sl[-1][2] == param_count(cfg)
        assert all(a[2] == b[1] for a, b in zip(sl, sl[1:]))
        names = [n for n, _, _ in sl]
        assert names[0] == "node_encoder.w0" and names[-1] == "node_decoder.skip"
        assert "edge_encoder.ln_b" in names and f"layer{M - 1}.node_update.b{k + 1}" in names
