"""HGNNGRB1 per-rank graph files (io.cpp:200-309).

- Writer: our file for our analytic graph is byte-identical to the reference's
  save_graph_binary output (golden sha256 per rank from tests/golden/
  make_golden.py, and the reference itself when oracle/_ref has io.cpp).
- Loader: a reference-written file loads into exactly the arrays of our
  builder, including the derived reciprocal degrees and CSR
  (finalize_loaded_graph, io.cpp:152-161).
- Errors: missing, JSON, truncated and out-of-range files raise IoError
  (error.hpp:69-73), never a device fault later.
"""
from __future__ import annotations

import hashlib
import json
import struct
from dataclasses import fields

import numpy as np
import pytest

import oracle as O
from paper_2410_01657_b200 import IoError, build_rank_graph, load_graph_binary, save_graph_binary


def same_graph(a, b):
    for f in fields(a):
        if f.name in ("_keep", "num_ranks"):
            continue
        x, y = getattr(a, f.name), getattr(b, f.name)
        if isinstance(x, np.ndarray):
            assert x.dtype == y.dtype and x.tobytes() == y.tobytes(), f.name
        else:
            assert x == y, f.name


@pytest.fixture(scope="module")
def golden(golden_dir):
    return json.load(open(golden_dir / "reference_hashes.json"))


def test_writer_matches_reference_file_hashes(golden, tmp_path):
    for key, case in golden["graphs"].items():
        fac = tuple(case["factors"]) if case["factors"] else None
        for r, want in enumerate(case["ranks"]):
            g = build_rank_graph(case["E"], case["p"], case["R"], r, case["strategy"], fac)
            f = tmp_path / f"{key}_{r}.bin"
            save_graph_binary(g, f)
            assert hashlib.sha256(f.read_bytes()).hexdigest() == want["binary_sha256"], (key, r)


@pytest.mark.parametrize("E,p,R,strat,fac", [(2, 2, 1, "verify", None), (4, 3, 4, "verify", None),
                                             (4, 2, 8, "block", (2, 2, 2)), (3, 2, 3, "slab", None)])
def test_round_trip(tmp_path, E, p, R, strat, fac):
    for r in range(R):
        g = build_rank_graph(E, p, R, r, strat, fac)
        f = tmp_path / f"r{r}.bin"
        save_graph_binary(g, f)
        h = load_graph_binary(f)
        assert h.num_ranks == 0
        same_graph(g, h)


@pytest.mark.skipif(not O.ref_has_io(), reason="oracle/_ref built without the reference's io.cpp")
@pytest.mark.parametrize("E,p,R,strat,fac", [(4, 3, 4, "verify", None), (6, 2, 12, "verify", None),
                                             (4, 2, 8, "block", (4, 2, 1))])
def test_reference_files(tmp_path, E, p, R, strat, fac):
    ref = O.RefGraph(E, p, R, strat, fac, features=False)
    for r in range(R):
        ref_file, ours = tmp_path / f"ref{r}.bin", tmp_path / f"ours{r}.bin"
        ref.save_binary(r, ref_file)
        g = build_rank_graph(E, p, R, r, strat, fac)
        save_graph_binary(g, ours)
        assert ref_file.read_bytes() == ours.read_bytes(), r
        same_graph(g, load_graph_binary(ref_file))


def test_io_errors(tmp_path):
    with pytest.raises(IoError):
        load_graph_binary(tmp_path / "missing.bin")
    js = tmp_path / "g.json"
    js.write_text('{"type": "halo-gnn-graph"}\n')
    with pytest.raises(IoError, match="HGNNGRB1"):
        load_graph_binary(js)
    g = build_rank_graph(2, 2, 2, 0, "slab")
    f = tmp_path / "g.bin"
    save_graph_binary(g, f)
    blob = f.read_bytes()
    for cut in (0, 7, 20, 64, len(blob) // 2, len(blob) - 1):
        (tmp_path / "t.bin").write_bytes(blob[:cut])
        with pytest.raises(IoError):
            load_graph_binary(tmp_path / "t.bin")
    # edge_src[0] := rows (out of range). Header: magic + 6 i64, then
    # global_ids (i64 len + rows*8), positions (i64 len + rows*24), edge_src (i64 len, ...)
    rows = g.num_local + g.num_halo
    off = 8 + 6 * 8 + 8 + rows * 8 + 8 + rows * 24 + 8
    bad = bytearray(blob)
    bad[off:off + 4] = struct.pack("<i", rows)
    (tmp_path / "b.bin").write_bytes(bytes(bad))
    with pytest.raises(IoError, match="edge_src"):
        load_graph_binary(tmp_path / "b.bin")
    with pytest.raises(IoError):
        save_graph_binary(g, tmp_path / "no_such_dir" / "g.bin")
