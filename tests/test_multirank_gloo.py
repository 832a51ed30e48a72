"""N>1 host logic on CPU (world_size 2 and 4, gloo, 127.0.0.1): each process
builds ITS rank graph with the host builder, runs the na2a halo plan the device
engine hands to NCCL (pack send_rows per neighbour -> point-to-point ->
unpack into the contiguous recv_rows) over real process boundaries, then the
ascending-owner-rank synchronisation; also the bench's uid broadcast and
max-over-ranks reduction. Checks: every halo row receives the value of the
same global id, and every synchronised aggregate equals node_degree copies
(model.cpp:243-257, comm.cpp:281-315)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def f_of_gid(gid: np.ndarray, H: int) -> np.ndarray:
    g = gid.astype(np.float64)[:, None]
    return np.concatenate([g, 0.5 * g, np.full_like(g, 3.0), (g % 7) - 3.0], axis=1)[:, :H]


def _worker(rank, world, port, E, p):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2410_01657_b200 import build_rank_graph
        g = build_rank_graph(E, p, world, rank, "verify")
        H = 4
        a = np.full((g.rows, H), np.nan)
        a[:g.num_local] = f_of_gid(g.global_ids[:g.num_local], H)
        # na2a exchange: one send/recv pair per neighbour (ascending), as the engine's NCCL group
        reqs, bufs = [], []
        for n, nbr in enumerate(g.neighbors):
            s0, s1 = g.send_offsets[n], g.send_offsets[n + 1]
            r0, r1 = g.recv_offsets[n], g.recv_offsets[n + 1]
            send = torch.from_numpy(np.ascontiguousarray(a[g.send_rows[s0:s1]]))
            recv = torch.empty((r1 - r0, H), dtype=torch.float64)
            bufs.append((recv, g.recv_rows[r0:r1]))
            if rank < nbr:
                reqs += [dist.isend(send, int(nbr)), dist.irecv(recv, int(nbr))]
            else:
                reqs += [dist.irecv(recv, int(nbr)), dist.isend(send, int(nbr))]
        for r in reqs:
            r.wait()
        for recv, rows in bufs:
            assert np.all(np.diff(rows) == 1), "recv rows of one neighbour must be consecutive"
            a[rows] = recv.numpy()
        halo = np.arange(g.num_local, g.rows)
        assert np.array_equal(a[halo], f_of_gid(g.global_ids[halo], H)), "halo pairing"
        # synchronisation in ascending owner-rank order
        for i, loc in enumerate(g.sync_local):
            slots = g.sync_slots[g.sync_offsets[i]:g.sync_offsets[i + 1]]
            acc = np.zeros(H)
            for s in slots:
                acc = acc + (a[loc] if s < 0 else a[s])
            assert len(slots) == g.node_degree[loc]
            assert np.array_equal(acc, len(slots) * f_of_gid(g.global_ids[[loc]], H)[0])
        # bench.py control plane: uid broadcast + max-over-ranks timing
        obj = [bytes(range(16)) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        assert obj[0] == bytes(range(16))
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        assert t.item() == float(world)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,E,p", [(2, 4, 2), (4, 4, 3)])
def test_halo_plan_across_processes(world, E, p):
    mp.spawn(_worker, args=(world, _free_port(), E, p), nprocs=world, join=True)
