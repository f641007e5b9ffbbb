"""Multi-rank sharded build on CPU (gloo, world sizes 2/4/8): the product's
distributed driver (paper_1302_5995_b200/shard.py) with an oracle-backed
engine, checked against the single-process oracle root S. The shard
geometry comes from the product (dtn_gpu_shard_info)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as tdist
import torch.multiprocessing as mp

import paper_1302_5995_b200 as dtn
from paper_1302_5995_b200 import shard as SH
from oracle import oracle as O

N = 66  # 64 x 64 interior, 16 x 16 leaves -> depth 2 (8 shards possible)
PROBLEM = ("helmholtz", 10.0)


class OracleShardEngine:
    """Test double of GpuShardEngine computing with the CPU oracle."""

    def __init__(self):
        self.p = O.Problem(PROBLEM[0], N, PROBLEM[1])
        self.t = O.Tree(N, uniform_side=16)
        self.tree = dtn.build_tree_uniform(N, 16)
        self.ref = O.build_root_dense(self.p, self.t, keep_all=True)

    def rect(self, bid):
        b = self.t.boxes[bid]
        return (b["x0"], b["x1"], b["y0"], b["y1"])

    def merge(self, ra, Sa, rb, Sb):
        return O.merge_given(self.p, ra, Sa, rb, Sb)

    def shard_nb(self, nshards, s):
        return dtn.shard_info(self.tree, nshards, s)["nb"]

    def build_shard(self, nshards, s):
        q = self.t.boxes[0]["children"]
        if nshards == 4:
            rect, S = self.rect(q[s]), self.ref.box_S(q[s])
        elif nshards == 2:
            a, b = (q[0], q[2]) if s == 0 else (q[1], q[3])
            rect, S = self.merge(self.rect(a), self.ref.box_S(a), self.rect(b), self.ref.box_S(b))
        else:
            c = self.t.boxes[q[s // 2]]["children"]
            a, b = (c[0], c[2]) if s % 2 == 0 else (c[1], c[3])
            rect, S = self.merge(self.rect(a), self.ref.box_S(a), self.rect(b), self.ref.box_S(b))
        assert tuple(rect) == dtn.shard_info(self.tree, nshards, s)["rect"]
        return torch.from_numpy(np.ascontiguousarray(S))

    def build_top(self, nshards, blocks):
        info = [dtn.shard_info(self.tree, nshards, s)["rect"] for s in range(nshards)]
        S = [b.numpy() for b in blocks]
        if nshards == 8:  # quadrant = W|E halves
            quads = [self.merge(info[2 * i], S[2 * i], info[2 * i + 1], S[2 * i + 1]) for i in range(4)]
            info = [q[0] for q in quads]
            S = [q[1] for q in quads]
            nshards = 4
        if nshards == 4:  # W = SW+NW, E = SE+NE (merge_four, dense_nd.cpp:188-194)
            w = self.merge(info[0], S[0], info[2], S[2])
            e = self.merge(info[1], S[1], info[3], S[3])
            info, S = [w[0], e[0]], [w[1], e[1]]
        return self.merge(info[0], S[0], info[1], S[1])[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = SH.build_distributed(OracleShardEngine(), rank, world)
        if rank == 0:
            q.put(np.asarray(out))
    finally:
        tdist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.timeout(600)
@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_build_matches_single_process(world):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    pc = mp.start_processes(_worker, args=(world, _free_port(), q), nprocs=world, join=False, start_method="spawn")
    S = q.get()  # read before joining: a large put blocks until consumed
    while not pc.join():
        pass
    ref = O.build_root_dense(O.Problem(PROBLEM[0], N, PROBLEM[1]), O.Tree(N, uniform_side=16))
    assert O.rel_fro(S, ref.S) <= 1e-12


def test_shard_geometry_tiles_the_domain():
    tree = dtn.build_tree_uniform(130, 16)
    for ns in (1, 2, 4, 8):
        cells = set()
        for s in range(ns):
            x0, x1, y0, y1 = dtn.shard_info(tree, ns, s)["rect"]
            part = {(x, y) for x in range(x0, x1 + 1) for y in range(y0, y1 + 1)}
            assert not (cells & part)
            cells |= part
        assert len(cells) == 128 * 128
    with pytest.raises(ValueError):
        dtn.shard_info(dtn.build_tree_uniform(34, 16), 8, 0)  # depth 1: too shallow for 8
