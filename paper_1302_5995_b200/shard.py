"""Multi-GPU build by subtree sharding: one process per GPU,
torch.distributed for the plumbing. Rank r builds the Schur complement of
shard r (the root's W|E halves for 2 GPUs, its quadrants for 4, the quadrant
halves for 8) with no communication; the shard S blocks are then sent to rank
0, which runs the top merges of the tree (the only exchange step of the
build) and the root inverse. The reference has no distributed path; its own
top merges are merge_four at the top levels (dense_nd.cpp:188-216).

The driver is written against a small engine interface (`shard_nb`,
`build_shard`, `build_top`) so the same protocol runs on B200s (GpuShardEngine,
NCCL over NVLink) and is exercised on CPU with gloo in the tests.
"""
from __future__ import annotations

from . import dtn


class GpuShardEngine:
    """The B200 engine behind the C ABI (dtn_gpu_build with opts.nshards/shard)."""

    def __init__(self, op: dtn.DiscreteOperator, tree: dtn.BoxTree, ctx: dtn.Context | None = None,
                 stencil_device_ptr: int | None = None, device=None, accel: dtn.AccelOptions | None = None):
        """accel: build the root in compressed form (build_root_accel) on rank 0."""
        self.op, self.tree, self.ctx = op, tree, ctx
        self.accel = accel
        self.stencil_device_ptr = stencil_device_ptr
        self.device = device
        self.last_shard_op = None

    def shard_nb(self, nshards: int, shard: int) -> int:
        return dtn.shard_info(self.tree, nshards, shard)["nb"]

    def build_full(self):
        if self.accel is not None:
            return dtn.build_root_accel(self.op, self.tree, self.accel, ctx=self.ctx,
                                        stencil_device_ptr=self.stencil_device_ptr)
        return dtn.build_root_gpu(self.op, self.tree, want_G=True, ctx=self.ctx,
                                  stencil_device_ptr=self.stencil_device_ptr)

    def build_shard(self, nshards: int, shard: int):
        import torch
        # with accel: the shard's subtree uses the structured merges above the crossover
        sol = dtn.build_root_gpu(self.op, self.tree, want_G=False, ctx=self.ctx,
                                 stencil_device_ptr=self.stencil_device_ptr, nshards=nshards, shard=shard,
                                 accel=self.accel)
        nb = len(sol.boundary)
        # device-to-device copy of the shard S into a column-major tensor
        S = torch.empty((nb, nb), dtype=torch.float64, device=self.device or "cuda").t()
        sol.export_device(S.data_ptr(), nb)
        sol.free()
        return S

    def build_top(self, nshards: int, shard_S: list):
        if self.accel is not None:
            return dtn.build_root_accel(self.op, self.tree, self.accel, ctx=self.ctx,
                                        stencil_device_ptr=self.stencil_device_ptr, nshards=nshards, shard_S=shard_S)
        return dtn.build_root_gpu(self.op, self.tree, want_G=True, ctx=self.ctx,
                                  stencil_device_ptr=self.stencil_device_ptr, nshards=nshards, shard=-1,
                                  shard_S=shard_S)


def build_distributed(engine, rank: int, world: int):
    """Sharded build over `world` ranks (1, 2, 4 or 8). Returns rank 0's result
    of engine.build_top (None on the other ranks)."""
    if world == 1:
        return engine.build_full()
    import torch.distributed as tdist
    mine = engine.build_shard(world, rank)
    if rank == 0:
        blocks = [mine]
        for src in range(1, world):
            nb = engine.shard_nb(world, src)
            buf = mine.new_empty((nb, nb))
            tdist.recv(buf, src=src)
            blocks.append(buf)
        return engine.build_top(world, blocks)
    tdist.send(mine.contiguous(), dst=0)
    return None
