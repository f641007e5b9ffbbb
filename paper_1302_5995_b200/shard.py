"""Multi-GPU build by subtree sharding: one process per GPU.

build_collective -- the production path: the whole sharded build runs in the
engine (C++ host side, its own NCCL communicator): rank r builds the Schur
complement of shard r (the root's W|E halves for 2 GPUs, its quadrants for 4,
the quadrant halves for 8) with no communication, the shard S blocks are
all-gathered, and the merges above the shards are column-sharded over the
ranks (interface LU redundant, the boundary columns' substitutions and Schur
GEMM split, all-gathered per wave), as is the root inverse.

build_distributed -- the same subtree split with the top of the tree on rank 0,
driven from Python through a small engine interface (`shard_nb`,
`build_shard`, `build_top`), so the protocol also runs on CPU with gloo in the
tests. The reference has no distributed path; its own top merges are
merge_four at the top levels (dense_nd.cpp:188-216).
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


def build_collective(op, tree, ctx: dtn.Context, stencil_device_ptr: int | None = None,
                     accel: dtn.AccelOptions | None = None, want_G: bool = True):
    """The collective build over ctx's NCCL world (one process per GPU, every rank calls
    this): shard `rank` built locally, the shard S blocks all-gathered in the engine's
    communicator, the top merges column-sharded with their chunks all-gathered after
    each wave, the root inverse column-sharded likewise (dtn_opts.shard = -2, C++ host
    side). Every rank returns the root operator."""
    if ctx.world == 1:
        if accel is not None:
            return dtn.build_root_accel(op, tree, accel, ctx=ctx, stencil_device_ptr=stencil_device_ptr)
        return dtn.build_root_gpu(op, tree, want_G=want_G, ctx=ctx, stencil_device_ptr=stencil_device_ptr)
    if accel is not None:
        return dtn.build_root_accel(op, tree, accel, ctx=ctx, stencil_device_ptr=stencil_device_ptr,
                                    nshards=ctx.world, collective=-2)
    return dtn.build_root_gpu(op, tree, want_G=want_G, ctx=ctx, stencil_device_ptr=stencil_device_ptr,
                              nshards=ctx.world, shard=-2)


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
