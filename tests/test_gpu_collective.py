"""The collective multi-GPU build (dtn_opts.shard = -2 over the
context's NCCL world) checked on one device: shard = -3 runs the same split --
every shard subtree, every rank's column chunk of each top merge and of the root
inverse -- on this GPU, with the same descriptors a rank would launch for its
chunk (only the ncclAllGather between waves is absent, since every chunk is
already local). The result must equal the unsharded build."""
import numpy as np
import pytest

import paper_1302_5995_b200 as dtn
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("name,n,leaf", [("helmholtz", 514, 16), ("laplace", 258, 16), ("diffconv1", 130, 16)])
def test_collective_split_equals_full_build(world, name, n, leaf):
    spec = (dtn.baseline_problem(2, n - 2) if name == "helmholtz" else dtn.catalog(name, n, seed=1))
    op = dtn.discretize(spec)
    tree = dtn.build_tree_uniform(n, leaf)
    full = dtn.build_root_gpu(op, tree)
    col = dtn.build_root_gpu(op, tree, nshards=world, shard=-3)
    assert np.array_equal(col.boundary, full.boundary)
    assert rel(col.S_dense, full.S_dense) <= 1e-12
    nb = len(full.boundary)
    # G by column chunks (redundant LU + this chunk's substitutions) vs the getri-style inverse
    assert np.linalg.norm(full.S_dense @ col.G_dense - np.eye(nb)) / np.sqrt(nb) <= 1e-11 * max(1.0, full.cond_estimate)
    assert col.cond_estimate == pytest.approx(full.cond_estimate, rel=1e-6)


def test_collective_config2_vs_oracle():
    """BASELINE config 2 (Helmholtz kappa = 40, n = 512, 16 x 16 leaves) through the
    8-way split: S and Neumann data against the oracle at 1e-10."""
    n = 514
    op = dtn.discretize(dtn.baseline_problem(2, 512))
    col = dtn.build_root_gpu(op, dtn.build_tree_uniform(n, 16), nshards=8, shard=-3)
    ref = O.build_root_dense(O.Problem("helmholtz", n, 40.0), O.Tree(n, uniform_side=16), threads=16, mode=2)
    g = np.random.Generator(np.random.MT19937(1)).uniform(-1, 1, (len(ref.boundary), 16))
    assert rel(col.S_dense, ref.S) <= 1e-10
    assert rel(dtn.apply_schur(col, g), ref.S @ g) <= 1e-10


@pytest.mark.parametrize("world", [2, 8])
def test_collective_structured_shards(world):
    """Compressed engine over the split: structured shards, dense column-sharded top,
    compressed root -- S_hbs against the unsharded compressed build."""
    n = 514
    op = dtn.discretize(dtn.baseline_problem(2, 512))
    tree = dtn.build_tree_uniform(n, 16)
    opt = dtn.AccelOptions(epsilon=1e-10, crossover=256)
    a = dtn.build_root_accel(op, tree, opt)
    b = dtn.build_root_accel(op, tree, opt, nshards=world, collective=-3)
    g = np.random.Generator(np.random.MT19937(2)).uniform(-1, 1, (a.boundary_size(), 8))
    assert rel(dtn.apply_schur(b, g), dtn.apply_schur(a, g)) <= 1e-9


@pytest.mark.parametrize("world", [2, 8])
def test_collective_nccl_loopback(world):
    """shard = -4: the single-device split with every NCCL call of the real collective
    path (the shard-S all-gather, the grouped per-wave all-gathers captured in the build
    graph, the G column all-gather) issued in place on a 1-rank communicator the context
    owns -- checks the dlopen'ed NCCL entry points, ncclCommInitRank from a unique id and
    graph capture of the collectives on the one GPU available here."""
    ctx = dtn.Context(0, 1, 0, dtn.nccl_unique_id())
    n, leaf = 258, 16
    op = dtn.discretize(dtn.catalog("helmholtz1", n, seed=1))
    tree = dtn.build_tree_uniform(n, leaf)
    full = dtn.build_root_gpu(op, tree, ctx=ctx)
    for _ in range(2):  # second build: the cached plan's graph replays its collectives
        col = dtn.build_root_gpu(op, tree, nshards=world, shard=-4, ctx=ctx)
        assert rel(col.S_dense, full.S_dense) <= 1e-12
        nb = len(full.boundary)
        assert np.linalg.norm(full.S_dense @ col.G_dense - np.eye(nb)) / np.sqrt(nb) <= 1e-11 * max(1.0, full.cond_estimate)
        col.free()
    acc = dtn.build_root_accel(op, tree, dtn.AccelOptions(epsilon=1e-10, crossover=100, hbs_leaf=32), ctx=ctx,
                               nshards=world, collective=-4)
    g = np.random.default_rng(1).uniform(-1, 1, (len(full.boundary), 3))
    assert rel(dtn.apply_schur(acc, g), full.S_dense @ g) <= 1e-8
