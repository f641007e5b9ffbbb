"""Sharded GPU build on one device: every shard built by the B200
engine (dtn_gpu_build with opts.shard), then the top of the tree from the
shard S blocks (opts.shard = -1) — must equal the single build and the oracle.
The multi-process protocol itself is covered by tests/test_shard_gloo.py."""
import numpy as np
import pytest

import paper_1302_5995_b200 as dtn
from paper_1302_5995_b200 import shard as SH
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("nshards", [2, 4, 8])
@pytest.mark.parametrize("n_int,leaf", [(128, 16), (512, 16)])
def test_sharded_equals_full(nshards, n_int, leaf):
    import torch
    n = n_int + 2
    op = dtn.discretize(dtn.baseline_problem(2, n_int))
    tree = dtn.build_tree_uniform(n, leaf)
    eng = SH.GpuShardEngine(op, tree)
    blocks = [eng.build_shard(nshards, s) for s in range(nshards)]
    for s, b in enumerate(blocks):
        assert b.shape[0] == dtn.shard_info(tree, nshards, s)["nb"]
    top = eng.build_top(nshards, blocks)
    full = eng.build_full()
    assert O.rel_fro(top.S_dense, full.S_dense) <= 1e-12
    assert O.rel_fro(top.G_dense, full.G_dense) <= 1e-10
    if n_int <= 128:
        ref = O.build_root_dense(O.Problem("helmholtz", n, 40.0), O.Tree(n, uniform_side=leaf))
        assert O.rel_fro(top.S_dense, ref.S) <= 1e-10
    # host shard blocks work too
    top_h = eng.build_top(nshards, [b.cpu().numpy() for b in blocks])
    assert O.rel_fro(top_h.S_dense, full.S_dense) <= 1e-12


@pytest.mark.parametrize("nshards", [2, 8])
def test_sharded_compressed_root(nshards):
    """Sharded build with the compressed root on the top rank (BASELINE
    config 4's layout at n=512): S_hbs / G_hbs equal the unsharded compressed
    build's operators to 10 eps, and S_hbs g the dense S g."""
    n_int, leaf = 512, 16
    n = n_int + 2
    op = dtn.discretize(dtn.baseline_problem(4, n_int))
    tree = dtn.build_tree_uniform(n, leaf)
    opt = dtn.AccelOptions(epsilon=1e-10, crossover=256, hbs_leaf=64)
    eng = SH.GpuShardEngine(op, tree, accel=opt)
    blocks = [eng.build_shard(nshards, s) for s in range(nshards)]
    top = eng.build_top(nshards, blocks)
    assert isinstance(top, dtn.CompressedSolutionOperator)
    full = eng.build_full()
    dense = dtn.build_root_gpu(op, tree)
    g = np.random.default_rng(3).uniform(-1, 1, (len(dense.boundary), 8))
    Sg = dense.S_dense @ g
    assert O.rel_fro(dtn.apply_schur(top, g), Sg) <= 1e-9
    assert O.rel_fro(dtn.apply_schur(top, g), dtn.apply_schur(full, g)) <= 1e-9
    assert O.rel_fro(dtn.apply_dtn(top, Sg), g) <= 1e-9 * dense.cond_estimate
