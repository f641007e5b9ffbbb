"""The HBS oracle (oracle/hbs_oracle.py) against the reference's own HBS tests
(proj/tests/test_hbs.cpp:51-200), plus the DTNHBS01 byte layout and the
host-side index tree of the product package. CPU only."""
import struct

import numpy as np
import pytest

from oracle import hbs_oracle as HO
from oracle import oracle as O
from paper_1302_5995_b200 import hbs as PH


def rel_fro(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def test_index_tree_shapes():  # test_hbs.cpp:51-78
    t = HO.build_index_tree(400, 50)
    assert t.depth == 3
    assert (t.nodes[0].begin, t.nodes[0].end) == (0, 400)
    left = t.nodes[t.nodes[0].left]
    assert (left.begin, left.end) == (0, 200)
    leaves = [i for i in range(t.num_nodes()) if t.is_leaf(i)]
    assert len(leaves) == 8 and all(t.node_size(i) == 50 for i in leaves)
    assert HO.build_index_tree(50, 50).num_nodes() == 1
    t7 = HO.build_index_tree(7, 2)
    assert [t7.node_size(i) for i in range(t7.num_nodes()) if t7.is_leaf(i)] == [2, 2, 2, 1]


@pytest.mark.parametrize("M,cap", [(400, 50), (7, 2), (2044, 64), (8188, 64), (37, 4), (1, 2)])
def test_product_index_tree_matches_oracle(M, cap):
    a, b = PH.build_index_tree(M, cap), HO.build_index_tree(M, cap)
    assert a.depth == b.depth and a.num_nodes() == b.num_nodes()
    for x, y in zip(a.nodes, b.nodes):
        assert (x.begin, x.end, x.left, x.right, x.parent, x.level) == \
            (y.begin, y.end, y.left, y.right, y.parent, y.level)


def test_identity_rank_zero():  # test_hbs.cpp:88-100
    h = HO.compress(np.eye(96), 1e-10, 16)
    assert h.max_rank() == 0
    assert rel_fro(HO.reconstruct(h), np.eye(96)) <= 1e-14


def test_rank_one():  # test_hbs.cpp:102-108
    rng = np.random.default_rng(1)
    u, v = rng.standard_normal((80, 1)), rng.standard_normal((80, 1))
    H = u @ v.T
    c = HO.compress(H, 1e-10, 16)
    assert c.max_rank() <= 1
    assert rel_fro(HO.reconstruct(c), H) <= 1e-12


def test_laplace_root_schur():  # test_hbs.cpp:110-116
    S = O.build_root_dense(O.Problem("laplace", 64), O.Tree(64, 4096)).S
    h = HO.compress(S, 1e-7, 64)
    assert rel_fro(HO.reconstruct(h), S) <= 1e-6
    assert h.max_rank() < S.shape[0] / 4
    assert HO.orthonormality_defect(h) <= 1e-12


def test_apply_matches_dense():  # test_hbs.cpp:118-125
    H = HO.kernel_matrix(150, 3)
    c = HO.compress(H, 1e-9, 32)
    x = np.random.default_rng(4).standard_normal((150, 3))
    assert rel_fro(HO.apply(c, x), H @ x) <= 1e-8
    assert np.linalg.norm(HO.apply(c, np.zeros((150, 2)))) == 0.0


@pytest.mark.parametrize("eps", [1e-4, 1e-7, 1e-10])
@pytest.mark.parametrize("seed", [11, 12, 13])
def test_roundtrip_budget(eps, seed):  # test_hbs.cpp:127-136
    H = HO.kernel_matrix(130, seed)
    c = HO.compress(H, eps, 16)
    assert rel_fro(HO.reconstruct(c), H) <= 10.0 * eps * (c.tree.depth + 1)
    assert HO.orthonormality_defect(c) <= 1e-12


def test_ranks_monotone():  # test_hbs.cpp:138-146
    H = HO.kernel_matrix(128, 5)
    tree = HO.build_index_tree(128, 16)
    loose, tight = HO.compress(H, 1e-4, tree=tree), HO.compress(H, 1e-9, tree=tree)
    assert all(loose.rank(t) <= tight.rank(t) for t in range(1, tree.num_nodes()))


def test_serialization_layout_and_roundtrip():  # test_hbs.cpp:177-196, hbs.cpp:446-505
    H = HO.kernel_matrix(90, 9)
    c = HO.compress(H, 1e-8, 16)
    b1, b2 = HO.serialize(c), HO.serialize(HO.compress(H, 1e-8, 16))
    assert b1 == b2
    assert b1[:8] == b"DTNHBS01"
    M, nn, depth = struct.unpack_from("<qqq", b1, 8)
    assert (M, nn, depth) == (90, c.tree.num_nodes(), c.tree.depth)
    # node table then, for node 0 (a parent), its B matrix header
    off = 32 + 48 * nn
    r, cc = struct.unpack_from("<qq", b1, off)
    assert (r, cc) == c.B[0].shape
    back = HO.deserialize(b1)
    assert rel_fro(HO.reconstruct(back), HO.reconstruct(c)) == 0.0
    with pytest.raises(ValueError):
        HO.deserialize(bytes([1, 2, 3]))


def test_exported_hbs_symbols():
    import ctypes
    from paper_1302_5995_b200 import _lib
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in ("dtn_gpu_hbs_compress", "dtn_gpu_hbs_compress_op", "dtn_gpu_hbs_apply", "dtn_gpu_hbs_serialize",
                 "dtn_gpu_hbs_deserialize", "dtn_gpu_hbs_info", "dtn_gpu_hbs_tree", "dtn_gpu_hbs_factor",
                 "dtn_gpu_hbs_free"):
        assert hasattr(lib, name), name


# ---- multi-level inversion (hbs_ops.cpp:148-205), pinned to test_hbs_ops.cpp:164-216 ----

def test_invert_diagonal_divides_elementwise():  # test_hbs_ops.cpp:164-172
    d = 1.0 + (np.arange(64) % 7)
    inv = HO.invert_hbs(HO.compress(np.diag(d), 1e-12, 16))
    x = np.linspace(-1.0, 2.0, 64)
    assert np.linalg.norm(HO.apply_inverse(inv, x) - x / d) <= 1e-12


def test_invert_two_level_synthetic():  # test_hbs_ops.cpp:174-180
    h = HO.synthetic_hbs(16, 4, 2, 6)
    dense = HO.reconstruct(h)
    g = HO.apply_inverse(HO.invert_hbs(h), np.eye(16))
    assert rel_fro(g, np.linalg.inv(dense)) <= 1e-9


def test_invert_compressed_laplace_schur():  # test_hbs_ops.cpp:182-190
    S = O.build_root_dense(O.Problem("laplace", 64), O.Tree(64, 4096)).S
    h = HO.compress(S, 1e-7, 64)
    x = np.random.default_rng(7).standard_normal((S.shape[0], 2))
    back = HO.apply(h, HO.apply_inverse(HO.invert_hbs(h), x))
    assert np.linalg.norm(back - x) / np.linalg.norm(x) <= 1e-5


@pytest.mark.parametrize("n", [32, 64])
def test_invert_residual_within_100_eps(n):  # test_hbs_ops.cpp:192-203
    eps = 1e-7
    S = O.build_root_dense(O.Problem("laplace", n), O.Tree(n, 4096)).S
    h = HO.compress(S, eps, 32)
    x = np.random.default_rng(8).standard_normal((S.shape[0], 1))
    back = HO.apply(h, HO.apply_inverse(HO.invert_hbs(h), x))
    assert np.linalg.norm(back - x) / np.linalg.norm(x) <= 100 * eps


def test_invert_names_failing_node():  # test_hbs_ops.cpp:205-216
    h = HO.synthetic_hbs(16, 4, 2, 9)
    for t in range(h.tree.num_nodes()):
        if h.tree.is_leaf(t):
            h.D[t][:] = 0.0
            break
    with pytest.raises(HO.FactorizationError, match="node"):
        HO.invert_hbs(h)
