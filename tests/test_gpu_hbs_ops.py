"""The HBS algebra on the device (csrc/hbs_ops.cu through the C ABI:
dtn_gpu_hbs_flip / _subtree / _scale* / _add / _from_lowrank / _add_lowrank /
_rebase / _split_at / _consolidate, dtn_gpu_lowrank_*) against the numpy
restatement of hbs.cpp / hbs_ops.cpp / lowrank.cpp (oracle/accel_oracle.py) and the
reference's own properties (proj/tests/test_hbs_ops.cpp:221-353).

Factor transforms (flip, subtree, scale) are data movement: bit-identical to the
oracle on the same factors (the GPU operand is the oracle's HBS shipped as
DTNHBS01 bytes). Re-compressing operations agree with the oracle's results within
the compression tolerance and reproduce the oracle's index trees exactly."""
import numpy as np
import pytest

from oracle import accel_oracle as AO
from oracle import hbs_oracle as HO

pytestmark = pytest.mark.gpu


def rel_fro(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.fixture(scope="module")
def H():
    from paper_1302_5995_b200 import hbs
    return hbs


def to_gpu(H, h):
    return H.deserialize(HO.serialize(h))


def same_tree(gtree, otree):
    return len(gtree.nodes) == len(otree.nodes) and all(
        (a.begin, a.end, a.left, a.right, a.parent, a.level) == (b.begin, b.end, b.left, b.right, b.parent, b.level)
        for a, b in zip(gtree.nodes, otree.nodes))


def assert_factors_equal(g, o):
    """every factor bit-identical (the GPU HbsMatrix vs the oracle Hbs)"""
    assert same_tree(g.tree, o.tree)
    for t in range(o.tree.num_nodes()):
        if o.tree.is_leaf(t):
            assert np.array_equal(g.factor(t, "D"), o.D[t]), ("D", t)
        else:
            assert np.array_equal(g.factor(t, "B"), o.B[t]), ("B", t)
        if t != 0:
            assert np.array_equal(g.factor(t, "U"), o.U[t]), ("U", t)
            assert np.array_equal(g.factor(t, "V"), o.V[t]), ("V", t)


@pytest.fixture(scope="module")
def ref100():
    a = HO.kernel_matrix(100, 18)
    return a, HO.compress(a, 1e-9, 16)


# ---------------------------------------------------------------- exact factor transforms
def test_flip_bit_identical(H, ref100):  # hbs.cpp:322-375
    a, h = ref100
    g = H.flip(to_gpu(H, h))
    o = AO.flip(h)
    assert_factors_equal(g, o)
    assert same_tree(g.tree, H.mirror(to_gpu(H, h).tree))
    P = np.eye(100)[::-1]
    assert rel_fro(H.reconstruct(g), P @ HO.reconstruct(h) @ P) <= 1e-14


def test_flip_twice_is_identity(H, ref100):
    _, h = ref100
    g = to_gpu(H, h)
    assert_factors_equal(H.flip(H.flip(g)), h)


@pytest.mark.parametrize("t", [0, 1, 2, 5])
def test_subtree_bit_identical(H, ref100, t):  # hbs.cpp:290-320
    _, h = ref100
    assert_factors_equal(H.subtree_matrix(to_gpu(H, h), t), AO.subtree_matrix(h, t))


def test_scale_bit_identical(H, ref100):  # hbs.cpp:377-402
    _, h = ref100
    rng = np.random.default_rng(3)
    wr, wc = rng.uniform(0.5, 2.0, 100), rng.uniform(0.5, 2.0, 100)
    g = to_gpu(H, h)
    H.scale_rows(g, wr)
    H.scale_cols(g, wc)
    H.scale(g, -0.75)
    o = HO.deserialize(HO.serialize(h))
    AO.scale_rows(o, wr)
    AO.scale_cols(o, wc)
    AO.scale(o, -0.75)
    assert_factors_equal(g, o)
    # the apply path sees the new factors (its packed copy is invalidated)
    ref = -0.75 * (wr[:, None] * HO.reconstruct(h) * wc[None, :])
    assert rel_fro(H.reconstruct(g), ref) <= 1e-13
    x = rng.standard_normal((100, 3))
    assert rel_fro(H.apply(g, x), ref @ x) <= 1e-13


def test_scale_single_node(H):
    a = np.random.default_rng(5).standard_normal((12, 12))
    g = H.compress(a, 1e-10, 64)  # one node, stored densely
    w = np.arange(1.0, 13.0)
    H.scale_rows(g, w)
    assert np.array_equal(H.reconstruct(g), w[:, None] * a)


# ---------------------------------------------------------------- addition (hbs_ops.cpp:386-404)
def test_add_zero_preserves(H):  # test_hbs_ops.cpp:221-231
    a = HO.kernel_matrix(96, 10)
    ha = H.compress(a, 1e-7, 16)
    zero = H.compress(np.zeros((96, 96)), 1e-7, 16)
    assert zero.max_rank() == 0
    s = H.add_hbs(ha, zero, 1e-7)
    assert rel_fro(H.reconstruct(s), a) <= 1e-6
    for t in range(1, ha.tree.num_nodes()):
        assert s.rank(t) == ha.rank(t), t


def test_add_negative_is_rank_zero(H):  # test_hbs_ops.cpp:233-242
    a = HO.kernel_matrix(80, 11)
    ha = H.compress(a, 1e-9, 16)
    neg = H.deserialize(H.serialize(ha))
    H.scale(neg, -1.0)
    s = H.add_hbs(ha, neg, 1e-9)
    assert s.max_rank() == 0
    assert np.linalg.norm(H.reconstruct(s)) <= 1e-9 * np.linalg.norm(a)


def test_add_matches_dense_and_commutes(H):  # test_hbs_ops.cpp:244-256
    a, b = HO.kernel_matrix(120, 12), HO.kernel_matrix(120, 13)
    eps = 1e-8
    ha, hb = H.compress(a, eps, 16), H.compress(b, eps, 16)
    ab, ba = H.add_hbs(ha, hb, eps), H.add_hbs(hb, ha, eps)
    assert rel_fro(H.reconstruct(ab), a + b) <= 10 * eps
    assert rel_fro(H.reconstruct(ab), H.reconstruct(ba)) <= 1e-12
    assert H.basis_orthonormality_defect(ab) <= 1e-12
    # the oracle's add_hbs (stack_sum + orthonormalize + truncate) on the oracle's operands
    o = AO.add_hbs(HO.compress(a, eps, 16), HO.compress(b, eps, 16), eps)
    assert rel_fro(H.reconstruct(ab), HO.reconstruct(o)) <= 10 * eps
    assert same_tree(ab.tree, o.tree)
    assert max(abs(ab.rank(t) - o.rank(t)) for t in range(1, o.tree.num_nodes())) <= 2


def test_add_rejects_mismatched_trees(H):  # test_hbs_ops.cpp:258-263
    a = HO.kernel_matrix(64, 14)
    with pytest.raises(ValueError, match="different index trees"):
        H.add_hbs(H.compress(a, 1e-8, 16), H.compress(a, 1e-8, 32), 1e-8)


# ---------------------------------------------------------------- low-rank conversion (hbs_ops.cpp:409-470)
def test_lowrank_conversion_exact(H):  # test_hbs_ops.cpp:265-286
    tree = H.build_index_tree(64, 8)
    rng = np.random.default_rng(15)
    zero = H.lowrank_to_bs(np.zeros((64, 0)), np.zeros((0, 64)), tree)
    assert np.linalg.norm(H.reconstruct(zero)) == 0.0
    u, v = rng.standard_normal((64, 1)), rng.standard_normal((1, 64))
    r1 = H.lowrank_to_bs(u, v, tree)
    assert r1.max_rank() <= 1
    assert np.abs(H.reconstruct(r1) - u @ v).max() <= 1e-12
    q, r = rng.standard_normal((64, 3)), rng.standard_normal((3, 64))
    r3 = H.lowrank_to_bs(q, r, tree)
    assert r3.max_rank() <= 3
    assert rel_fro(H.reconstruct(r3), q @ r) <= 1e-12
    assert H.basis_orthonormality_defect(r3) <= 1e-12
    assert same_tree(r3.tree, tree)
    o = AO.lowrank_to_bs(q, r, HO.build_index_tree(64, 8))
    assert rel_fro(H.reconstruct(r3), HO.reconstruct(o)) <= 1e-12


def test_add_lowrank(H):  # test_hbs_ops.cpp:288-302
    a = HO.kernel_matrix(72, 16)
    eps = 1e-8
    ha = H.compress(a, eps, 8)
    same = H.add_lowrank(ha, np.zeros((72, 0)), np.zeros((0, 72)), eps)
    assert rel_fro(H.reconstruct(same), a) <= 10 * eps
    rng = np.random.default_rng(17)
    q, r = rng.standard_normal((72, 2)), rng.standard_normal((2, 72))
    s = H.add_lowrank(ha, q, r, eps)
    assert rel_fro(H.reconstruct(s), a + q @ r) <= 10 * eps


# ---------------------------------------------------------------- split / consolidate / rebase
@pytest.mark.parametrize("pos", [1, 13, 50, 77, 99])
def test_split_reassembles(H, ref100, pos):  # test_hbs_ops.cpp:304-334
    _, h = ref100
    g = to_gpu(H, h)
    sp = H.split_at(g, pos, 1e-13)
    back = np.zeros((100, 100))
    back[:pos, :pos] = H.reconstruct(sp.lo)
    back[pos:, pos:] = H.reconstruct(sp.hi)
    back[:pos, pos:] = sp.lo_hi.dense()
    back[pos:, :pos] = sp.hi_lo.dense()
    assert rel_fro(back, HO.reconstruct(h)) <= 1e-11
    # both sides on the oracle's consolidated (spine) trees
    lo, hi, _, _ = AO.split_at(h, pos)
    assert same_tree(sp.lo.tree, AO.consolidate(lo, 1e-9).tree)
    assert same_tree(sp.hi.tree, AO.consolidate(hi, 1e-9).tree)


def test_split_at_ends(H, ref100):
    _, h = ref100
    g = to_gpu(H, h)
    s0 = H.split_at(g, 0)
    assert s0.lo is None and s0.lo_hi.rank() == 0
    assert_factors_equal(s0.hi, h)
    with pytest.raises(ValueError):
        H.split_at(g, 101)


def test_consolidation(H):  # test_hbs_ops.cpp:336-344
    a = HO.kernel_matrix(90, 19)
    h = HO.compress(a, 1e-9, 16)
    sp = H.split_at(to_gpu(H, h), 37, 1e-9)
    assert rel_fro(H.reconstruct(sp.lo), HO.reconstruct(h)[:37, :37]) <= 1e-7
    assert H.basis_orthonormality_defect(sp.lo) <= 1e-12


def test_consolidate_pieces_and_corrections(H, ref100):  # hbs_ops.cpp:710-735
    _, h = ref100
    g = to_gpu(H, h)
    full = HO.reconstruct(h)
    l, r = h.tree.nodes[0].left, h.tree.nodes[0].right
    mid = h.tree.nodes[l].end
    pieces = [H.subtree_matrix(g, l), H.subtree_matrix(g, r)]
    corr = [H.Placed(0, mid, H.lowrank_from_dense(full[:mid, mid:], 1e-14)),
            H.Placed(mid, 0, H.lowrank_from_dense(full[mid:, :mid], 1e-14))]
    c = H.consolidate(pieces, [0, mid], corr, 1e-12)
    assert same_tree(c.tree, h.tree)
    assert rel_fro(H.reconstruct(c), full) <= 1e-11
    assert H.basis_orthonormality_defect(c) <= 1e-12
    # one piece, no corrections: the piece itself (bit-identical copy)
    assert_factors_equal(H.consolidate([g], [0]), h)
    with pytest.raises(ValueError, match="tile"):
        H.consolidate(pieces, [0, mid + 1], size=100)


def test_rebase(H):  # test_hbs_ops.cpp:346-353
    a = HO.kernel_matrix(84, 20)
    h = H.compress(a, 1e-9, 32)
    target = H.build_index_tree(84, 8)
    r = H.rebase(h, target, 1e-9)
    assert r.tree == target
    assert rel_fro(H.reconstruct(r), a) <= 1e-7
    same = H.rebase(h, h.tree, 1e-9)
    assert np.array_equal(H.reconstruct(same), H.reconstruct(h))


def test_compress_onto_tree(H):  # compress(H, tree, eps): the mirrored tree of a flip
    a = HO.kernel_matrix(100, 21)
    tree = H.mirror(H.build_index_tree(100, 16))
    c = H.compress(a, 1e-10, tree=tree)
    assert c.tree == tree
    assert rel_fro(H.reconstruct(c), a) <= 1e-9
    o = HO.compress(a, 1e-10, tree=AO.mirror(HO.build_index_tree(100, 16)))
    assert max(abs(c.rank(t) - o.rank(t)) for t in range(1, o.tree.num_nodes())) <= 2


# ---------------------------------------------------------------- low-rank blocks (lowrank.cpp)
def test_lowrank_from_dense_and_recompress(H):
    rng = np.random.default_rng(22)
    X = rng.standard_normal((300, 5)) @ rng.standard_normal((5, 170))
    lr = H.lowrank_from_dense(X, 1e-12)
    assert lr.rank() == 5
    assert rel_fro(lr.dense(), X) <= 1e-12
    # a redundant representation recompresses to the numerical rank
    Lf = np.hstack([lr.L, lr.L])
    R = np.vstack([0.5 * lr.R, 0.5 * lr.R])
    rc = H.lowrank_recompress(H.LowRank.from_factors(Lf, R), 1e-12)
    assert rc.rank() == 5 and rel_fro(rc.dense(), X) <= 1e-12
    o = AO.lowrank_from_dense(X, 1e-12)
    assert o.rank() == lr.rank()
    # wide blocks (min dimension above the 256-column QR): the randomized path
    Y = rng.standard_normal((400, 7)) @ rng.standard_normal((7, 600))
    ly = H.lowrank_from_dense(Y, 1e-12)
    assert ly.rank() == 7 and rel_fro(ly.dense(), Y) <= 1e-11
    z = H.lowrank_from_dense(np.zeros((20, 30)), 1e-12)
    assert z.rank() == 0


def test_lowrank_sum(H):  # lowrank.cpp:58-72
    rng = np.random.default_rng(23)
    terms, ref = [], np.zeros((60, 50))
    oterms = []
    for (r0, c0, m, n, k) in [(0, 0, 30, 20, 2), (10, 25, 40, 25, 3), (0, 0, 60, 50, 1)]:
        Lf, R = rng.standard_normal((m, k)), rng.standard_normal((k, n))
        terms.append(H.Placed(r0, c0, H.LowRank.from_factors(Lf, R)))
        oterms.append(AO.Placed(r0, c0, AO.LowRank(Lf, R)))
        ref[r0:r0 + m, c0:c0 + n] += Lf @ R
    s = H.lowrank_sum(60, 50, terms, 1e-12)
    assert rel_fro(s.dense(), ref) <= 1e-12
    o = AO.lowrank_sum(60, 50, oterms, 1e-12)
    assert s.rank() == o.rank() == 6
