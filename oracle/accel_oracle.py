"""TEST INFRASTRUCTURE ONLY -- a CPU restatement of the reference's compressed
(accelerated) engine, build_root_accel (proj/src/accel_nd.cpp:707-859), with the
HBS arithmetic it needs (proj/src/hbs.cpp flip/scale/subtree, proj/src/hbs_ops.cpp
add_hbs / lowrank_to_bs / split_at / consolidate / rebase, proj/src/lowrank.cpp,
proj/src/index_tree.cpp mirror/spine). Only tests/ and bench.py's CPU legs may
use it; the product path never does.

It follows the reference's data flow step by step -- boxes at or above the
crossover carry a StructuredSchur ([J;K] boundary, HBS s_jj / s_kk, low-rank
s_jk / s_kj), merge_pair densifies mixed pairs, accel_merge runs the paper's Steps
1-3 with HBS inversion, flip/scale/rebase/add_hbs, low-rank T-terms, split_at /
consolidate of the kept blocks and lowrank_sum of the couplings -- on top of the
C++ dense oracle (leaf_schur, merge_two: oracle.py) and the numpy HBS oracle
(compress, apply, invert_hbs: hbs_oracle.py). Eigen's BDCSVD / HouseholderQR /
FullPivLU become LAPACK's gesdd / geqrf / getrf through numpy: factors agree to
rounding, ranks except at exact ties with a cutoff.

Pinned to the reference's own engine-equivalence tests (test_accel_nd.cpp:26-149:
compress_box 1e-5, one structured merge vs dense 1e-5, engine equivalence 1e-4 at
eps 1e-7) and acceptance criterion 2 (acceptance.cpp:116-146) in
tests/test_accel_oracle.py, against the dense oracle.
"""
from __future__ import annotations

import time

import numpy as np

from . import hbs_oracle as HO
from . import oracle as O

NONE, NORTH, SOUTH, EAST, WEST = 0, 1, 2, 3, 4


# ------------------------------------------------------------------ low rank (lowrank.cpp)
class LowRank:
    __slots__ = ("L", "R")

    def __init__(self, L, R):
        self.L, self.R = L, R

    def rows(self):
        return self.L.shape[0]

    def cols(self):
        return self.R.shape[1]

    def rank(self):
        return self.L.shape[1]

    def dense(self):
        return self.L @ self.R

    def block(self, r0, nr, c0, nc):
        return LowRank(self.L[r0:r0 + nr], self.R[:, c0:c0 + nc])

    @staticmethod
    def zero(m, n):
        return LowRank(np.zeros((m, 0)), np.zeros((0, n)))


def _trunc_rank(sigma, eps, floor=0.0):  # lowrank.cpp:9-16, hbs_ops.cpp:14-20
    if sigma.size == 0 or sigma[0] <= floor:
        return 0
    cut = max(eps * sigma[0], floor)
    return int(np.count_nonzero(sigma > cut))


def lowrank_from_dense(X, eps):  # lowrank.cpp:27-36
    if X.shape[0] == 0 or X.shape[1] == 0:
        return LowRank.zero(*X.shape)
    u, s, vt = np.linalg.svd(X, full_matrices=False)
    k = _trunc_rank(s, eps)
    return LowRank(u[:, :k].copy(), s[:k, None] * vt[:k])


def _thin_qr(a):  # hbs_ops.cpp:279-285
    r = min(a.shape)
    if a.shape[1] == 0:
        return np.zeros((a.shape[0], 0)), np.zeros((0, 0))
    q, rr = np.linalg.qr(a, mode="reduced")
    return q[:, :r], rr[:r]


def lowrank_recompress(x: LowRank, eps):  # lowrank.cpp:38-56
    if x.rank() == 0:
        return x
    ql, rl = _thin_qr(x.L)
    qr_, rr = _thin_qr(x.R.T)
    u, s, vt = np.linalg.svd(rl @ rr.T, full_matrices=False)
    k = _trunc_rank(s, eps)
    return LowRank(ql @ u[:, :k], s[:k, None] * (qr_ @ vt[:k].T).T)


class Placed:
    __slots__ = ("row_offset", "col_offset", "lr")

    def __init__(self, r, c, lr):
        self.row_offset, self.col_offset, self.lr = r, c, lr


def lowrank_sum(m, n, terms, eps):  # lowrank.cpp:58-72
    ktot = sum(t.lr.rank() for t in terms)
    if ktot == 0:
        return LowRank.zero(m, n)
    l = np.zeros((m, ktot))
    r = np.zeros((ktot, n))
    at = 0
    for t in terms:
        k = t.lr.rank()
        l[t.row_offset:t.row_offset + t.lr.rows(), at:at + k] = t.lr.L
        r[at:at + k, t.col_offset:t.col_offset + t.lr.cols()] = t.lr.R
        at += k
    return lowrank_recompress(LowRank(l, r), eps)


# ------------------------------------------------------------------ trees (index_tree.cpp)
def single_node_tree(M):
    return HO.Tree([HO.Node(0, M, -1, -1, -1, 0)], 0)


def trees_equal(a, b):  # index_tree.cpp:19-31
    if len(a.nodes) != len(b.nodes):
        return False
    return all(x.begin == y.begin and x.end == y.end and x.left == y.left and x.right == y.right
               for x, y in zip(a.nodes, b.nodes))


def mirror(tree):  # index_tree.cpp:71-93
    M = tree.size()
    out = []
    depth = [0]

    def rec(t, parent, level):
        n = tree.nodes[t]
        i = len(out)
        out.append(HO.Node(M - n.end, M - n.begin, -1, -1, parent, level))
        depth[0] = max(depth[0], level)
        if n.left >= 0:
            l_ = rec(n.right, i, level + 1)
            r_ = rec(n.left, i, level + 1)
            out[i].left, out[i].right = l_, r_
        return i

    rec(0, -1, 0)
    return HO.Tree(out, depth[0])


def _node_rows(h, t):
    tr = h.tree
    if tr.is_leaf(t):
        return tr.node_size(t)
    return h.rank(tr.nodes[t].left) + h.rank(tr.nodes[t].right)


# ------------------------------------------------------------------ HBS transforms (hbs.cpp)
def apply_col_basis(h, t, X):  # hbs.cpp:234-244
    if h.tree.is_leaf(t):
        return h.U[t] @ X
    c1, c2 = h.tree.nodes[t].left, h.tree.nodes[t].right
    y = h.U[t] @ X
    k1 = h.rank(c1)
    return np.vstack([apply_col_basis(h, c1, y[:k1]), apply_col_basis(h, c2, y[k1:])])


def apply_row_basis(h, t, X):  # hbs.cpp:246-256
    if h.tree.is_leaf(t):
        return h.V[t] @ X
    c1, c2 = h.tree.nodes[t].left, h.tree.nodes[t].right
    y = h.V[t] @ X
    k1 = h.rank(c1)
    return np.vstack([apply_row_basis(h, c1, y[:k1]), apply_row_basis(h, c2, y[k1:])])


def _new_like(nodes, depth):
    h = HO.Hbs(HO.Tree(nodes, depth))
    return h


def subtree_matrix(h, t):  # hbs.cpp:290-320
    nodes, D, U, V, B = [], [], [], [], []
    depth = [0]
    off = h.tree.nodes[t].begin

    def rec(s, parent, level):
        n = h.tree.nodes[s]
        i = len(nodes)
        nodes.append(HO.Node(n.begin - off, n.end - off, -1, -1, parent, level))
        depth[0] = max(depth[0], level)
        D.append(h.D[s])
        U.append(None if i == 0 else h.U[s])
        V.append(None if i == 0 else h.V[s])
        B.append(h.B[s])
        if n.left >= 0:
            l_ = rec(n.left, i, level + 1)
            r_ = rec(n.right, i, level + 1)
            nodes[i].left, nodes[i].right = l_, r_
        return i

    rec(t, -1, 0)
    out = HO.Hbs(HO.Tree(nodes, depth[0]))
    out.D, out.U, out.V, out.B = D, U, V, B
    return out


def flip(h):  # hbs.cpp:322-375
    M = h.tree.size()
    nodes, D, U, V, B = [], [], [], [], []
    depth = [0]

    def rec(t, parent, level):
        n = h.tree.nodes[t]
        i = len(nodes)
        nodes.append(HO.Node(M - n.end, M - n.begin, -1, -1, parent, level))
        depth[0] = max(depth[0], level)
        if n.left < 0:
            D.append(h.D[t][::-1, ::-1].copy())
            U.append(None if i == 0 else h.U[t][::-1].copy())
            V.append(None if i == 0 else h.V[t][::-1].copy())
            B.append(None)
            return i
        k1, k2 = h.rank(n.left), h.rank(n.right)
        D.append(None)
        if i == 0:
            U.append(None)
            V.append(None)
        else:
            U.append(np.vstack([h.U[t][k1:], h.U[t][:k1]]))
            V.append(np.vstack([h.V[t][k1:], h.V[t][:k1]]))
        b = np.empty((k1 + k2, k1 + k2))
        bt = h.B[t]
        b[:k2, :k2] = bt[k1:, k1:]
        b[:k2, k2:] = bt[k1:, :k1]
        b[k2:, :k2] = bt[:k1, k1:]
        b[k2:, k2:] = bt[:k1, :k1]
        B.append(b)
        l_ = rec(n.right, i, level + 1)
        r_ = rec(n.left, i, level + 1)
        nodes[i].left, nodes[i].right = l_, r_
        return i

    rec(0, -1, 0)
    out = HO.Hbs(HO.Tree(nodes, depth[0]))
    out.D, out.U, out.V, out.B = D, U, V, B
    return out


def scale_rows(h, w):  # hbs.cpp:377-386
    for t in range(h.tree.num_nodes()):
        if not h.tree.is_leaf(t):
            continue
        nd = h.tree.nodes[t]
        d = w[nd.begin:nd.end][:, None]
        h.D[t] = d * h.D[t]
        if t != 0:
            h.U[t] = d * h.U[t]


def scale_cols(h, w):  # hbs.cpp:388-397
    for t in range(h.tree.num_nodes()):
        if not h.tree.is_leaf(t):
            continue
        nd = h.tree.nodes[t]
        d = w[nd.begin:nd.end]
        h.D[t] = h.D[t] * d[None, :]
        if t != 0:
            h.V[t] = d[:, None] * h.V[t]


def scale(h, s):  # hbs.cpp:399-402
    h.D = [None if m is None else m * s for m in h.D]
    h.B = [None if m is None else m * s for m in h.B]


# ------------------------------------------------------------------ addition (hbs_ops.cpp)
def _stack_sum(A, Bm):  # hbs_ops.cpp:213-262
    tree = A.tree
    C = HO.Hbs(tree)
    for t in range(tree.num_nodes()):
        if tree.is_leaf(t):
            C.D[t] = A.D[t] + Bm.D[t]
            if t != 0:
                C.U[t] = np.hstack([A.U[t], Bm.U[t]])
                C.V[t] = np.hstack([A.V[t], Bm.V[t]])
            continue
        c1, c2 = tree.nodes[t].left, tree.nodes[t].right
        ka1, kb1, ka2, kb2 = A.rank(c1), Bm.rank(c1), A.rank(c2), Bm.rank(c2)
        rows = ka1 + kb1 + ka2 + kb2
        if t != 0:
            ka, kb = A.rank(t), Bm.rank(t)
            u = np.zeros((rows, ka + kb))
            v = np.zeros((rows, ka + kb))
            for dst, src_a, src_b in ((u, A.U[t], Bm.U[t]), (v, A.V[t], Bm.V[t])):
                dst[0:ka1, 0:ka] = src_a[:ka1]
                dst[ka1:ka1 + kb1, ka:] = src_b[:kb1]
                dst[ka1 + kb1:ka1 + kb1 + ka2, 0:ka] = src_a[ka1:]
                dst[ka1 + kb1 + ka2:, ka:] = src_b[kb1:]
            C.U[t], C.V[t] = u, v
        bn = np.zeros((rows, rows))
        a_, b_ = A.B[t], Bm.B[t]
        i1, j1, i2, j2 = 0, ka1, ka1 + kb1, ka1 + kb1 + ka2  # slot starts: a1 b1 a2 b2
        bn[i1:i1 + ka1, i1:i1 + ka1] = a_[:ka1, :ka1]
        bn[i1:i1 + ka1, i2:i2 + ka2] = a_[:ka1, ka1:]
        bn[i2:i2 + ka2, i1:i1 + ka1] = a_[ka1:, :ka1]
        bn[i2:i2 + ka2, i2:i2 + ka2] = a_[ka1:, ka1:]
        bn[j1:j1 + kb1, j1:j1 + kb1] = b_[:kb1, :kb1]
        bn[j1:j1 + kb1, j2:j2 + kb2] = b_[:kb1, kb1:]
        bn[j2:j2 + kb2, j1:j1 + kb1] = b_[kb1:, :kb1]
        bn[j2:j2 + kb2, j2:j2 + kb2] = b_[kb1:, kb1:]
        C.B[t] = bn
    return C


def _fold(H, t, tu, tv):  # hbs_ops.cpp:264-277 fold_child_transforms
    c1, c2 = H.tree.nodes[t].left, H.tree.nodes[t].right
    o1, o2 = tu[c1].shape[1], tu[c2].shape[1]
    n1, n2 = tu[c1].shape[0], tu[c2].shape[0]
    if t != 0:
        H.U[t] = np.vstack([tu[c1] @ H.U[t][:o1], tu[c2] @ H.U[t][o1:]])
        H.V[t] = np.vstack([tv[c1] @ H.V[t][:o1], tv[c2] @ H.V[t][o1:]])
    b = H.B[t]
    nb = np.empty((n1 + n2, n1 + n2))
    nb[:n1, :n1] = tu[c1] @ b[:o1, :o1] @ tv[c1].T
    nb[:n1, n1:] = tu[c1] @ b[:o1, o1:] @ tv[c2].T
    nb[n1:, :n1] = tu[c2] @ b[o1:, :o1] @ tv[c1].T
    nb[n1:, n1:] = tu[c2] @ b[o1:, o1:] @ tv[c2].T
    H.B[t] = nb


def _orthonormalize(H):  # hbs_ops.cpp:287-305
    if H.tree.num_nodes() == 1:
        return
    N = H.tree.num_nodes()
    tu, tv = [None] * N, [None] * N
    for t in H.tree.bottom_up():
        if not H.tree.is_leaf(t):
            _fold(H, t, tu, tv)
        if t == 0:
            break
        qu, ru = _thin_qr(H.U[t])
        qv, rv = _thin_qr(H.V[t])
        H.U[t], H.V[t], tu[t], tv[t] = qu, qv, ru, rv


def _truncate(H, eps, floor):  # hbs_ops.cpp:307-375
    tree = H.tree
    if tree.num_nodes() == 1:
        return
    N = tree.num_nodes()
    wrow, wcol = [None] * N, [None] * N
    for t in range(N):  # top-down
        if tree.is_leaf(t):
            continue
        c1, c2 = tree.nodes[t].left, tree.nodes[t].right
        k1, k2 = H.rank(c1), H.rank(c2)
        bt = H.B[t]
        parts_r1 = [bt[:k1, k1:], bt[:k1, :k1]]
        parts_r2 = [bt[k1:, :k1], bt[k1:, k1:]]
        parts_c1 = [bt[k1:, :k1].T, bt[:k1, :k1].T]
        parts_c2 = [bt[:k1, k1:].T, bt[k1:, k1:].T]
        if t != 0:
            parts_r1.append(H.U[t][:k1] @ wrow[t])
            parts_r2.append(H.U[t][k1:] @ wrow[t])
            parts_c1.append(H.V[t][:k1] @ wcol[t])
            parts_c2.append(H.V[t][k1:] @ wcol[t])
        wrow[c1], wrow[c2] = np.hstack(parts_r1), np.hstack(parts_r2)
        wcol[c1], wcol[c2] = np.hstack(parts_c1), np.hstack(parts_c2)
    tu, tv = [None] * N, [None] * N
    for t in tree.bottom_up():
        if not tree.is_leaf(t):
            _fold(H, t, tu, tv)
        if t == 0:
            break
        cr = H.U[t] @ wrow[t]
        cc = H.V[t] @ wcol[t]
        un = np.zeros((cr.shape[0], 0))
        vn = np.zeros((cc.shape[0], 0))
        if cr.shape[1] > 0 and cr.shape[0] > 0:
            su, ssu, _ = np.linalg.svd(cr, full_matrices=False)
            sv, ssv, _ = np.linalg.svd(cc, full_matrices=False)
            k = max(_trunc_rank(ssu, eps, floor), _trunc_rank(ssv, eps, floor))
            k = min(k, su.shape[1], sv.shape[1])
            un, vn = su[:, :k].copy(), sv[:, :k].copy()
        tu[t] = un.T @ H.U[t]
        tv[t] = vn.T @ H.V[t]
        H.U[t], H.V[t] = un, vn


def add_hbs(A, Bm, eps):  # hbs_ops.cpp:386-404
    if not trees_equal(A.tree, Bm.tree):
        raise ValueError("add_hbs: operands use different index trees")
    scl = 0.0
    for h in (A, Bm):
        for m in h.D + h.B:
            if m is not None and m.size:
                scl = max(scl, float(np.abs(m).max()))
    C = _stack_sum(A, Bm)
    _orthonormalize(C)
    _truncate(C, eps, 1e-13 * scl)
    return C


def lowrank_to_bs(Q, R, tree):  # hbs_ops.cpp:409-465
    N = tree.num_nodes()
    out = HO.Hbs(tree)
    if N == 1:
        out.D[0] = Q @ R
        return out
    sq, cf = [None] * N, [None] * N
    for t in tree.bottom_up():
        nd = tree.nodes[t]
        if tree.is_leaf(t):
            qt, rt = Q[nd.begin:nd.end], R[:, nd.begin:nd.end]
            out.D[t] = qt @ rt
            if t == 0:
                break
            out.U[t], sq[t] = _thin_qr(qt)
            vq, vr = _thin_qr(rt.T)
            out.V[t], cf[t] = vq, vr.T
            continue
        c1, c2 = nd.left, nd.right
        k1, k2 = sq[c1].shape[0], sq[c2].shape[0]
        b = np.zeros((k1 + k2, k1 + k2))
        b[:k1, k1:] = sq[c1] @ cf[c2]
        b[k1:, :k1] = sq[c2] @ cf[c1]
        out.B[t] = b
        if t == 0:
            break
        out.U[t], sq[t] = _thin_qr(np.vstack([sq[c1], sq[c2]]))
        vq, vr = _thin_qr(np.hstack([cf[c1], cf[c2]]).T)
        out.V[t], cf[t] = vq, vr.T
    return out


def add_lowrank(A, Q, R, eps):  # hbs_ops.cpp:467-470
    return add_hbs(A, lowrank_to_bs(Q, R, A.tree), eps)


# ------------------------------------------------------------------ split / consolidate (hbs_ops.cpp)
class Accumulation:
    def __init__(self, size=0):
        self.size = size
        self.piece_offsets = []
        self.pieces = []
        self.corrections = []


def _dense_single(D):
    h = HO.Hbs(single_node_tree(D.shape[0]))
    h.D[0] = D.copy()
    return h


def split_at(H, pos):  # hbs_ops.cpp:620-640 and helpers :476-605
    lo, hi = Accumulation(pos), Accumulation(H.tree.size() - pos)
    lo_hi, hi_lo = [], []

    def emit_piece(t):
        b = H.tree.nodes[t].begin
        if b >= pos:
            hi.piece_offsets.append(b - pos)
            hi.pieces.append(subtree_matrix(H, t))
        else:
            lo.piece_offsets.append(b)
            lo.pieces.append(subtree_matrix(H, t))

    def split_range(b, e):
        rs = []
        if b < pos:
            rs.append((b, min(e, pos) - b, b, False))
        if e > pos:
            s = max(b, pos)
            rs.append((s, e - s, s - pos, True))
        return rs

    def emit_coupling(row_node, col_node, bblock):
        k = bblock.shape[1]
        if k == 0 or H.rank(row_node) == 0:
            return
        L = apply_col_basis(H, row_node, bblock)
        Rm = apply_row_basis(H, col_node, np.eye(k)).T
        rb, re_ = H.tree.nodes[row_node].begin, H.tree.nodes[row_node].end
        cb, ce = H.tree.nodes[col_node].begin, H.tree.nodes[col_node].end
        for rbeg, rlen, roff, rhi in split_range(rb, re_):
            for cbeg, clen, coff, chi in split_range(cb, ce):
                placed = Placed(roff, coff, LowRank(L[rbeg - rb:rbeg - rb + rlen], Rm[:, cbeg - cb:cbeg - cb + clen]))
                if not rhi and not chi:
                    lo.corrections.append(placed)
                elif rhi and chi:
                    hi.corrections.append(placed)
                elif not rhi and chi:
                    lo_hi.append(placed)
                else:
                    hi_lo.append(placed)

    def split_node(t):
        nd = H.tree.nodes[t]
        if H.tree.is_leaf(t):
            p, sz = pos - nd.begin, nd.end - nd.begin
            lo.piece_offsets.append(nd.begin)
            lo.pieces.append(_dense_single(H.D[t][:p, :p]))
            hi.piece_offsets.append(0)
            hi.pieces.append(_dense_single(H.D[t][p:, p:]))
            lo_hi.append(Placed(nd.begin, 0, lowrank_from_dense(H.D[t][:p, p:], 1e-14)))
            hi_lo.append(Placed(0, nd.begin, lowrank_from_dense(H.D[t][p:, :p], 1e-14)))
            return
        c1, c2 = nd.left, nd.right
        mid = H.tree.nodes[c1].end
        k1, k2 = H.rank(c1), H.rank(c2)
        emit_coupling(c1, c2, H.B[t][:k1, k1:])
        emit_coupling(c2, c1, H.B[t][k1:, :k1])
        if pos == mid:
            emit_piece(c1)
            emit_piece(c2)
        elif pos < mid:
            split_node(c1)
            emit_piece(c2)
        else:
            emit_piece(c1)
            split_node(c2)

    if pos == 0:
        hi.piece_offsets.append(0)
        hi.pieces.append(H)
    elif pos == H.tree.size():
        lo.piece_offsets.append(0)
        lo.pieces.append(H)
    else:
        split_node(0)
    for acc in (lo, hi):
        order = sorted(range(len(acc.pieces)), key=lambda i: acc.piece_offsets[i])
        acc.piece_offsets = [acc.piece_offsets[i] for i in order]
        acc.pieces = [acc.pieces[i] for i in order]
    return lo, hi, lo_hi, hi_lo


def consolidate(acc, eps):  # hbs_ops.cpp:710-735 (+ graft_piece / build_spine :647-708)
    covered = 0
    for off, p in zip(acc.piece_offsets, acc.pieces):
        if off != covered:
            raise ValueError("consolidate: pieces do not tile the range")
        covered += p.tree.size()
    if covered != acc.size:
        raise ValueError("consolidate: pieces do not cover the range")
    if len(acc.pieces) == 1:
        joined = acc.pieces[0]
    else:
        nodes, D, U, V, B = [], [], [], [], []
        depth = [0]

        def graft(src, s, parent, level, offset):
            n = src.tree.nodes[s]
            i = len(nodes)
            nodes.append(HO.Node(n.begin + offset, n.end + offset, -1, -1, parent, level))
            depth[0] = max(depth[0], level)
            D.append(src.D[s])
            if s == 0:
                r = _node_rows(src, 0)
                U.append(np.zeros((r, 0)))
                V.append(np.zeros((r, 0)))
            else:
                U.append(src.U[s])
                V.append(src.V[s])
            B.append(src.B[s])
            if n.left >= 0:
                l_ = graft(src, n.left, i, level + 1, offset)
                r_ = graft(src, n.right, i, level + 1, offset)
                nodes[i].left, nodes[i].right = l_, r_
            return i

        def spine(lo_, hi_, parent, level):
            if hi_ - lo_ == 1:
                return graft(acc.pieces[lo_], 0, parent, level, acc.piece_offsets[lo_])
            begin = acc.piece_offsets[lo_]
            end = acc.piece_offsets[hi_ - 1] + acc.pieces[hi_ - 1].tree.size()
            target = begin + (end - begin + 1) // 2
            best = lo_ + 1
            for s in range(lo_ + 1, hi_):
                if abs(acc.piece_offsets[s] - target) < abs(acc.piece_offsets[best] - target):
                    best = s
            i = len(nodes)
            nodes.append(HO.Node(begin, end, -1, -1, parent, level))
            depth[0] = max(depth[0], level)
            D.append(None)
            U.append(np.zeros((0, 0)))
            V.append(np.zeros((0, 0)))
            B.append(np.zeros((0, 0)))
            l_ = spine(lo_, best, i, level + 1)
            r_ = spine(best, hi_, i, level + 1)
            nodes[i].left, nodes[i].right = l_, r_
            return i

        spine(0, len(acc.pieces), -1, 0)
        joined = HO.Hbs(HO.Tree(nodes, depth[0]))
        joined.D, joined.U, joined.V, joined.B = D, U, V, B
        # a spine node's B must be sized by its children's ranks (zero coupling)
        for t in range(len(nodes)):
            if nodes[t].left >= 0 and (B[t] is None or B[t].shape[0] != _node_rows(joined, t)):
                r = _node_rows(joined, t)
                if B[t] is None or B[t].size == 0:
                    joined.B[t] = np.zeros((r, r))
    if not acc.corrections:
        return joined
    corr = lowrank_sum(acc.size, acc.size, acc.corrections, eps)
    if corr.rank() == 0:
        return joined
    return add_lowrank(joined, corr.L, corr.R, eps)


def rebase(H, target, eps):  # hbs_ops.cpp:737-743
    if trees_equal(H.tree, target):
        return H
    return HO.compress(HO.reconstruct(H), eps, tree=target)


# ------------------------------------------------------------------ accelerated engine (accel_nd.cpp)
class Structured:
    """StructuredSchur (accel_nd.hpp:31-48)."""

    def __init__(self):
        self.x0 = self.x1 = self.y0 = self.y1 = 0
        self.j_side = NONE
        self.boundary = None  # [J; K] order
        self.j_size = 0
        self.s_jj = self.s_kk = None
        self.s_jk = self.s_kj = None

    def size(self):
        return len(self.boundary)

    def k_size(self):
        return self.size() - self.j_size

    def max_rank(self):
        k = max(self.s_kk.max_rank(), self.s_jj.max_rank() if self.s_jj is not None else 0)
        return max(k, self.s_jk.rank(), self.s_kj.rank())


class Dense:
    """SchurData (dense_nd.hpp:18-26): rect, CCW boundary ids, S."""

    def __init__(self, rect, boundary, S):
        self.x0, self.x1, self.y0, self.y1 = rect
        self.boundary, self.S = boundary, S


def _uid(n, x, y):
    return (y - 1) * (n - 2) + (x - 1)


def arc_boundary(n, x0, x1, y0, y1, j_side):  # accel_nd.cpp:46-88
    per = O.rect_perimeter_ccw(x0, x1, y0, y1)
    m = len(per)
    if j_side == NONE:
        return [_uid(n, x, y) for x, y in per], 0

    def in_j(p):
        x, y = p
        if j_side == NORTH:
            return y == y1 and x0 < x < x1
        if j_side == SOUTH:
            return y == y0 and x0 < x < x1
        if j_side == EAST:
            return x == x1 and y0 < y < y1
        return x == x0 and y0 < y < y1

    start, count = -1, 0
    for i in range(m):
        if in_j(per[i]):
            count += 1
            if not in_j(per[(i + m - 1) % m]):
                start = i
    if count == 0 or start < 0:
        raise ValueError("arc_boundary: box too small to carry a J edge")
    ids = [_uid(n, *per[(start + i) % m]) for i in range(m)]
    return ids, count


def compress_box(d: Dense, j_side, n, eps, leaf):  # accel_nd.cpp:93-130
    out = Structured()
    out.x0, out.x1, out.y0, out.y1 = d.x0, d.x1, d.y0, d.y1
    out.j_side = j_side
    out.boundary, out.j_size = arc_boundary(n, d.x0, d.x1, d.y0, d.y1, j_side)
    pos = {int(b): i for i, b in enumerate(d.boundary)}
    perm = np.array([pos[b] for b in out.boundary])
    s = d.S[np.ix_(perm, perm)]
    j = out.j_size
    k = len(perm) - j
    out.s_jj = HO.compress(s[:j, :j], eps, leaf)
    out.s_kk = HO.compress(s[j:, j:], eps, leaf)
    out.s_jk = lowrank_from_dense(s[:j, j:], eps)
    out.s_kj = lowrank_from_dense(s[j:, :j], eps)
    return out


def densify(s: Structured, n):  # accel_nd.cpp:132-167
    m, j = s.size(), s.j_size
    full = np.empty((m, m))
    full[:j, :j] = HO.reconstruct(s.s_jj) if j else np.zeros((0, 0))
    full[j:, j:] = HO.reconstruct(s.s_kk)
    full[:j, j:] = s.s_jk.dense()
    full[j:, :j] = s.s_kj.dense()
    pos = {int(b): i for i, b in enumerate(s.boundary)}
    ccw = [_uid(n, x, y) for x, y in O.rect_perimeter_ccw(s.x0, s.x1, s.y0, s.y1)]
    perm = np.array([pos[b] for b in ccw])
    return Dense((s.x0, s.x1, s.y0, s.y1), np.array(ccw, dtype=np.int64), full[np.ix_(perm, perm)])


def interface_coupling(prob, n, b3, b4):  # accel_nd.cpp:169-215
    if b3.j_size != b4.j_size:
        raise ValueError("interface_coupling: interface length mismatch")
    j = b3.j_size
    alpha, beta = np.empty(j), np.empty(j)
    for s_ in range(j):
        p4, q3 = b4.boundary[s_], b3.boundary[j - 1 - s_]
        alpha[s_] = prob.coeff(p4, q3)
        beta[j - 1 - s_] = prob.coeff(q3, p4)
    return alpha, beta


def _antidiag(w, x):  # accel_nd.cpp:24-26: diag(w) * reverse_rows(x)
    return w[:, None] * x[::-1]


def _split_child(s_kk, cuts):  # accel_nd.cpp:241-304
    pieces = [(0, s_kk)]
    corrections = []
    for cut in cuts:
        nxt = []
        for off, piece in pieces:
            if off + piece.tree.size() <= cut or off >= cut:
                nxt.append((off, piece))
                continue
            lo, hi, lo_hi, hi_lo = split_at(piece, cut - off)
            for po, p in zip(lo.piece_offsets, lo.pieces):
                nxt.append((off + po, p))
            for po, p in zip(hi.piece_offsets, hi.pieces):
                nxt.append((cut + po, p))
            for c in lo.corrections:
                corrections.append(Placed(off + c.row_offset, off + c.col_offset, c.lr))
            for c in hi.corrections:
                corrections.append(Placed(cut + c.row_offset, cut + c.col_offset, c.lr))
            for c in lo_hi:
                corrections.append(Placed(off + c.row_offset, cut + c.col_offset, c.lr))
            for c in hi_lo:
                corrections.append(Placed(cut + c.row_offset, off + c.col_offset, c.lr))
        pieces = nxt
        sliced = []
        for c in corrections:
            r0, r1 = c.row_offset, c.row_offset + c.lr.rows()
            c0, c1 = c.col_offset, c.col_offset + c.lr.cols()
            rparts = [(r0, cut), (cut, r1)] if r0 < cut < r1 else [(r0, r1)]
            cparts = [(c0, cut), (cut, c1)] if c0 < cut < c1 else [(c0, c1)]
            for rb, re_ in rparts:
                for cb, ce in cparts:
                    sliced.append(Placed(rb, cb, c.lr.block(rb - r0, re_ - rb, cb - c0, ce - cb)))
        corrections = sliced
    return pieces, corrections


class _Run:
    __slots__ = ("k_begin", "k_end", "in_j", "out_offset")

    def __init__(self, kb, ke, in_j, oo):
        self.k_begin, self.k_end, self.in_j, self.out_offset = kb, ke, in_j, oo


def _output_map(n, b3, b4, ux, out_side):  # accel_nd.cpp:322-398
    if out_side == NONE:
        boundary = list(b3.boundary[b3.j_size:]) + list(b4.boundary[b4.j_size:])
        out_j = 0
    else:
        boundary, out_j = arc_boundary(n, *ux, out_side)
    where = {}
    for c, b in enumerate((b3, b4)):
        for i in range(b.j_size, b.size()):
            where[b.boundary[i]] = (c, i - b.j_size)
    child_of, kpos_of = [], []
    for p in boundary:
        c, kp = where[p]
        child_of.append(c)
        kpos_of.append(kp)
    out_n = len(boundary)
    runs = [[], []]
    for p in range(out_n):
        c = child_of[p]
        in_j = p < out_j
        local = p if in_j else p - out_j
        r = runs[c]
        if (r and r[-1].in_j == in_j and r[-1].k_end == kpos_of[p]
                and local == r[-1].out_offset + (r[-1].k_end - r[-1].k_begin) and p > 0 and child_of[p - 1] == c):
            r[-1].k_end += 1
            continue
        r.append(_Run(kpos_of[p], kpos_of[p] + 1, in_j, local))
    cuts = [[], []]
    for c in range(2):
        srt = sorted(runs[c], key=lambda r: r.k_begin)
        for i in range(len(srt) - 1):
            if srt[i].k_end != srt[i + 1].k_begin:
                raise RuntimeError("accel_merge: child runs are not contiguous")
            cuts[c].append(srt[i].k_end)
    return boundary, out_j, child_of, kpos_of, runs, cuts


def _run_of(runs, c, begin, length):  # accel_nd.cpp:400-407
    for r in runs[c]:
        if begin >= r.k_begin and begin + length <= r.k_end:
            return r
    raise RuntimeError("accel_merge: item straddles a run boundary")


def accel_merge(b3, b4, prob, n, out_side, eps, leaf):  # accel_nd.cpp:434-628
    alpha, beta = interface_coupling(prob, n, b3, b4)
    inv33 = HO.invert_hbs(b3.s_jj)
    w = flip(inv33)
    scale_rows(w, alpha)
    scale_cols(w, beta[::-1].copy())
    scale(w, -1.0)
    w2 = rebase(w, b4.s_jj.tree, eps)
    inv_mid = HO.invert_hbs(add_hbs(b4.s_jj, w2, eps))
    y3 = HO.apply_inverse(inv33, b3.s_jk.L)
    x4a = -HO.apply_inverse(inv_mid, _antidiag(alpha, y3))
    x4b = HO.apply_inverse(inv_mid, b4.s_jk.L)
    x3a = y3 - HO.apply_inverse(inv33, _antidiag(beta, x4a))
    x3b = -HO.apply_inverse(inv33, _antidiag(beta, x4b))
    t_terms = [(0, 0, LowRank(b3.s_kj.L @ (b3.s_kj.R @ x3a), b3.s_jk.R)),
               (0, 1, LowRank(b3.s_kj.L @ (b3.s_kj.R @ x3b), b4.s_jk.R)),
               (1, 0, LowRank(b4.s_kj.L @ (b4.s_kj.R @ x4a), b3.s_jk.R)),
               (1, 1, LowRank(b4.s_kj.L @ (b4.s_kj.R @ x4b), b4.s_jk.R))]
    ux = (min(b3.x0, b4.x0), max(b3.x1, b4.x1), min(b3.y0, b4.y0), max(b3.y1, b4.y1))
    boundary, out_j, child_of, kpos_of, runs, cuts = _output_map(n, b3, b4, ux, out_side)
    out_n = len(boundary)
    jj, kk = Accumulation(out_j), Accumulation(out_n - out_j)
    jk, kj = [], []

    def place(row_child, row_begin, col_child, col_begin, lr):  # accel_nd.cpp:409-431
        rr = _run_of(runs, row_child, row_begin, lr.rows())
        cr = _run_of(runs, col_child, col_begin, lr.cols())
        term = Placed(rr.out_offset + (row_begin - rr.k_begin), cr.out_offset + (col_begin - cr.k_begin), lr)
        if rr.in_j and cr.in_j:
            jj.corrections.append(term)
        elif not rr.in_j and not cr.in_j:
            kk.corrections.append(term)
        elif rr.in_j:
            jk.append(term)
        else:
            kj.append(term)

    for c, b in enumerate((b3, b4)):  # Step 3a
        pieces, corrs = _split_child(b.s_kk, cuts[c])
        for off, piece in pieces:
            r = _run_of(runs, c, off, piece.tree.size())
            acc = jj if r.in_j else kk
            acc.piece_offsets.append(r.out_offset + (off - r.k_begin))
            acc.pieces.append(piece)
        for corr in corrs:
            if corr.lr.rank() == 0:
                continue
            place(c, corr.row_offset, c, corr.col_offset, corr.lr)
    out_pos = {p: i for i, p in enumerate(boundary)}  # Step 3b: junction couplings
    k3 = set(b3.boundary[b3.j_size:])
    for i in range(b4.j_size, b4.size()):
        q = b4.boundary[i]
        gx, gy = q % (n - 2) + 1, q // (n - 2) + 1
        for dx, dy in ((1, 0), (-1, 0), (0, 1), (0, -1)):
            x, y = gx + dx, gy + dy
            if not (1 <= x <= n - 2 and 1 <= y <= n - 2):
                continue
            p = _uid(n, x, y)
            if p not in k3:
                continue
            for rid, cid in ((p, q), (q, p)):
                v = prob.coeff(rid, cid)
                if v == 0.0:
                    continue
                rp, cp = out_pos[rid], out_pos[cid]
                place(child_of[rp], kpos_of[rp], child_of[cp], kpos_of[cp],
                      LowRank(np.array([[v]]), np.array([[1.0]])))
    for rc, cc, lr in t_terms:  # Step 3c
        if lr.rank() == 0:
            continue
        for rr in runs[rc]:
            for cr in runs[cc]:
                place(rc, rr.k_begin, cc, cr.k_begin,
                      LowRank(lr.L[rr.k_begin:rr.k_end], -lr.R[:, cr.k_begin:cr.k_end]))
    out = Structured()
    out.x0, out.x1, out.y0, out.y1 = ux
    out.j_side = out_side
    out.boundary = boundary
    out.j_size = out_j
    for acc in (jj, kk):
        order = sorted(range(len(acc.pieces)), key=lambda i: acc.piece_offsets[i])
        acc.piece_offsets = [acc.piece_offsets[i] for i in order]
        acc.pieces = [acc.pieces[i] for i in order]
    out.s_jj = consolidate(jj, eps) if out_j > 0 else None
    out.s_kk = consolidate(kk, eps)
    out.s_jk = lowrank_sum(out_j, out_n - out_j, jk, eps)
    out.s_kj = lowrank_sum(out_n - out_j, out_j, kj, eps)
    return out


class Result:
    def __init__(self):
        self.S_hbs = self.G_hbs = None
        self.S_dense = self.G_dense = None
        self.boundary = None
        self.rep_to_canonical = None
        self.cond = 0.0
        self.level_stats = []  # (level, max_rank, bytes, seconds)
        self.seconds = 0.0


def build_root_accel(prob, tree, eps=1e-7, crossover=1024, leaf=64):  # accel_nd.cpp:707-859
    """prob: oracle.Problem; tree: oracle.Tree (the reference's or the uniform partition)."""
    t_start = time.perf_counter()
    n = tree.n
    res = Result()

    def child_side(box):
        par = tree.boxes[box["parent"]]
        ci = par["children"].index(box["id"])
        return NORTH if ci < 2 else SOUTH  # accel_nd.cpp:661-665

    def rect(b):
        return (b["x0"], b["x1"], b["y0"], b["y1"])

    def merge_pair(a, b, out_side):  # accel_nd.cpp:667-689
        if isinstance(a, Structured) and isinstance(b, Structured):
            return accel_merge(a, b, prob, n, out_side, eps, leaf)
        da = densify(a, n) if isinstance(a, Structured) else a
        db = densify(b, n) if isinstance(b, Structured) else b
        r, S = O.merge_given(prob, (da.x0, da.x1, da.y0, da.y1), da.S, (db.x0, db.x1, db.y0, db.y1), db.S)
        ccw = np.array([_uid(n, x, y) for x, y in O.rect_perimeter_ccw(*r)], dtype=np.int64)
        merged = Dense(r, ccw, S)
        if out_side != NONE and len(ccw) >= crossover:
            return compress_box(merged, out_side, n, eps, leaf)
        return merged

    def stats_of(ops):
        mr, by = 0, 0
        for o in ops:
            if isinstance(o, Structured):
                mr = max(mr, o.max_rank())
                by += 8 * sum(m.size for h in (o.s_jj, o.s_kk) if h is not None
                              for lst in (h.D, h.U, h.V, h.B) for m in lst if m is not None)
                by += 8 * (o.s_jk.L.size + o.s_jk.R.size + o.s_kj.L.size + o.s_kj.R.size)
            else:
                by += 8 * o.S.size
        return mr, by

    current = {}
    t0 = time.perf_counter()
    for bid in tree.levels[tree.depth]:
        box = tree.boxes[bid]
        S = O.leaf_rect(prob, *rect(box))
        d = Dense(rect(box), np.asarray(box["boundary"], dtype=np.int64), S)
        side = NONE if tree.depth == 0 else child_side(box)
        current[bid] = compress_box(d, side, n, eps, leaf) if side != NONE and len(d.boundary) >= crossover else d
    mr, by = stats_of(current.values())
    res.level_stats.append((tree.depth, mr, by, time.perf_counter() - t0))
    for lev in range(tree.depth - 1, -1, -1):
        t0 = time.perf_counter()
        nxt = {}
        for bid in tree.levels[lev]:
            box = tree.boxes[bid]
            my_side = NONE if lev == 0 else child_side(box)
            ch = box["children"]
            west = merge_pair(current[ch[0]], current[ch[2]], EAST)
            east = merge_pair(current[ch[1]], current[ch[3]], WEST)
            nxt[bid] = merge_pair(west, east, my_side)
        current = nxt
        mr, by = stats_of(current.values())
        res.level_stats.append((lev, mr, by, time.perf_counter() - t0))
    root = current[0]
    res.boundary = np.asarray(tree.root()["boundary"], dtype=np.int64)
    if not isinstance(root, Structured):  # accel_nd.cpp:796-818
        res.S_dense = root.S
        res.G_dense = np.linalg.inv(root.S)
        res.cond = np.abs(res.S_dense).sum(0).max() * np.abs(res.G_dense).sum(0).max()
        res.rep_to_canonical = np.arange(len(res.boundary))
        res.seconds = time.perf_counter() - t_start
        return res
    t0 = time.perf_counter()
    res.S_hbs = root.s_kk
    res.G_hbs = HO.invert_hbs(res.S_hbs)
    canon = {int(b): i for i, b in enumerate(res.boundary)}
    res.rep_to_canonical = np.array([canon[int(b)] for b in root.boundary], dtype=np.int64)
    m = len(res.boundary)
    probe = np.ones(m)
    sx = HO.apply(res.S_hbs, probe)
    gx = HO.apply_inverse(res.G_hbs, probe)
    res.cond = (np.abs(sx).sum() / m) * (np.abs(gx).sum() / m) * m  # accel_nd.cpp:834-841
    res.level_stats.append((-1, res.S_hbs.max_rank(), 0, time.perf_counter() - t0))
    res.seconds = time.perf_counter() - t_start
    return res


def canonical_S(res) -> np.ndarray:
    """S of a build_root_accel result in the canonical ring order (dense)."""
    if res.S_hbs is None:
        return res.S_dense
    rep = HO.reconstruct(res.S_hbs)
    p = res.rep_to_canonical
    out = np.empty_like(rep)
    out[np.ix_(p, p)] = rep
    return out
