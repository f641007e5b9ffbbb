"""TEST INFRASTRUCTURE ONLY -- the CPU checker for the HBS (compressed) path.

A numpy restatement of the reference's HBS compression, apply and DTNHBS01
serialization (proj/src/hbs.cpp, proj/src/index_tree.cpp). Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline leg may import it; the
product path (paper_1302_5995_b200.hbs) never does.

Pinning: the reference's own HBS tests (proj/tests/test_hbs.cpp:51-200) are
formula-level properties (index-tree shapes, identity -> rank 0, rank-one ->
rank <= 1, Laplace root Schur complement at eps 1e-7 -> rel_fro <= 1e-6 with
max rank < M/4, apply vs dense <= 1e-8, round trip <= 10 eps (depth + 1),
orthonormal bases, monotone ranks, byte-stable serialization); tests/
test_hbs_oracle.py checks this restatement against each of them. The
reference's BDCSVD (Eigen, unpinned) is replaced by LAPACK's gesdd via
numpy: singular values/vectors agree to rounding, so ranks agree except at
exact ties with the cutoff.
"""
from __future__ import annotations

import struct

import numpy as np


class Node:
    __slots__ = ("begin", "end", "left", "right", "parent", "level")

    def __init__(self, begin, end, left=-1, right=-1, parent=-1, level=0):
        self.begin, self.end, self.left, self.right, self.parent, self.level = begin, end, left, right, parent, level


class Tree:
    def __init__(self, nodes, depth):
        self.nodes, self.depth = nodes, depth

    def size(self):
        return self.nodes[0].end

    def num_nodes(self):
        return len(self.nodes)

    def is_leaf(self, t):
        return self.nodes[t].left < 0

    def node_size(self, t):
        return self.nodes[t].end - self.nodes[t].begin

    def bottom_up(self):  # index_tree.cpp:8-12 (reverse preorder)
        return list(reversed(range(len(self.nodes))))


def build_index_tree(M: int, leaf_cap: int) -> Tree:
    """index_tree.cpp:37-67 (subdivide: mid = begin + (size + 1) / 2)."""
    nodes = []
    depth = [0]

    def sub(b, e, parent, level):
        i = len(nodes)
        nodes.append(Node(b, e, -1, -1, parent, level))
        depth[0] = max(depth[0], level)
        if e - b > leaf_cap:
            mid = b + (e - b + 1) // 2
            l_ = sub(b, mid, i, level + 1)
            r_ = sub(mid, e, i, level + 1)
            nodes[i].left, nodes[i].right = l_, r_
        return i

    sub(0, M, -1, 0)
    return Tree(nodes, depth[0])


def _svd_rank(sigma, eps):  # hbs.cpp:33-40
    if sigma.size == 0 or sigma[0] <= 0.0:
        return 0
    cut = eps * sigma[0]
    return int(np.count_nonzero(sigma > cut))


def _node_bases(row_block, col_block, eps):  # hbs.cpp:42-57
    if row_block.shape[1] == 0 or row_block.shape[0] == 0:
        return np.zeros((row_block.shape[0], 0)), np.zeros((col_block.shape[1], 0))
    su, ssu, _ = np.linalg.svd(row_block, full_matrices=False)
    sv, ssv, _ = np.linalg.svd(col_block.T, full_matrices=False)
    k = max(_svd_rank(ssu, eps), _svd_rank(ssv, eps))
    return su[:, :k].copy(), sv[:, :k].copy()


class Hbs:
    def __init__(self, tree):
        n = tree.num_nodes()
        self.tree = tree
        self.D = [None] * n
        self.U = [None] * n
        self.V = [None] * n
        self.B = [None] * n

    def rank(self, t):
        return 0 if t == 0 else self.U[t].shape[1]

    def max_rank(self):
        return max([self.rank(t) for t in range(1, self.tree.num_nodes())], default=0)

    def payload_bytes(self):
        return 8 * sum(m.size for lst in (self.D, self.U, self.V, self.B) for m in lst if m is not None)


def compress(H: np.ndarray, eps: float, leaf_cap: int = 64, tree: Tree | None = None) -> Hbs:
    """hbs.cpp:61-178 (frontier of compressed nodes and the reduced matrix R)."""
    H = np.asarray(H, dtype=np.float64)
    M = H.shape[0]
    tree = tree or build_index_tree(M, leaf_cap)
    out = Hbs(tree)
    if tree.num_nodes() == 1:
        out.D[0] = H.copy()
        return out
    members = []
    for t in range(tree.num_nodes()):
        if not tree.is_leaf(t):
            continue
        nd = tree.nodes[t]
        b, e = nd.begin, nd.end
        row_block = np.hstack([H[b:e, :b], H[b:e, e:]])
        col_block = np.vstack([H[:b, b:e], H[e:, b:e]])
        out.D[t] = H[b:e, b:e].copy()
        out.U[t], out.V[t] = _node_bases(row_block, col_block, eps)
        members.append(t)
    members.sort(key=lambda t: tree.nodes[t].begin)
    ranks = [out.U[t].shape[1] for t in members]
    offsets = list(np.cumsum([0] + ranks[:-1]))
    total = sum(ranks)
    R = np.zeros((total, total))
    for i, ti in enumerate(members):
        ni = tree.nodes[ti]
        row_red = out.U[ti].T @ H[ni.begin:ni.end, :]
        for j, tj in enumerate(members):
            nj = tree.nodes[tj]
            R[offsets[i]:offsets[i] + ranks[i], offsets[j]:offsets[j] + ranks[j]] = \
                row_red[:, nj.begin:nj.end] @ out.V[tj]
    for t in tree.bottom_up():
        if tree.is_leaf(t):
            continue
        c1, c2 = tree.nodes[t].left, tree.nodes[t].right
        p = members.index(c1)
        if p + 1 >= len(members) or members[p + 1] != c2:
            raise RuntimeError("compress: children not adjacent in frontier")
        o1, k1, o2, k2 = offsets[p], ranks[p], offsets[p + 1], ranks[p + 1]
        rest = total - k1 - k2
        Bt = np.zeros((k1 + k2, k1 + k2))
        Bt[:k1, k1:] = R[o1:o1 + k1, o2:o2 + k2]
        Bt[k1:, :k1] = R[o2:o2 + k2, o1:o1 + k1]
        out.B[t] = Bt
        if t == 0:
            break
        keep = np.r_[0:o1, o2 + k2:total]
        pair = np.r_[o1:o2 + k2]
        row_block = R[np.ix_(pair, keep)]
        col_block = R[np.ix_(keep, pair)]
        Ut, Vt = _node_bases(row_block, col_block, eps)
        out.U[t], out.V[t] = Ut, Vt
        kt = Ut.shape[1]
        Rn = np.zeros((rest + kt, rest + kt))
        newpos = np.r_[0:o1, o1 + kt:rest + kt]
        Rn[np.ix_(newpos, newpos)] = R[np.ix_(keep, keep)]
        Rn[o1:o1 + kt, newpos] = Ut.T @ row_block
        Rn[newpos, o1:o1 + kt] = col_block @ Vt
        R = Rn
        members[p:p + 2] = [t]
        ranks[p:p + 2] = [kt]
        total = rest + kt
        offsets = list(np.cumsum([0] + ranks[:-1]))
    return out


def apply(h: Hbs, x: np.ndarray) -> np.ndarray:
    """hbs.cpp:187-232."""
    tree = h.tree
    x = np.asarray(x, dtype=np.float64)
    vec = x.ndim == 1
    X = x.reshape(tree.size(), -1)
    if tree.num_nodes() == 1:
        y = h.D[0] @ X
        return y[:, 0] if vec else y
    xhat = [None] * tree.num_nodes()
    yhat = [None] * tree.num_nodes()
    for t in tree.bottom_up():
        if t == 0:
            continue
        if tree.is_leaf(t):
            nd = tree.nodes[t]
            xhat[t] = h.V[t].T @ X[nd.begin:nd.end]
        else:
            c1, c2 = tree.nodes[t].left, tree.nodes[t].right
            xhat[t] = h.V[t].T @ np.vstack([xhat[c1], xhat[c2]])
    Y = np.zeros_like(X)
    for t in range(tree.num_nodes()):
        nd = tree.nodes[t]
        if tree.is_leaf(t):
            Y[nd.begin:nd.end] = h.D[t] @ X[nd.begin:nd.end]
            if t != 0 and yhat[t] is not None and yhat[t].size:
                Y[nd.begin:nd.end] += h.U[t] @ yhat[t]
            continue
        c1, c2 = nd.left, nd.right
        k1 = h.rank(c1)
        given = h.B[t] @ np.vstack([xhat[c1], xhat[c2]])
        if t != 0 and yhat[t] is not None and yhat[t].size:
            given = given + h.U[t] @ yhat[t]
        yhat[c1], yhat[c2] = given[:k1], given[k1:]
    return Y[:, 0] if vec else Y


def reconstruct(h: Hbs) -> np.ndarray:
    return apply(h, np.eye(h.tree.size()))


def orthonormality_defect(h: Hbs) -> float:
    d = 0.0
    for t in range(1, h.tree.num_nodes()):
        for b in (h.U[t], h.V[t]):
            if b.shape[1]:
                d = max(d, float(np.abs(b.T @ b - np.eye(b.shape[1])).max()))
    return d


def serialize(h: Hbs) -> bytes:
    """hbs.cpp:446-470: magic, M, num_nodes, depth, 6 int64 per node, then per
    node D (leaves), U and V (non-root), B (parents), each as rows, cols and
    column-major doubles; all integers little-endian int64."""
    tree = h.tree
    out = bytearray(b"DTNHBS01")
    out += struct.pack("<qqq", tree.size(), tree.num_nodes(), tree.depth)
    for n in tree.nodes:
        out += struct.pack("<qqqqqq", n.begin, n.end, n.left, n.right, n.parent, n.level)

    def mat(m):
        nonlocal out
        out += struct.pack("<qq", m.shape[0], m.shape[1])
        out += np.asfortranarray(m, dtype="<f8").tobytes(order="F")

    for t in range(tree.num_nodes()):
        if tree.is_leaf(t):
            mat(h.D[t])
        if t != 0:
            mat(h.U[t])
            mat(h.V[t])
        if not tree.is_leaf(t):
            mat(h.B[t])
    return bytes(out)


def deserialize(data: bytes) -> Hbs:
    if len(data) < 8 or data[:8] != b"DTNHBS01":
        raise ValueError("deserialize: bad magic")
    p = 8

    def i64():
        nonlocal p
        if len(data) - p < 8:
            raise ValueError("deserialize: truncated input")
        v = struct.unpack_from("<q", data, p)[0]
        p += 8
        return v

    M, nn, depth = i64(), i64(), i64()
    nodes = [Node(*(i64() for _ in range(6))) for _ in range(nn)]
    tree = Tree(nodes, depth)
    if tree.size() != M:
        raise ValueError("deserialize: bad header")
    h = Hbs(tree)

    def mat():
        nonlocal p
        r, c = i64(), i64()
        nbytes = r * c * 8
        if len(data) - p < nbytes:
            raise ValueError("deserialize: truncated input")
        m = np.frombuffer(data, dtype="<f8", count=r * c, offset=p).reshape((r, c), order="F").copy()
        p += nbytes
        return m

    for t in range(nn):
        if tree.is_leaf(t):
            h.D[t] = mat()
        if t != 0:
            h.U[t] = mat()
            h.V[t] = mat()
        if not tree.is_leaf(t):
            h.B[t] = mat()
    return h


def kernel_matrix(m: int, seed: int) -> np.ndarray:
    """The reference test's model matrix (test_hbs.cpp:31-41): 1 / (1 + |i - j|)
    + 5 I + 0.01 N(0,1) / m. The Gaussian draws come from numpy's generator
    (std::normal_distribution is implementation-defined), so the values differ
    from the reference run but the structure and the tolerances are the same."""
    i = np.arange(m)
    h = 1.0 / (1.0 + np.abs(i[:, None] - i[None, :]).astype(np.float64))
    h += 5.0 * np.eye(m)
    h += 0.01 * np.random.default_rng(seed).standard_normal((m, m)) / m
    return h


# ---------------------------------------------------------------------------
# Multi-level inversion (hbs_ops.cpp:148-201) and the inverse's apply
# (hbs_ops.cpp:203-205): the factors {E, F, G} and the root core inverse are
# stored in an Hbs of the same tree -- E in U, F in V, G in D (leaves) / B
# (parents), the core inverse in the root B -- so apply() is the inverse's
# apply. Eigen's FullPivLU inverse is replaced by LAPACK's partial-pivoting
# inverse (numpy.linalg.inv); the results agree to rounding on the
# well-conditioned blocks these tests use.

class FactorizationError(RuntimeError):
    """errors.hpp:11-21: what + " [" + where + "]"."""

    def __init__(self, what, where):
        super().__init__(f"{what} [{where}]")
        self.where = where


def _checked_inverse(A, what, where):  # hbs_ops.cpp:27-37
    if A.size == 0:
        return A.copy()
    try:
        inv = np.linalg.inv(A)
    except np.linalg.LinAlgError:
        raise FactorizationError(f"{what} is singular", where) from None
    if not np.all(np.isfinite(inv)):
        raise FactorizationError(f"{what} is singular", where)
    return inv


def invert_hbs(h: Hbs) -> Hbs:
    tree = h.tree
    rep = Hbs(tree)
    if tree.num_nodes() == 1:
        rep.D[0] = _checked_inverse(h.D[0], "D", "root leaf")
        return rep
    dhat = [None] * tree.num_nodes()
    for t in tree.bottom_up():
        where = f"node {t} level {tree.nodes[t].level}"
        if tree.is_leaf(t):
            dtilde = h.D[t].copy()
        else:
            c1, c2 = tree.nodes[t].left, tree.nodes[t].right
            k1, k2 = h.rank(c1), h.rank(c2)
            dtilde = h.B[t].copy()
            dtilde[:k1, :k1] += dhat[c1]
            dtilde[k1:, k1:] += dhat[c2]
        if t == 0:
            rep.B[0] = _checked_inverse(dtilde, "root coupling block", where)
            break
        dinv = _checked_inverse(dtilde, "Dtilde", where)
        w = dinv @ h.U[t]
        dhat[t] = _checked_inverse(h.V[t].T @ w, "reduced block (V^T Dtilde^{-1} U)", where)
        e = w @ dhat[t]
        rep.U[t] = e
        rep.V[t] = dinv.T @ h.V[t] @ dhat[t].T
        g = dinv - e @ (h.V[t].T @ dinv)
        if tree.is_leaf(t):
            rep.D[t] = g
        else:
            rep.B[t] = g
    return rep


def apply_inverse(inv: Hbs, x: np.ndarray) -> np.ndarray:
    return apply(inv, x)


def synthetic_hbs(m_total: int, leaf: int, k: int, seed: int) -> Hbs:
    """test_hbs_ops.cpp:70-105: a well-conditioned HBS matrix with exact rank
    k everywhere (leaf D = N(0,1) + 20 k I, orthonormal U/V, zero-diagonal B).
    Gaussian draws from numpy (std::normal_distribution is
    implementation-defined): same structure and tolerances, other values."""
    rng = np.random.default_rng(seed)
    tree = build_index_tree(m_total, leaf)
    h = Hbs(tree)

    def orth(r, c):
        q, _ = np.linalg.qr(rng.standard_normal((r, c)))
        return q[:, :c]

    for t in tree.bottom_up():
        if tree.is_leaf(t):
            sz = tree.node_size(t)
            h.D[t] = rng.standard_normal((sz, sz)) + 20.0 * k * np.eye(sz)
            if t != 0:
                h.U[t], h.V[t] = orth(sz, min(k, sz)), orth(sz, min(k, sz))
            continue
        k1, k2 = h.U[tree.nodes[t].left].shape[1], h.U[tree.nodes[t].right].shape[1]
        b = np.zeros((k1 + k2, k1 + k2))
        b[:k1, k1:] = rng.standard_normal((k1, k2))
        b[k1:, :k1] = rng.standard_normal((k2, k1))
        h.B[t] = b
        if t != 0:
            h.U[t], h.V[t] = orth(k1 + k2, min(k, k1 + k2)), orth(k1 + k2, min(k, k1 + k2))
    return h
