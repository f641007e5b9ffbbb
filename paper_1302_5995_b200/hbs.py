"""Compressed (HBS) operators on the B200: the reference's HbsMatrix
(proj/include/dtn/hbs.hpp:30-51) with compress / apply / serialize
(proj/src/hbs.cpp:61-232, 422-519) running on the device through the C ABI
(include/dtn_gpu.h, dtn_gpu_hbs_*; kernels in csrc/k_hbs.cu, csrc/hbs.cu).

The factors stay in HBM; `factor()` / `D`, `U`, `V`, `B` fetch host copies.
There is no CPU fallback: every compute call goes through libdtn_b200.so.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .dtn import Context, default_context

__all__ = ["IndexTree", "build_index_tree", "HbsMatrix", "InverseFactors", "compress", "compress_operator", "apply",
           "invert_hbs", "apply_inverse", "reconstruct",
           "serialize", "deserialize", "write_hbs", "read_hbs", "basis_orthonormality_defect",
           "mirror", "subtree_matrix", "flip", "scale", "scale_rows", "scale_cols", "add_hbs", "lowrank_to_bs",
           "add_lowrank", "rebase", "SplitParts", "split_at", "consolidate", "LowRank", "Placed",
           "lowrank_from_dense", "lowrank_recompress", "lowrank_sum"]


@dataclass
class IndexNode:
    begin: int
    end: int
    left: int = -1
    right: int = -1
    parent: int = -1
    level: int = 0


class IndexTree:
    """index_tree.hpp:12-38: contiguous ranges, preorder ids."""

    def __init__(self, nodes, depth):
        self.nodes = list(nodes)
        self.depth = int(depth)

    def size(self):
        return self.nodes[0].end if self.nodes else 0

    def num_nodes(self):
        return len(self.nodes)

    def is_leaf(self, t):
        return self.nodes[t].left < 0

    def node_size(self, t):
        return self.nodes[t].end - self.nodes[t].begin

    def top_down(self):
        return list(range(len(self.nodes)))

    def bottom_up(self):
        return list(reversed(range(len(self.nodes))))

    def __eq__(self, other):
        if not isinstance(other, IndexTree) or len(self.nodes) != len(other.nodes):
            return False
        return all((a.begin, a.end, a.left, a.right) == (b.begin, b.end, b.left, b.right)
                   for a, b in zip(self.nodes, other.nodes))


def build_index_tree(M: int, leaf_cap: int) -> IndexTree:
    """build_index_tree (index_tree.cpp:37-67): balanced halving, the left half
    taking the extra index. Host bookkeeping (the device builds the same tree
    in hbs_index_tree, csrc/hbs.cu)."""
    if M < 1:
        raise ValueError("build_index_tree: M must be >= 1")
    if leaf_cap < 2:
        raise ValueError("build_index_tree: leaf_cap must be >= 2")
    nodes: list[IndexNode] = []
    depth = 0

    def sub(b, e, parent, level):
        nonlocal depth
        i = len(nodes)
        nodes.append(IndexNode(b, e, -1, -1, parent, level))
        depth = max(depth, level)
        if e - b > leaf_cap:
            mid = b + (e - b + 1) // 2
            l_ = sub(b, mid, i, level + 1)
            r_ = sub(mid, e, i, level + 1)
            nodes[i].left, nodes[i].right = l_, r_
        return i

    sub(0, M, -1, 0)
    return IndexTree(nodes, depth)


class HbsMatrix:
    """Device-resident HbsMatrix (hbs.hpp:30-51)."""

    def __init__(self, ctx: Context, handle: C.c_void_p):
        self.ctx, self.h = ctx, handle
        M, nn, mr, pb = C.c_int64(), C.c_int64(), C.c_int64(), C.c_uint64()
        dp = C.c_int32()
        ctx.check(L.lib().dtn_gpu_hbs_info(handle, C.byref(M), C.byref(nn), C.byref(dp), C.byref(mr), C.byref(pb)))
        self._M, self._max_rank, self._payload = M.value, mr.value, pb.value
        raw = np.zeros((nn.value, 6), dtype=np.int64)
        ranks = np.zeros(nn.value, dtype=np.int64)
        ctx.check(L.lib().dtn_gpu_hbs_tree(handle, raw.ctypes.data, ranks.ctypes.data))
        self.tree = IndexTree([IndexNode(*map(int, r)) for r in raw], dp.value)
        self.ranks = ranks
        self._cache: dict = {}

    def __del__(self):
        try:
            if getattr(self, "h", None):
                L.lib().dtn_gpu_hbs_free(self.h)
                self.h = None
        except Exception:
            pass

    # hbs.hpp:37-50
    def size(self) -> int:
        return self._M

    def rank(self, t: int) -> int:
        return 0 if t == 0 else int(self.ranks[t])

    def node_rows(self, t: int) -> int:
        if self.tree.is_leaf(t):
            return self.tree.node_size(t)
        n = self.tree.nodes[t]
        return self.rank(n.left) + self.rank(n.right)

    def max_rank(self) -> int:
        return self._max_rank

    def payload_bytes(self) -> int:
        return self._payload

    def factor(self, t: int, which: str) -> np.ndarray:
        key = (t, which)
        if key not in self._cache:
            w = {"D": 0, "U": 1, "V": 2, "B": 3}[which]
            r, c = C.c_int64(), C.c_int64()
            self.ctx.check(L.lib().dtn_gpu_hbs_factor(self.h, t, w, None, C.byref(r), C.byref(c)))
            out = np.zeros((r.value, c.value), dtype=np.float64, order="F")
            self.ctx.check(L.lib().dtn_gpu_hbs_factor(self.h, t, w, out.ctypes.data, C.byref(r), C.byref(c)))
            self._cache[key] = out
        return self._cache[key]

    def _all(self, which, pred):
        return [self.factor(t, which) if pred(t) else None for t in range(self.tree.num_nodes())]

    @property
    def D(self):
        return self._all("D", self.tree.is_leaf)

    @property
    def U(self):
        return self._all("U", lambda t: t != 0)

    @property
    def V(self):
        return self._all("V", lambda t: t != 0)

    @property
    def B(self):
        return self._all("B", lambda t: not self.tree.is_leaf(t))

    def apply(self, x):
        return apply(self, x)

    def serialize(self) -> memoryview:
        return serialize(self)


class InverseFactors(HbsMatrix):
    """InverseFactors (hbs_ops.hpp:46-55): the telescoping inverse factors of an
    HbsMatrix on its tree, E in the U slots, F in the V slots, G in the D
    (leaves) / B (parents) slots and the root core inverse in the root B, so the
    HBS apply sweep is apply_inverse. `rep` is the object itself."""

    @property
    def rep(self) -> "InverseFactors":
        return self

    def E(self, t: int) -> np.ndarray:
        return self.factor(t, "U")

    def F(self, t: int) -> np.ndarray:
        return self.factor(t, "V")

    def G(self, t: int) -> np.ndarray:
        return self.factor(t, "D" if self.tree.is_leaf(t) else "B")


def invert_hbs(H: HbsMatrix) -> InverseFactors:
    """invert_hbs (hbs_ops.hpp:64, hbs_ops.cpp:148-201) on the device. Raises
    FactorizationError naming the node ("... is singular [node t level l]")."""
    out = C.c_void_p()
    H.ctx.check(L.lib().dtn_gpu_hbs_invert(H.h, C.byref(out)))
    return InverseFactors(H.ctx, out)


def apply_inverse(inv: InverseFactors, x):
    """apply_inverse (hbs_ops.cpp:203-205): y = H^{-1} x through the inverse factors."""
    return apply(inv, x)


def _ctx(ctx):
    return ctx if ctx is not None else default_context()


def compress(H, eps: float, leaf_cap: int = 64, ctx: Context | None = None,
             tree: IndexTree | None = None) -> HbsMatrix:
    """compress(H, eps, leaf_cap) (hbs.hpp:58-62): H is a host array or a
    float64 CUDA tensor (column-major or row-major contiguous). With `tree`:
    compress(H, tree, eps) onto that index tree (hbs.hpp:58-60)."""
    ctx = _ctx(ctx)
    out = C.c_void_p()
    if tree is not None:
        A = np.asfortranarray(np.asarray(H, dtype=np.float64))
        if A.ndim != 2 or A.shape[0] != A.shape[1] or A.shape[0] != tree.size():
            raise ValueError("compress: matrix/tree size mismatch")
        t = _tree_array(tree)
        ctx.check(L.lib().dtn_gpu_hbs_compress_tree(ctx.h, A.ctypes.data, A.shape[0], A.shape[0], 0, float(eps),
                                                    t.ctypes.data, t.shape[0], C.byref(out)))
        return HbsMatrix(ctx, out)
    try:
        import torch
        is_t = isinstance(H, torch.Tensor)
    except ImportError:  # pragma: no cover
        is_t = False
    if is_t:
        if H.dtype != torch.float64 or not H.is_cuda or H.dim() != 2 or H.shape[0] != H.shape[1]:
            raise ValueError("compress: H must be a square float64 CUDA tensor")
        Hc = H.t().contiguous().t() if H.stride(0) != 1 else H  # column-major
        with ctx.torch_stream():
            ctx.check(L.lib().dtn_gpu_hbs_compress(ctx.h, Hc.data_ptr(), H.shape[0],
                                                   Hc.stride(1) if H.shape[0] > 1 else 1, 1, float(eps),
                                                   int(leaf_cap), C.byref(out)))
    else:
        A = np.asfortranarray(np.asarray(H, dtype=np.float64))
        if A.ndim != 2 or A.shape[0] != A.shape[1]:
            raise ValueError("compress: matrix/tree size mismatch")
        ctx.check(L.lib().dtn_gpu_hbs_compress(ctx.h, A.ctypes.data, A.shape[0], A.shape[0], 0, float(eps),
                                               int(leaf_cap), C.byref(out)))
    return HbsMatrix(ctx, out)


def compress_operator(sol, which: str = "G", eps: float = 1e-10, leaf_cap: int = 64) -> HbsMatrix:
    """Compress a built operator's resident G (apply_dtn) or S (apply_schur)
    in place in HBM: SolutionOperator::G_hbs / S_hbs (solution_operator.hpp:38-42)."""
    out = C.c_void_p()
    sol.ctx.check(L.lib().dtn_gpu_hbs_compress_op(sol.h, 0 if which == "G" else 1, float(eps), int(leaf_cap),
                                                  C.byref(out)))
    return HbsMatrix(sol.ctx, out)


def apply(H: HbsMatrix, x):
    """apply(H, x) (hbs.hpp:66, hbs.cpp:187-232): x is (M,) / (M, k) host, or a
    float64 CUDA tensor (result stays on the device)."""
    M = H.size()
    try:
        import torch
        is_t = isinstance(x, torch.Tensor)
    except ImportError:  # pragma: no cover
        is_t = False
    if is_t:
        if x.dtype != torch.float64 or not x.is_cuda:
            raise ValueError("apply: torch input must be a float64 CUDA tensor")
        vec = x.dim() == 1
        X = x.reshape(M, -1) if vec else x
        if X.shape[0] != M:
            raise ValueError("apply: dimension mismatch")
        colmajor = X.stride(0) == 1 and (X.shape[1] <= 1 or X.stride(1) >= M)
        Xf = X if colmajor else X.t().contiguous().t()  # column-major with ld >= M
        Y = torch.empty((X.shape[1], M), dtype=torch.float64, device=x.device).t()
        ldx = Xf.stride(1) if Xf.shape[1] > 1 else M
        with H.ctx.torch_stream():
            H.ctx.check(L.lib().dtn_gpu_hbs_apply(H.h, Xf.data_ptr(), ldx, Xf.shape[1], Y.data_ptr(), M, 1))
        return Y.reshape(M) if vec else Y
    X = np.asarray(x, dtype=np.float64)
    vec = X.ndim == 1
    if X.shape[0] != M:
        raise ValueError("apply: dimension mismatch")
    X2 = np.asfortranarray(X.reshape(M, -1))
    Y = np.zeros_like(X2, order="F")
    if X2.shape[1]:
        H.ctx.check(L.lib().dtn_gpu_hbs_apply(H.h, X2.ctypes.data, M, X2.shape[1], Y.ctypes.data, M, 0))
    return Y[:, 0].copy() if vec else Y


def reconstruct(H: HbsMatrix) -> np.ndarray:
    """Exact dense evaluation of the stored factorization (hbs.hpp:69, a testing
    aid): the telescoping apply of the identity, on the device."""
    M = H.size()
    out = np.zeros((M, M), dtype=np.float64, order="F")
    H.ctx.check(L.lib().dtn_gpu_hbs_reconstruct(H.h, out.ctypes.data, M, 0))
    return out


def basis_orthonormality_defect(H: HbsMatrix) -> float:
    """hbs.cpp:405-417: max_t ||U^T U - I||_max over U and V (a host check on the fetched bases)."""
    d = 0.0
    for t in range(1, H.tree.num_nodes()):
        for w in ("U", "V"):
            b = H.factor(t, w)
            if b.shape[1] == 0:
                continue
            d = max(d, float(np.abs(b.T @ b - np.eye(b.shape[1])).max()))
    return d


def serialize(H: HbsMatrix) -> memoryview:
    """DTNHBS01 (hbs.cpp:446-470), as a read-only bytes-like view (compares equal to the
    same bytes; `bytes(...)` copies it). The buffer is written in place by ONE device-to-host
    copy into fresh, unzeroed memory (a bytearray would first zero-fill every page)."""
    n = C.c_uint64()
    H.ctx.check(L.lib().dtn_gpu_hbs_serialize(H.h, None, 0, C.byref(n)))
    out = np.empty(n.value, dtype=np.uint8)
    if n.value:
        H.ctx.check(L.lib().dtn_gpu_hbs_serialize(H.h, out.ctypes.data, n.value,
                                                  C.byref(n)))
    return memoryview(out).toreadonly()


def deserialize(data: bytes, ctx: Context | None = None) -> HbsMatrix:
    """hbs.cpp:472-505: the factors are uploaded to the device."""
    ctx = _ctx(ctx)
    out = C.c_void_p()
    b = (C.c_uint8 * len(data)).from_buffer_copy(data) if len(data) else (C.c_uint8 * 1)()
    ctx.check(L.lib().dtn_gpu_hbs_deserialize(ctx.h, b, len(data), C.byref(out)))
    return HbsMatrix(ctx, out)


def write_hbs(H: HbsMatrix, path: str) -> None:
    with open(path, "wb") as f:
        f.write(serialize(H))


def read_hbs(path: str, ctx: Context | None = None) -> HbsMatrix:
    with open(path, "rb") as f:
        return deserialize(f.read(), ctx)


# ---------------------------------------------------------------------------- HBS algebra
# hbs.cpp:290-402 (subtree / flip / scale), hbs_ops.cpp:213-743 (add_hbs, lowrank_to_bs,
# add_lowrank, split_at, consolidate, rebase), lowrank.cpp; device work in csrc/hbs_ops.cu.

def _tree_array(tree: IndexTree) -> np.ndarray:
    return np.ascontiguousarray([[n.begin, n.end, n.left, n.right, n.parent, n.level] for n in tree.nodes],
                                dtype=np.int64).reshape(-1, 6)


def _host(a, rows, cols):
    A = np.asfortranarray(np.asarray(a, dtype=np.float64).reshape(rows, cols))
    return A, max(rows, 1)


def mirror(tree: IndexTree) -> IndexTree:
    """mirror (index_tree.cpp:71-93): the tree of the reversed index order."""
    M = tree.size()
    nodes: list[IndexNode] = []
    depth = 0

    def rec(t, parent, level):
        nonlocal depth
        n = tree.nodes[t]
        i = len(nodes)
        nodes.append(IndexNode(M - n.end, M - n.begin, -1, -1, parent, level))
        depth = max(depth, level)
        if n.left >= 0:
            lft = rec(n.right, i, level + 1)
            rgt = rec(n.left, i, level + 1)
            nodes[i].left, nodes[i].right = lft, rgt
        return i

    rec(0, -1, 0)
    return IndexTree(nodes, depth)


def subtree_matrix(H: HbsMatrix, t: int) -> HbsMatrix:
    """subtree_matrix (hbs.cpp:290-320): the diagonal block of node t as its own HBS matrix."""
    out = C.c_void_p()
    H.ctx.check(L.lib().dtn_gpu_hbs_subtree(H.h, int(t), C.byref(out)))
    return HbsMatrix(H.ctx, out)


def flip(H: HbsMatrix) -> HbsMatrix:
    """flip (hbs.cpp:322-375): P H P with P the index reversal, on the mirrored tree."""
    out = C.c_void_p()
    H.ctx.check(L.lib().dtn_gpu_hbs_flip(H.h, C.byref(out)))
    return HbsMatrix(H.ctx, out)


def scale(H: HbsMatrix, s: float) -> None:
    """scale (hbs.cpp:399-402): H *= s, in place."""
    H.ctx.check(L.lib().dtn_gpu_hbs_scale(H.h, float(s)))
    H._cache.clear()


def scale_rows(H: HbsMatrix, w) -> None:
    """scale_rows (hbs.cpp:377-386): diag(w) H, in place."""
    W = np.ascontiguousarray(w, dtype=np.float64).reshape(-1)
    if W.shape[0] != H.size():
        raise ValueError("scale_rows: size mismatch")
    H.ctx.check(L.lib().dtn_gpu_hbs_scale_rows(H.h, W.ctypes.data, 0))
    H._cache.clear()


def scale_cols(H: HbsMatrix, w) -> None:
    """scale_cols (hbs.cpp:388-397): H diag(w), in place."""
    W = np.ascontiguousarray(w, dtype=np.float64).reshape(-1)
    if W.shape[0] != H.size():
        raise ValueError("scale_cols: size mismatch")
    H.ctx.check(L.lib().dtn_gpu_hbs_scale_cols(H.h, W.ctypes.data, 0))
    H._cache.clear()


def add_hbs(A: HbsMatrix, B: HbsMatrix, eps: float) -> HbsMatrix:
    """add_hbs (hbs_ops.cpp:386-404): A + B on their common tree, recompressed at eps.
    Different trees raise ValueError ("add_hbs: operands use different index trees")."""
    out = C.c_void_p()
    A.ctx.check(L.lib().dtn_gpu_hbs_add(A.h, B.h, float(eps), C.byref(out)))
    return HbsMatrix(A.ctx, out)


def lowrank_to_bs(Q, R, tree: IndexTree, ctx: Context | None = None) -> HbsMatrix:
    """lowrank_to_bs (hbs_ops.cpp:409-465): Q R (M x k times k x M) as an HBS matrix on `tree`."""
    ctx = _ctx(ctx)
    M = tree.size()
    k = np.asarray(Q).shape[1] if np.asarray(Q).ndim == 2 else 0
    Qh, ldq = _host(Q, M, k)
    Rh, ldr = _host(R, k, M)
    t = _tree_array(tree)
    out = C.c_void_p()
    ctx.check(L.lib().dtn_gpu_hbs_from_lowrank(ctx.h, Qh.ctypes.data, ldq, Rh.ctypes.data, max(k, 1), k,
                                               t.ctypes.data, t.shape[0], 0, C.byref(out)))
    return HbsMatrix(ctx, out)


def add_lowrank(A: HbsMatrix, Q, R, eps: float) -> HbsMatrix:
    """add_lowrank (hbs_ops.cpp:467-470): A + Q R recompressed at eps on A's tree."""
    M = A.size()
    k = np.asarray(Q).shape[1] if np.asarray(Q).ndim == 2 else 0
    Qh, ldq = _host(Q, M, k)
    Rh, _ = _host(R, k, M)
    out = C.c_void_p()
    A.ctx.check(L.lib().dtn_gpu_hbs_add_lowrank(A.h, Qh.ctypes.data, ldq, Rh.ctypes.data, max(k, 1), k, float(eps), 0,
                                                C.byref(out)))
    return HbsMatrix(A.ctx, out)


def rebase(H: HbsMatrix, target: IndexTree, eps: float) -> HbsMatrix:
    """rebase (hbs_ops.cpp:737-743): H re-expressed on the target tree."""
    t = _tree_array(target)
    out = C.c_void_p()
    H.ctx.check(L.lib().dtn_gpu_hbs_rebase(H.h, t.ctypes.data, t.shape[0], float(eps), C.byref(out)))
    return HbsMatrix(H.ctx, out)


class LowRank:
    """LowRank (lowrank.hpp): L (m x k) R (k x n) held on the device."""

    def __init__(self, ctx: Context, handle: C.c_void_p):
        self.ctx, self.h = ctx, handle
        m, n, k = C.c_int64(), C.c_int64(), C.c_int64()
        ctx.check(L.lib().dtn_gpu_lowrank_info(handle, C.byref(m), C.byref(n), C.byref(k)))
        self._m, self._n, self._k = m.value, n.value, k.value
        self._lr = None

    @staticmethod
    def from_factors(Lf, R, ctx: Context | None = None) -> "LowRank":
        ctx = _ctx(ctx)
        Lh = np.asfortranarray(np.asarray(Lf, dtype=np.float64))
        Rh = np.asfortranarray(np.asarray(R, dtype=np.float64))
        m, k = Lh.shape
        k2, n = Rh.shape
        if k != k2:
            raise ValueError("lowrank: inner dimensions differ")
        out = C.c_void_p()
        ctx.check(L.lib().dtn_gpu_lowrank_create(ctx.h, Lh.ctypes.data, max(m, 1), Rh.ctypes.data, max(k, 1), m, n, k,
                                                 0, C.byref(out)))
        return LowRank(ctx, out)

    def __del__(self):
        try:
            if getattr(self, "h", None):
                L.lib().dtn_gpu_lowrank_free(self.h)
                self.h = None
        except Exception:
            pass

    def rows(self) -> int:
        return self._m

    def cols(self) -> int:
        return self._n

    def rank(self) -> int:
        return self._k

    def _fetch(self):
        if self._lr is None:
            Lf = np.zeros((self._m, self._k), order="F")
            R = np.zeros((self._k, self._n), order="F")
            self.ctx.check(L.lib().dtn_gpu_lowrank_get(self.h, Lf.ctypes.data, max(self._m, 1), R.ctypes.data,
                                                       max(self._k, 1)))
            self._lr = (Lf, R)
        return self._lr

    @property
    def L(self) -> np.ndarray:
        return self._fetch()[0]

    @property
    def R(self) -> np.ndarray:
        return self._fetch()[1]

    def dense(self) -> np.ndarray:
        Lf, R = self._fetch()
        return Lf @ R


@dataclass
class Placed:
    """PlacedLowRank (lowrank.hpp): a low-rank block at (row_offset, col_offset)."""
    row_offset: int
    col_offset: int
    lr: LowRank


def lowrank_from_dense(X, eps: float, ctx: Context | None = None) -> LowRank:
    """lowrank_from_dense (lowrank.cpp:27-36): the eps-truncated factorization of X."""
    ctx = _ctx(ctx)
    A = np.asfortranarray(np.asarray(X, dtype=np.float64))
    out = C.c_void_p()
    ctx.check(L.lib().dtn_gpu_lowrank_from_dense(ctx.h, A.ctypes.data, max(A.shape[0], 1), A.shape[0], A.shape[1], 0,
                                                 float(eps), C.byref(out)))
    return LowRank(ctx, out)


def lowrank_recompress(x: LowRank, eps: float) -> LowRank:
    """lowrank_recompress (lowrank.cpp:38-56)."""
    out = C.c_void_p()
    x.ctx.check(L.lib().dtn_gpu_lowrank_recompress(x.h, float(eps), C.byref(out)))
    return LowRank(x.ctx, out)


def lowrank_sum(m: int, n: int, terms, eps: float, ctx: Context | None = None) -> LowRank:
    """lowrank_sum (lowrank.cpp:58-72): the sum of placed low-rank terms, recompressed."""
    ctx = _ctx(ctx if ctx is not None else (terms[0].lr.ctx if terms else None))
    hs = (C.c_void_p * max(len(terms), 1))(*[t.lr.h for t in terms])
    offs = np.ascontiguousarray([[t.row_offset, t.col_offset] for t in terms] or [[0, 0]], dtype=np.int64)
    out = C.c_void_p()
    ctx.check(L.lib().dtn_gpu_lowrank_sum(ctx.h, int(m), int(n), len(terms), hs, offs.ctypes.data, float(eps),
                                          C.byref(out)))
    return LowRank(ctx, out)


@dataclass
class SplitParts:
    """SplitParts (hbs_ops.hpp) with both accumulations consolidated: lo = H[:pos, :pos],
    hi = H[pos:, pos:] (None when empty) on the reference's spine trees, lo_hi = H[:pos, pos:],
    hi_lo = H[pos:, :pos] as low-rank blocks."""
    lo: HbsMatrix | None
    hi: HbsMatrix | None
    lo_hi: LowRank
    hi_lo: LowRank


def split_at(H: HbsMatrix, pos: int, eps: float = 1e-12) -> SplitParts:
    """split_at (hbs_ops.cpp:620-640) followed by consolidate of each side (hbs_ops.cpp:710-735)."""
    lo, hi, a, b = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_void_p()
    H.ctx.check(L.lib().dtn_gpu_hbs_split_at(H.h, int(pos), float(eps), C.byref(lo), C.byref(hi), C.byref(a),
                                             C.byref(b)))
    return SplitParts(HbsMatrix(H.ctx, lo) if lo.value else None, HbsMatrix(H.ctx, hi) if hi.value else None,
                      LowRank(H.ctx, a), LowRank(H.ctx, b))


def consolidate(pieces, offsets, corrections=(), eps: float = 1e-12, size: int | None = None) -> HbsMatrix:
    """consolidate (hbs_ops.cpp:710-735): HBS pieces tiling [0, size) at `offsets` joined on the
    reference's spine tree (build_spine, hbs_ops.cpp:676-708), plus the placed low-rank
    corrections (Placed), recompressed at eps."""
    if not pieces:
        raise ValueError("consolidate: no pieces")
    ctx = pieces[0].ctx
    if size is None:
        size = int(offsets[-1]) + pieces[-1].size()
    ph = (C.c_void_p * len(pieces))(*[p.h for p in pieces])
    po = np.ascontiguousarray(offsets, dtype=np.int64)
    corrections = list(corrections)
    ch = (C.c_void_p * max(len(corrections), 1))(*[c.lr.h for c in corrections])
    co = np.ascontiguousarray([[c.row_offset, c.col_offset] for c in corrections] or [[0, 0]], dtype=np.int64)
    out = C.c_void_p()
    ctx.check(L.lib().dtn_gpu_hbs_consolidate(ctx.h, int(size), len(pieces), ph, po.ctypes.data, len(corrections), ch,
                                              co.ctypes.data, float(eps), C.byref(out)))
    return HbsMatrix(ctx, out)
