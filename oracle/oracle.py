"""ORACLE — TEST INFRASTRUCTURE ONLY (see dense_oracle.cpp header).

ctypes wrapper over oracle/_build/liboracle.so, the C++ restatement of the
reference's dense build (proj/src/grid.cpp, proj/src/dense_nd.cpp), plus
`brute_schur`, the reference tests' independent checker
(proj/tests/test_dense_nd.cpp:35-54): one dense elimination of the assembled
matrix. Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs
may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        vp, i32, i64, f64 = C.c_void_p, C.c_int, C.c_int64, C.c_double
        P = C.POINTER
        L.orc_last_error.restype = C.c_char_p
        L.orc_problem_create.argtypes = [C.c_char_p, i32, f64, C.c_uint64, P(vp)]
        L.orc_problem_free.argtypes = [vp]
        L.orc_problem_stencil.argtypes = [vp, P(f64)]
        L.orc_problem_coeff.argtypes = [vp, i64, i64]
        L.orc_problem_coeff.restype = f64
        L.orc_tree_create.argtypes = [i32, i32, i32, P(vp)]
        L.orc_tree_free.argtypes = [vp]
        L.orc_tree_depth.argtypes = [vp]
        L.orc_tree_num_boxes.argtypes = [vp]
        L.orc_tree_level_size.argtypes = [vp, i32]
        L.orc_tree_level.argtypes = [vp, i32, P(i32)]
        L.orc_tree_box.argtypes = [vp, i32, P(i64)]
        L.orc_tree_box_sets.argtypes = [vp, i32, P(i64), P(i64)]
        L.orc_build_dense.argtypes = [vp, vp, i32, i32, i32, P(vp)]
        L.orc_result_free.argtypes = [vp]
        L.orc_result_nb.argtypes = [vp]
        L.orc_result_nb.restype = i64
        L.orc_result_root.argtypes = [vp, P(i64), P(f64), P(f64), P(f64), P(f64)]
        L.orc_result_box.argtypes = [vp, i32, P(f64)]
        L.orc_result_box.restype = i64
        L.orc_leaf_rect.argtypes = [vp, i32, i32, i32, i32, P(f64), P(i64)]
        L.orc_merge_rects.argtypes = [vp, P(i32), P(i32), P(f64), P(i64)]
        L.orc_merge_given.argtypes = [vp, P(i32), P(f64), P(i32), P(f64), P(f64), P(i64)]
        L.orc_random_unit_boundary.argtypes = [i64, C.c_uint64, P(f64)]
        L.orc_smooth_boundary.argtypes = [i64, P(f64)]
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def _check(rc: int):
    if rc != 0:
        raise OracleError(rc, lib().orc_last_error().decode())


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _ip(a: np.ndarray, t=C.c_int64):
    return a.ctypes.data_as(C.POINTER(t))


class Problem:
    """Discretized operator (grid.cpp:106-168); name = catalog name
    (problems.cpp:26-73) or 'helmholtz' / 'varcoef' with param = kappa."""

    def __init__(self, name: str, n: int, param: float = 0.0, seed: int = 0):
        h = C.c_void_p()
        _check(lib().orc_problem_create(name.encode(), n, float(param), seed, C.byref(h)))
        self.h, self.n = h, n

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.orc_problem_free(self.h)

    @property
    def nu(self) -> int:
        return (self.n - 2) ** 2

    def stencil(self) -> np.ndarray:
        out = np.zeros((5, self.nu))
        lib().orc_problem_stencil(self.h, _dp(out))
        return out

    def coeff(self, row: int, col: int) -> float:
        return lib().orc_problem_coeff(self.h, row, col)

    def dense_A(self) -> np.ndarray:
        """Assembled A (nu x nu) — small n only."""
        st = self.stencil()
        s = self.n - 2
        A = np.zeros((self.nu, self.nu))
        idx = np.arange(self.nu)
        x, y = idx % s, idx // s
        A[idx, idx] = st[0]
        for r, (dx, dy) in enumerate([(1, 0), (-1, 0), (0, 1), (0, -1)], start=1):
            qx, qy = x + dx, y + dy
            ok = (qx >= 0) & (qx < s) & (qy >= 0) & (qy < s)
            A[idx[ok], (qy * s + qx)[ok]] = st[r][ok]
        return A


class Tree:
    """build_tree (grid.cpp:213-266); uniform_side > 0 = exact halving."""

    def __init__(self, n: int, n_leaf: int = 16, uniform_side: int = 0):
        h = C.c_void_p()
        _check(lib().orc_tree_create(n, n_leaf, uniform_side, C.byref(h)))
        self.h, self.n = h, n
        L = lib()
        self.depth = L.orc_tree_depth(h)
        self.levels = []
        for lev in range(self.depth + 1):
            ids = np.zeros(L.orc_tree_level_size(h, lev), dtype=np.int32)
            L.orc_tree_level(h, lev, _ip(ids, C.c_int))
            self.levels.append([int(i) for i in ids])
        self.boxes = []
        for bid in range(L.orc_tree_num_boxes(h)):
            info = np.zeros(16, dtype=np.int64)
            L.orc_tree_box(h, bid, _ip(info))
            nb, ni = int(info[14]), int(info[15])
            bnd = np.zeros(max(nb, 1), dtype=np.int64)
            inr = np.zeros(max(ni, 1), dtype=np.int64)
            L.orc_tree_box_sets(h, bid, _ip(bnd), _ip(inr))
            self.boxes.append(dict(id=bid, level=int(info[0]), parent=int(info[1]),
                                   children=[int(c) for c in info[2:6]],
                                   x0=int(info[6]), x1=int(info[7]), y0=int(info[8]), y1=int(info[9]),
                                   gx0=int(info[10]), gx1=int(info[11]), gy0=int(info[12]), gy1=int(info[13]),
                                   boundary=bnd[:nb].copy(), interior=inr[:ni].copy()))

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.orc_tree_free(self.h)

    def root(self):
        return self.boxes[0]


class DenseResult:
    def __init__(self, h):
        self.h = h
        L = lib()
        nb = L.orc_result_nb(h)
        self.boundary = np.zeros(nb, dtype=np.int64)
        self.S = np.zeros((nb, nb), order="F")
        self.G = np.zeros((nb, nb), order="F")
        cond = C.c_double()
        secs = np.zeros(2)
        L.orc_result_root(h, _ip(self.boundary), _dp(self.S), _dp(self.G), C.byref(cond), _dp(secs))
        self.cond = cond.value
        self.seconds_build, self.seconds_inverse = float(secs[0]), float(secs[1])

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.orc_result_free(self.h)

    def box_S(self, box_id: int) -> np.ndarray | None:
        nb = lib().orc_result_box(self.h, box_id, None)
        if nb < 0:
            return None
        S = np.zeros((nb, nb), order="F")
        lib().orc_result_box(self.h, box_id, _dp(S))
        return S


def build_root_dense(problem: Problem, tree: Tree, threads: int = 1, mode: int = 0,
                     keep_all: bool = False) -> DenseResult:
    """build_root_dense (dense_nd.cpp:196-225). mode 0: all-core BLAS,
    boxes serial; mode 1: boxes of a level over `threads` workers, 1 BLAS
    thread each (the reference's own threading, accel_nd.cpp:635-659)."""
    h = C.c_void_p()
    _check(lib().orc_build_dense(problem.h, tree.h, threads, mode, int(keep_all), C.byref(h)))
    return DenseResult(h)


def leaf_rect(problem: Problem, x0: int, x1: int, y0: int, y1: int) -> np.ndarray:
    """leaf_schur (dense_nd.cpp:37-103) of an arbitrary unknown rectangle."""
    nb = C.c_int64()
    _check(lib().orc_leaf_rect(problem.h, x0, x1, y0, y1, None, C.byref(nb)))
    S = np.zeros((nb.value, nb.value), order="F")
    _check(lib().orc_leaf_rect(problem.h, x0, x1, y0, y1, _dp(S), C.byref(nb)))
    return S


def merge_rects(problem: Problem, ra, rb) -> np.ndarray:
    """merge_two (dense_nd.cpp:105-186) of two leaf rectangles (x0,x1,y0,y1)."""
    a = np.asarray(ra, dtype=np.int32)
    b = np.asarray(rb, dtype=np.int32)
    nb = C.c_int64()
    _check(lib().orc_merge_rects(problem.h, _ip(a, C.c_int), _ip(b, C.c_int), None, C.byref(nb)))
    S = np.zeros((nb.value, nb.value), order="F")
    _check(lib().orc_merge_rects(problem.h, _ip(a, C.c_int), _ip(b, C.c_int), _dp(S), C.byref(nb)))
    return S


def merge_given(problem: Problem, ra, Sa, rb, Sb):
    """merge_two (dense_nd.cpp:105-186) of two given Schur complements on
    rectangles ra, rb = (x0, x1, y0, y1); returns (rect, S)."""
    a = np.asarray(ra, dtype=np.int32)
    b = np.asarray(rb, dtype=np.int32)
    Sa = np.asfortranarray(Sa, dtype=np.float64)
    Sb = np.asfortranarray(Sb, dtype=np.float64)
    nb = C.c_int64()
    _check(lib().orc_merge_given(problem.h, _ip(a, C.c_int), _dp(Sa), _ip(b, C.c_int), _dp(Sb), None, C.byref(nb)))
    S = np.zeros((nb.value, nb.value), order="F")
    _check(lib().orc_merge_given(problem.h, _ip(a, C.c_int), _dp(Sa), _ip(b, C.c_int), _dp(Sb), _dp(S), C.byref(nb)))
    rect = (min(a[0], b[0]), max(a[1], b[1]), min(a[2], b[2]), max(a[3], b[3]))
    return rect, S


# ----------------------------------------------------------------- checkers
def rect_perimeter_ccw(x0, x1, y0, y1):
    """grid.cpp:170-190 (checker copy for brute-force index sets)."""
    if x0 > x1 or y0 > y1:
        return []
    if x0 == x1 and y0 == y1:
        return [(x0, y0)]
    if x0 == x1:
        return [(x0, y) for y in range(y0, y1 + 1)]
    if y0 == y1:
        return [(x, y0) for x in range(x0, x1 + 1)]
    p = [(x, y0) for x in range(x0, x1 + 1)]
    p += [(x1, y) for y in range(y0 + 1, y1 + 1)]
    p += [(x, y1) for x in range(x1 - 1, x0 - 1, -1)]
    p += [(x0, y) for y in range(y1 - 1, y0, -1)]
    return p


def rect_sets(n: int, x0, x1, y0, y1):
    s = n - 2
    uid = lambda x, y: (y - 1) * s + (x - 1)
    bnd = [uid(x, y) for x, y in rect_perimeter_ccw(x0, x1, y0, y1)]
    inr = [uid(x, y) for y in range(y0 + 1, y1) for x in range(x0 + 1, x1)]
    return np.array(bnd, dtype=np.int64), np.array(inr, dtype=np.int64)


def brute_schur(A: np.ndarray, b, i) -> np.ndarray:
    """test_dense_nd.cpp:35-54: abb - abi * aii^{-1} * aib, one dense solve."""
    b = np.asarray(b, dtype=np.int64)
    i = np.asarray(i, dtype=np.int64)
    abb = A[np.ix_(b, b)]
    if len(i) == 0:
        return abb.copy()
    return abb - A[np.ix_(b, i)] @ np.linalg.solve(A[np.ix_(i, i)], A[np.ix_(i, b)])


def rel_fro(a, b) -> float:
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))


CATALOG = ["laplace", "diffconv1", "diffconv2", "diffconv3", "diffconv4", "helmholtz1",
           "helmholtz2", "helmholtz3", "helmholtz4", "random1", "random2"]


def ring_dtn(problem: Problem, result: DenseResult) -> np.ndarray:
    """Dirichlet-ring DtN map on the 4 n_int non-corner ring nodes (ring_id
    order, grid.cpp:40-47): T = (1/h)(I + P G D_b) (SURVEY f-1; follows from
    A u = -D g, grid.hpp:88-90, with D's couplings from grid.cpp:151-157).
    Test infrastructure: restated independently of the product's adapter."""
    n = problem.n
    m, s, h = n - 1, n - 2, 1.0 / (n - 1)
    st = problem.stencil()
    pos = {int(b): i for i, b in enumerate(result.boundary)}
    adj, coef = [], []
    for rid in range(4 * m):
        side, off = divmod(rid, m)
        if off == 0:
            continue
        # (unknown adjacent to the ring node, stencil row toward the ring)
        ux, uy, r = [(off, 1, 4), (m - 1, off, 1), (m - off, m - 1, 3), (1, m - off, 2)][side]
        uid = (uy - 1) * s + (ux - 1)
        adj.append(pos[uid])
        coef.append(st[r, uid])
    adj = np.array(adj)
    coef = np.array(coef)
    return (np.eye(len(adj)) + result.G[np.ix_(adj, adj)] * coef[None, :]) / h



def random_unit_boundary(size: int, seed: int) -> np.ndarray:
    """reference.cpp:139-152 (restated in dense_oracle.cpp with std::mt19937_64)."""
    r = np.zeros(size)
    lib().orc_random_unit_boundary(size, seed, _dp(r))
    return r


def smooth_boundary(size: int) -> np.ndarray:
    """reference.cpp:154-161."""
    r = np.zeros(size)
    lib().orc_smooth_boundary(size, _dp(r))
    return r


def sparse_system(stencil: np.ndarray, n: int):
    """The full system matrix A (grid.cpp:128-166) from a 5 x (n-2)^2 stencil."""
    import scipy.sparse as sp
    s = n - 2
    idx = np.arange(s * s)
    x, y = idx % s, idx // s
    rows, cols, vals = [idx], [idx], [stencil[0]]
    for r, (dx, dy) in enumerate([(1, 0), (-1, 0), (0, 1), (0, -1)], start=1):
        ok = (x + dx >= 0) & (x + dx < s) & (y + dy >= 0) & (y + dy < s)
        rows.append(idx[ok]); cols.append((idx + dx + dy * s)[ok]); vals.append(stencil[r][ok])
    return sp.csc_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(s * s, s * s))


def error_metrics(apply_dtn, stencil: np.ndarray, n: int, boundary: np.ndarray, seed: int):
    """error_metrics (reference.cpp:163-177): e1 with the seeded random unit
    boundary vector, e2 with the smooth one; the exact answer from a sparse
    direct solve of the full system with boundary right-hand side
    (reference_dtn_apply, :122-137; SuperLU here in place of Eigen SparseLU,
    with the reference's residual check and up to 3 refinement steps)."""
    import scipy.sparse.linalg as spla
    A = sparse_system(stencil, n)
    lu = spla.splu(A)
    out = []
    for r in (random_unit_boundary(len(boundary), seed), smooth_boundary(len(boundary))):
        rhs = np.zeros(A.shape[0])
        rhs[boundary] = r
        x = lu.solve(rhs)
        res = np.linalg.norm(A @ x - rhs) / np.linalg.norm(rhs)
        for _ in range(3):
            if res <= 1e-6:
                break
            x = x + lu.solve(rhs - A @ x)
            res = np.linalg.norm(A @ x - rhs) / np.linalg.norm(rhs)
        if res > 1e-6:
            raise RuntimeError(f"error_metrics: direct solve residual {res:.3g} exceeds 1e-6")
        exact = x[boundary]
        approx = apply_dtn(r)
        out.append(float(np.linalg.norm(approx - exact) / np.linalg.norm(exact)))
    return tuple(out)
