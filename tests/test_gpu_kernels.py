"""Kernel-level GPU checks of the blocked partial LU (panel / rowpanel /
trailing DMMA GEMM) against numpy/scipy."""
import ctypes as C

import numpy as np
import pytest
import scipy.linalg as sla

from paper_1302_5995_b200 import _lib as L

pytestmark = pytest.mark.gpu


def gpu_partial_lu(A, ni):
    n = A.shape[0]
    A = np.asfortranarray(A, dtype=np.float64)
    out = np.zeros_like(A, order="F")
    ipiv = np.zeros(ni, dtype=np.int32)
    ps = np.zeros(2)
    rc = L.lib().dtn_debug_partial_lu(n, ni, A.ctypes.data, out.ctypes.data, ipiv.ctypes.data, ps.ctypes.data)
    assert rc == 0, L.lib().dtn_gpu_last_error(None).decode()
    return out, ipiv, ps


@pytest.mark.parametrize("n", [5, 20, 33, 64, 100, 257, 600, 1100, 2100, 4100, 8190])
def test_full_lu_matches_scipy(n):
    rng = np.random.default_rng(n)
    A = rng.standard_normal((n, n))
    out, ipiv, ps = gpu_partial_lu(A, n)
    # P A = L U with the GPU's row permutation perm[pos] = original row (partial
    # pivoting; near-ties may resolve differently from LAPACK, so compare the
    # factorization, not the pivot sequence)
    assert sorted(ipiv.tolist()) == list(range(n))
    PA = A[ipiv]
    Lm = np.tril(out, -1) + np.eye(n)
    Um = np.triu(out)
    assert np.max(np.abs(Lm)) <= 1.0 + 1e-12          # partial pivoting bound |l_ij| <= 1
    assert np.linalg.norm(Lm @ Um - PA) / np.linalg.norm(A) <= 1e-13
    assert ps[0] == pytest.approx(np.min(np.abs(np.diag(Um))))


@pytest.mark.parametrize("n", [33, 64, 100, 600, 2100, 4100, 8190])
def test_full_lu_fused_lookahead(n, monkeypatch):
    """The fused look-ahead sequence (panel prologue applies the previous step
    to its own columns; rowpanel / trailing skip them) gives a valid P A = L U."""
    monkeypatch.setenv("DTN_DEBUG_LU_FUSED", "1")
    rng = np.random.default_rng(n + 7)
    A = rng.standard_normal((n, n))
    out, ipiv, ps = gpu_partial_lu(A, n)
    assert sorted(ipiv.tolist()) == list(range(n))
    Lm = np.tril(out, -1) + np.eye(n)
    Um = np.triu(out)
    assert np.max(np.abs(Lm)) <= 1.0 + 1e-12
    assert np.linalg.norm(Lm @ Um - A[ipiv]) / np.linalg.norm(A) <= 1e-13
    assert ps[0] == pytest.approx(np.min(np.abs(np.diag(Um))))


@pytest.mark.parametrize("n", [64, 300, 1100, 2100])
@pytest.mark.parametrize("swap_at", [None, 0, 45, 97])
def test_full_lu_no_interchange_fast_path(n, swap_at, monkeypatch):
    """Diagonally dominant systems take the panel's no-interchange path (result
    identical to partial pivoting: identity permutation); a single off-diagonal
    entry larger than its pivot forces that panel back onto the pivoted loop."""
    monkeypatch.setenv("DTN_DEBUG_LU_FUSED", "1")
    rng = np.random.default_rng(n)
    A = rng.uniform(-1, 1, (n, n))
    A[np.arange(n), np.arange(n)] = 2.0 * n
    if swap_at is not None and swap_at + 5 < n:
        A[swap_at + 5, swap_at] = 4.0 * n  # partial pivoting must interchange at step swap_at
    out, ipiv, _ = gpu_partial_lu(A, n)
    Lm = np.tril(out, -1) + np.eye(n)
    Um = np.triu(out)
    assert np.max(np.abs(Lm)) <= 1.0 + 1e-12
    assert np.linalg.norm(Lm @ Um - A[ipiv]) / np.linalg.norm(A) <= 1e-14
    moved = np.flatnonzero(ipiv != np.arange(n))
    if swap_at is None or swap_at + 5 >= n:
        assert moved.size == 0
    else:
        assert swap_at in moved


@pytest.mark.parametrize("n,ni", [(40, 12), (184, 60), (376, 124), (1528, 508), (3064, 1020), (6136, 2044)])
def test_partial_lu_schur(n, ni):
    rng = np.random.default_rng(ni)
    A = rng.standard_normal((n, n))
    out, ipiv, ps = gpu_partial_lu(A, ni)
    S = A[ni:, ni:] - A[ni:, :ni] @ np.linalg.solve(A[:ni, :ni], A[:ni, ni:])
    assert np.linalg.norm(out[ni:, ni:] - S) / np.linalg.norm(S) <= 1e-11


def _check_lu_by_products(A, out, ipiv, tol):
    """P A = L U checked through products with random vectors (O(n^2), any size)."""
    n = A.shape[0]
    assert sorted(ipiv.tolist()) == list(range(n))
    Lm = np.tril(out, -1)
    Um = np.triu(out)
    assert np.max(np.abs(Lm)) <= 1.0 + 1e-12
    X = np.random.default_rng(1).standard_normal((n, 4))
    UX = Um @ X
    LUX = Lm @ UX + UX
    r = np.linalg.norm(LUX - A[ipiv] @ X) / (np.linalg.norm(A) * np.linalg.norm(X))
    assert r <= tol


@pytest.mark.parametrize("n", [5, 100, 600, 2100])
def test_tall_panel_full_lu(n, monkeypatch):
    """The tall panel (global-memory pivot exchange across TG CTAs, one software grid
    barrier per pivot), forced at small sizes: a valid partial-pivoting P A = L U whose
    pivot sequence is LAPACK's (largest |a|, ties to the lowest row) on random data."""
    monkeypatch.setenv("DTN_PANEL_TALL_MIN", "1")
    rng = np.random.default_rng(n + 11)
    A = rng.standard_normal((n, n))
    out, ipiv, ps = gpu_partial_lu(A, n)
    _check_lu_by_products(A, out, ipiv, 1e-14)
    assert ps[0] == pytest.approx(np.min(np.abs(np.diag(out))))
    # LAPACK getrf's row permutation
    lu, piv = sla.lu_factor(A)
    perm = np.arange(n)
    for i, p in enumerate(piv):
        perm[[i, p]] = perm[[p, i]]
    assert np.array_equal(perm, ipiv)


@pytest.mark.parametrize("n,ni", [(376, 124), (3064, 1020)])
def test_tall_panel_schur(n, ni, monkeypatch):
    monkeypatch.setenv("DTN_PANEL_TALL_MIN", "1")
    rng = np.random.default_rng(ni + 3)
    A = rng.standard_normal((n, n))
    out, ipiv, ps = gpu_partial_lu(A, ni)
    S = A[ni:, ni:] - A[ni:, :ni] @ np.linalg.solve(A[:ni, :ni], A[:ni, ni:])
    assert np.linalg.norm(out[ni:, ni:] - S) / np.linalg.norm(S) <= 1e-11


@pytest.mark.parametrize("n", [8200, 16380])
def test_tall_panel_beyond_cluster_limit(n):
    """Beyond the cluster panel's 8192 rows the tall panel takes over by default
    (the config-4 root LU for G = S^{-1} is 16380 x 16380)."""
    rng = np.random.default_rng(n)
    A = rng.standard_normal((n, n))
    out, ipiv, ps = gpu_partial_lu(A, n)
    _check_lu_by_products(A, out, ipiv, 1e-13)


# ---- FP64 tensor-core GEMMs: cp.async-staged kernels and the TMA-staged kernel (k_tma.cu)
def gpu_gemm(A, B, C0, alpha, beta, path):
    m, k = A.shape
    n = B.shape[1]
    A = np.asfortranarray(A)
    B = np.asfortranarray(B)
    Cio = np.asfortranarray(C0).copy(order="F")
    rc = L.lib().dtn_debug_gemm(m, n, k, A.ctypes.data, B.ctypes.data, Cio.ctypes.data, alpha, beta, path)
    assert rc == 0, L.lib().dtn_gpu_last_error(None).decode()
    return Cio


@pytest.mark.parametrize("shape", [(128, 128, 64), (130, 131, 70), (300, 257, 129), (1000, 777, 70),
                                   (2044, 1916, 510), (4100, 520, 1030)])
@pytest.mark.parametrize("ab", [(-1.0, 1.0), (1.0, 0.0), (-1.0, 0.0), (0.5, 2.0)])
def test_gemm_tma_matches_numpy(shape, ab):
    """Ragged tiles in m, n and k (TMA zero-fill outside the tensor-map bounds), every
    (alpha, beta) the engine uses; the cp.async path on the same inputs beside it."""
    m, n, k = shape
    alpha, beta = ab
    rng = np.random.default_rng(m + 3 * n + 7 * k)
    A = rng.uniform(-1, 1, (m, k))
    B = rng.uniform(-1, 1, (k, n))
    C0 = rng.uniform(-1, 1, (m, n))
    ref = alpha * (A @ B) + beta * C0
    scale = np.abs(A) @ np.abs(B) + np.abs(C0)          # componentwise bound of the rounding error
    for path in (0, 1):
        got = gpu_gemm(A, B, C0, alpha, beta, path)
        assert np.max(np.abs(got - ref) / scale) <= 4e-16 * np.sqrt(k) + 1e-15, (path, shape, ab)
