"""Accuracy of the GPU partial LU (Schur complement) on ill-conditioned systems vs
LAPACK, both against an extended-precision (long double) GEPP reference."""
import os, sys, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1302_5995_b200 import _lib as L

def gpu_schur(A, ni):
    n = A.shape[0]; A = np.asfortranarray(A); out = np.zeros_like(A, order="F")
    ipiv = np.zeros(ni, dtype=np.int32); ps = np.zeros(2)
    assert L.lib().dtn_debug_partial_lu(n, ni, A.ctypes.data, out.ctypes.data, ipiv.ctypes.data, ps.ctypes.data) == 0
    return out[ni:, ni:]

def ld_schur(A, ni):
    M = A.astype(np.longdouble).copy(); n = M.shape[0]
    for j in range(ni):
        p = j + int(np.argmax(np.abs(M[j:ni, j])))
        M[[j, p], :] = M[[p, j], :]
        l = M[j + 1:, j] / M[j, j]
        M[j + 1:, j + 1:] -= np.outer(l, M[j, j + 1:])
    return M[ni:, ni:]

def lapack_schur(A, ni):
    return A[ni:, ni:] - A[ni:, :ni] @ np.linalg.solve(A[:ni, :ni], A[:ni, ni:])

rng = np.random.default_rng(0)
for n, ni, cond in [(600, 200, 1e8), (1000, 400, 1e8), (2000, 700, 1e8), (3064, 1020, 1e8), (4000, 1500, 1e8)]:
    U, _ = np.linalg.qr(rng.standard_normal((ni, ni))); V, _ = np.linalg.qr(rng.standard_normal((ni, ni)))
    s = np.logspace(0, -np.log10(cond), ni)
    A = rng.standard_normal((n, n))
    A[:ni, :ni] = (U * s) @ V.T
    ref = ld_schur(A, ni)
    rn = float(np.linalg.norm(ref.astype(np.float64)))
    eg = float(np.linalg.norm((gpu_schur(A, ni) - ref).astype(np.float64))) / rn
    el = float(np.linalg.norm((lapack_schur(A, ni) - ref).astype(np.float64))) / rn
    print(f"n {n} ni {ni} cond {cond:.0e}: gpu {eg:.3e}  lapack {el:.3e}", flush=True)
