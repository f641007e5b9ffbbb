import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1302_5995_b200 import _lib as L

def gpu(A, ni):
    n = A.shape[0]; A = np.asfortranarray(A); out = np.zeros_like(A, order="F")
    ipiv = np.zeros(ni, dtype=np.int32); ps = np.zeros(2)
    rc = L.lib().dtn_debug_partial_lu(n, ni, A.ctypes.data, out.ctypes.data, ipiv.ctypes.data, ps.ctypes.data)
    assert rc == 0
    return out, ipiv

def ref(A, ni):
    A = A.copy(); n = A.shape[0]; piv = []
    for j in range(ni):
        p = j + int(np.argmax(np.abs(A[j:ni, j]))); piv.append(p)
        A[[j, p], :] = A[[p, j], :]
        A[j+1:, j] /= A[j, j]
        A[j+1:, j+1:] -= np.outer(A[j+1:, j], A[j, j+1:])
    return A, np.array(piv)

rng = np.random.default_rng(20)
A = rng.standard_normal((20, 20))
for ni in range(1, 14):
    g, gp = gpu(A, ni); r, rp = ref(A, ni)
    print(ni, "piv ok" if np.array_equal(gp, rp) else f"piv {gp} vs {rp}", "maxdiff", np.abs(g - r).max(),
          "rows", sorted(set(np.where(np.abs(g - r) > 1e-9)[0]))[:10], "cols", sorted(set(np.where(np.abs(g - r) > 1e-9)[1]))[:10])
np.set_printoptions(linewidth=250, precision=2, suppress=True)
for ni in (9, 20):
    g, gp = gpu(A, ni); r, rp = ref(A, ni)
    print("ni", ni, "diff mask (rows x cols):")
    print((np.abs(g - r) > 1e-9).astype(int)[:20, :20])
    print("gpu col 8", g[:12, 8]); print("ref col 8", r[:12, 8])
    print("gpu row 8", g[8, :12]); print("ref row 8", r[8, :12])
