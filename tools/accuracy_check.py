"""Accuracy of S*g against an independent sparse direct solve (scipy SuperLU on the
assembled 5-point matrix) for the config-3 operator at n=1024: GPU vs oracle."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla
import paper_1302_5995_b200 as dtn
from oracle import oracle as O

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1026
nint = n - 2
op = dtn.discretize(dtn.baseline_problem(3, nint))
st = op.stencil
s = nint
idx = np.arange(s * s); x = idx % s; y = idx // s
rows = [idx]; cols = [idx]; vals = [st[0]]
for r, (dx, dy) in enumerate([(1, 0), (-1, 0), (0, 1), (0, -1)], start=1):
    ok = (x + dx >= 0) & (x + dx < s) & (y + dy >= 0) & (y + dy < s)
    rows.append(idx[ok]); cols.append((idx + dx + dy * s)[ok]); vals.append(st[r][ok])
A = sp.csc_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(s * s, s * s))
t0 = time.time(); lu = spla.splu(A); print("splu %.1fs" % (time.time() - t0), flush=True)
results = {}
sol_u = dtn.build_root_gpu(op, dtn.build_tree_uniform(n, 32))
sol_r = dtn.build_root_gpu(op, dtn.build_tree(n, 1089))
ref_u = O.build_root_dense(O.Problem("varcoef", n, 60.0), O.Tree(n, uniform_side=32), threads=16, mode=2)
ref_r = O.build_root_dense(O.Problem("varcoef", n, 60.0), O.Tree(n, 1089), threads=16, mode=1)
b = ref_u.boundary
rng = np.random.default_rng(3)
g = rng.standard_normal(len(b))
# exact: solve A u = e_b g (loads on the boundary ring), u_b = G g
rhs = np.zeros(s * s); rhs[b] = g
u = lu.solve(rhs)
# mixed-precision iterative refinement: residual of the 5-point stencil in long double
ld = np.longdouble
stl = st.astype(ld)
def resid(u):
    U = u.astype(ld).reshape(s, s)
    R = rhs.astype(ld).reshape(s, s) - stl[0].reshape(s, s) * U
    R[:, :-1] -= stl[1].reshape(s, s)[:, :-1] * U[:, 1:]
    R[:, 1:] -= stl[2].reshape(s, s)[:, 1:] * U[:, :-1]
    R[:-1, :] -= stl[3].reshape(s, s)[:-1, :] * U[1:, :]
    R[1:, :] -= stl[4].reshape(s, s)[1:, :] * U[:-1, :]
    return R.reshape(-1)
for it in range(4):
    r = resid(u)
    print("refinement", it, "residual %.3e" % float(np.linalg.norm(r.astype(np.float64)) / np.linalg.norm(rhs)), flush=True)
    du = lu.solve(r.astype(np.float64))
    u = (u.astype(ld) + du.astype(ld)).astype(np.float64)
    print("   correction %.3e" % (np.linalg.norm(du) / np.linalg.norm(u)), flush=True)
ub = u[b]
# residual-refined reference
for name, S, G in [("gpu-uniform", sol_u.S_dense, sol_u.G_dense), ("gpu-reftree", sol_r.S_dense, sol_r.G_dense),
                   ("oracle-uniform", ref_u.S, ref_u.G), ("oracle-reftree", ref_r.S, ref_r.G)]:
    print(f"{name:15s} |G g - u_b|/|u_b| = {np.linalg.norm(G @ g - ub) / np.linalg.norm(ub):.3e}   "
          f"|S u_b - g|/|g| = {np.linalg.norm(S @ ub - g) / np.linalg.norm(g):.3e}", flush=True)
print("S diffs: gpu-u vs oracle-u %.3e, gpu-r vs oracle-r %.3e, gpu-u vs gpu-r %.3e, oracle-u vs oracle-r %.3e" % (
    O.rel_fro(sol_u.S_dense, ref_u.S), O.rel_fro(sol_r.S_dense, ref_r.S), O.rel_fro(sol_u.S_dense, sol_r.S_dense),
    O.rel_fro(ref_u.S, ref_r.S)))
