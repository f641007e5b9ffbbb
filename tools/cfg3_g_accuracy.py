"""Config 3 (near-resonant): accuracy of the dense G g against a sparse direct solve, and S
against the oracle, for the current engine knobs (run once per knob setting: the knobs are
read once per process). Usage: python tools/cfg3_g_accuracy.py [micro_max]"""
import sys
import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla
sys.path.insert(0, ".")
import paper_1302_5995_b200 as dtn
from oracle import oracle as O

micro = int(sys.argv[1]) if len(sys.argv) > 1 else 128
n, s = 1026, 1024
op = dtn.discretize(dtn.baseline_problem(3, s))
sol = dtn.build_root_gpu(op, dtn.build_tree_uniform(n, 32), micro_max=micro)
ref = O.build_root_dense(O.Problem("varcoef", n, 60.0), O.Tree(n, uniform_side=32), threads=16, mode=2)
st = op.stencil
idx = np.arange(s * s)
x, y = idx % s, idx // s
rows, cols, vals = [idx], [idx], [st[0]]
for r, (dx, dy) in enumerate([(1, 0), (-1, 0), (0, 1), (0, -1)], start=1):
    ok = (x + dx >= 0) & (x + dx < s) & (y + dy >= 0) & (y + dy < s)
    rows.append(idx[ok]); cols.append((idx + dx + dy * s)[ok]); vals.append(st[r][ok])
A = sp.csc_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(s * s, s * s))
b = sol.boundary
lu = spla.splu(A)
out = []
for seed in (3, 4, 5):
    g = np.random.default_rng(seed).standard_normal(len(b))
    rhs = np.zeros(s * s)
    rhs[b] = g
    ub = lu.solve(rhs)[b]
    out.append((np.linalg.norm(dtn.apply_dtn(sol, g) - ub) / np.linalg.norm(ub),
                np.linalg.norm(ref.G @ g - ub) / np.linalg.norm(ub)))
print("S vs oracle", O.rel_fro(sol.S_dense, ref.S), "G g vs sparse direct (gpu, oracle):", out,
      "cond", sol.cond_estimate if hasattr(sol, "cond_estimate") else None)
