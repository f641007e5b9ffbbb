"""Which box Schur complements are accurate? S x vs a sparse solve (refined) for the worst boxes per level."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla
import paper_1302_5995_b200 as dtn
from oracle import oracle as O
nint, leaf, micro, cfg = 1024, 32, 64, 3
n = nint + 2; s = nint
op = dtn.discretize(dtn.baseline_problem(cfg, nint))
st = op.stencil
sol = dtn.build_root_gpu(op, dtn.build_tree_uniform(n, leaf), micro_max=micro)
t = O.Tree(n, uniform_side=leaf)
ref = O.build_root_dense(O.Problem("varcoef", n, 60.0), t, threads=16, mode=2, keep_all=True)
idx = np.arange(s * s); X = idx % s; Y = idx // s
rows = [idx]; cols = [idx]; vals = [st[0]]
for r, (dx, dy) in enumerate([(1, 0), (-1, 0), (0, 1), (0, -1)], start=1):
    ok = (X + dx >= 0) & (X + dx < s) & (Y + dy >= 0) & (Y + dy < s)
    rows.append(idx[ok]); cols.append((idx + dx + dy * s)[ok]); vals.append(st[r][ok])
A = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(s * s, s * s))
rng = np.random.default_rng(1)
for lev in [3, 2, 1, 0]:
    errs = [(O.rel_fro(sol.box_schur(b), ref.box_S(b)), b) for b in t.levels[lev]]
    e, bid = max(errs)
    bx = t.boxes[bid]
    B, I = bx["boundary"], bx["interior"]
    Aii = A[I][:, I].tocsc(); Aib = A[I][:, B]; Abi = A[B][:, I]; Abb = A[B][:, B]
    lu = spla.splu(Aii)
    x = rng.standard_normal(len(B))
    y = Aib @ x
    z = lu.solve(y)
    for _ in range(2):  # refinement
        z = z + lu.solve(y - Aii @ z)
    Sx = Abb @ x - Abi @ z
    eg = np.linalg.norm(sol.box_schur(bid) @ x - Sx) / np.linalg.norm(Sx)
    eo = np.linalg.norm(ref.box_S(bid) @ x - Sx) / np.linalg.norm(Sx)
    print(f"level {lev} box {bid} gpu-vs-oracle {e:.2e}: |S x - exact| gpu {eg:.2e} oracle {eo:.2e}", flush=True)
