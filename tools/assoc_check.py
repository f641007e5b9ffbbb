"""Oracle with the reference association vs the right-looking association, accuracy of S x
at the top boxes (config-3 operator, n=1024) against refined sparse solves."""
import os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
if len(sys.argv) > 1:
    import scipy.sparse as sp, scipy.sparse.linalg as spla
    import paper_1302_5995_b200 as dtn
    from oracle import oracle as O
    nint = 1024; n = nint + 2; s = nint
    op = dtn.discretize(dtn.baseline_problem(3, nint)); st = op.stencil
    t = O.Tree(n, uniform_side=32)
    ref = O.build_root_dense(O.Problem("varcoef", n, 60.0), t, threads=16, mode=2, keep_all=True)
    idx = np.arange(s * s); X = idx % s; Y = idx // s
    rows = [idx]; cols = [idx]; vals = [st[0]]
    for r, (dx, dy) in enumerate([(1, 0), (-1, 0), (0, 1), (0, -1)], start=1):
        ok = (X + dx >= 0) & (X + dx < s) & (Y + dy >= 0) & (Y + dy < s)
        rows.append(idx[ok]); cols.append((idx + dx + dy * s)[ok]); vals.append(st[r][ok])
    A = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(s * s, s * s))
    rng = np.random.default_rng(1)
    for lev, bid in [(1, 1), (0, 0)]:
        bx = t.boxes[bid]; B, I = bx["boundary"], bx["interior"]
        Aii = A[I][:, I].tocsc(); lu = spla.splu(Aii)
        x = rng.standard_normal(len(B)); y = A[I][:, B] @ x; z = lu.solve(y)
        for _ in range(2): z = z + lu.solve(y - Aii @ z)
        Sx = A[B][:, B] @ x - A[B][:, I] @ z
        print(sys.argv[1], f"level {lev}: |S x - exact| = {np.linalg.norm(ref.box_S(bid) @ x - Sx) / np.linalg.norm(Sx):.2e}", flush=True)
    sys.exit(0)
for mode in ["reference-assoc", "right-looking-assoc"]:
    e = dict(os.environ)
    if mode.startswith("right"): e["ORC_RIGHT_LOOKING_ASSOC"] = "1"
    print(subprocess.run([sys.executable, __file__, mode], env=e, capture_output=True, text=True).stdout, flush=True)
