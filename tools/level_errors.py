"""Per-level relative error of the GPU box Schur complements vs the oracle (same tree)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1302_5995_b200 as dtn
from oracle import oracle as O
nint = int(sys.argv[1]); leaf = int(sys.argv[2]); micro = int(sys.argv[3]); cfg = int(sys.argv[4])
n = nint + 2
oname = {1: ("laplace", 0.0), 2: ("helmholtz", 40.0), 3: ("varcoef", 60.0), 5: ("helmholtz", 100.0)}[cfg]
sol = dtn.build_root_gpu(dtn.discretize(dtn.baseline_problem(cfg, nint)), dtn.build_tree_uniform(n, leaf), micro_max=micro)
t = O.Tree(n, uniform_side=leaf)
ref = O.build_root_dense(O.Problem(oname[0], n, oname[1]), t, threads=16, mode=2, keep_all=True)
for lev in range(t.depth, -1, -1):
    errs = [O.rel_fro(sol.box_schur(b), ref.box_S(b)) for b in t.levels[lev][:64]]
    print(f"level {lev}: boxes {len(t.levels[lev])} max rel err {max(errs):.3e} median {np.median(errs):.3e}", flush=True)
