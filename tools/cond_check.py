"""How far apart are two valid FP64 eliminations of the same operator?
(oracle vs oracle with a different partition / BLAS blocking) — the parity floor."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as O
for name, n, par in [("varcoef", 1026, 60.0), ("helmholtz", 514, 40.0), ("helmholtz", 258, 0.0)]:
    p = O.Problem(name, n, par)
    t0 = time.time()
    a = O.build_root_dense(p, O.Tree(n, uniform_side=32 if n > 600 else 16), threads=16, mode=2)
    b = O.build_root_dense(p, O.Tree(n, 1089 if n > 600 else 289), threads=16, mode=1)
    print(name, n, "uniform-vs-reference-tree rel_fro(S) = %.3e" % O.rel_fro(a.S, b.S), "cond %.3e" % a.cond, "%.1fs" % (time.time() - t0), flush=True)
