"""Accuracy of the structured merges against the oracle and the exact dense GPU
engine, as a function of the factor-rank schedule (DTN_RANK_TOL in the env sets the
range-finder acceptance; 1e30 disables the adaptive retries).
Usage: DTN_RANK_TOL=1e30 python tools/k5_accuracy.py"""
import os
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_1302_5995_b200 as dtn
from oracle import oracle as O

CASES = [("varcoef", 60.0, 258, 32, 256), ("varcoef", 60.0, 1026, 32, 256), ("diffconv2", 0.0, 258, 16, 120),
         ("random1", 0.0, 130, 16, 90), ("helmholtz", 40.0, 514, 16, 256), ("laplace", 0.0, 514, 16, 256)]


def spec(name, n, par):
    if name == "helmholtz":
        return dtn.ProblemSpec.continuum("helmholtz", n, None, None, lambda x, y: np.full_like(x, -par * par))
    if name == "varcoef":
        return dtn.baseline_problem(3, n - 2)
    return dtn.catalog(name, n, seed=1)


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


bases = [int(x) for x in os.environ.get("BASES", "16,32,48,64,96,128").split(",")]
for name, par, n, leaf, cross in CASES:
    op = dtn.discretize(spec(name, n, par))
    tree = dtn.build_tree_uniform(n, leaf)
    ref = O.build_root_dense(O.Problem(name, n, par, seed=1), O.Tree(n, uniform_side=leaf), threads=16, mode=2)
    dense = dtn.build_root_gpu(op, tree, want_G=False)
    Sd = dense.S_dense
    print(f"{name} n={n}: dense GPU vs oracle {rel(Sd, ref.S):.2e}", flush=True)
    dense.free()
    for b in bases:
        sol = dtn.build_root_gpu(op, tree, want_G=False,
                                 accel=dtn.AccelOptions(epsilon=1e-10, crossover=cross, rank_base=b, rank_step=8))
        bs = sol.build_stats
        S = sol.S_dense
        print(f"   base {b:4d}: attempts {bs['rank_attempts']} tail {bs['sketch_tail']:.2e} max_rank {bs['max_rank']:4d}"
              f"  vs oracle {rel(S, ref.S):.2e}  vs dense {rel(S, Sd):.2e}  build {bs['build_ms']:.1f} ms", flush=True)
        sol.free()
