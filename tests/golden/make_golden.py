"""Generate the golden fixtures in tests/golden/ (run from the repo root).

The reference (a CMake/Eigen project) cannot be built in this image and ships
no golden data, so these fixtures are produced by the oracle
restatement (oracle/dense_oracle.cpp, pinned to the reference's own
known-answer tests in tests/test_oracle_*.py) and, for the body map, by a
sparse direct solve of the full system. They freeze small, exactly specified
cases so the product and any later oracle change are checked against the
same numbers."""
import os
import sys

import numpy as np
import scipy.sparse.linalg as spla

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def root_case(name, n, n_leaf, param=0.0, seed=0):
    pr = O.Problem(name, n, param, seed) if param or seed else O.Problem(name, n)
    res = O.build_root_dense(pr, O.Tree(n, n_leaf))
    return {"n": n, "n_leaf": n_leaf, "name": name, "param": param, "seed": seed,
            "stencil": pr.stencil(), "boundary": res.boundary, "S": res.S, "G": res.G}


def main():
    cases = {
        "laplace_n10": root_case("laplace", 10, 16),
        "helmholtz1_n18": root_case("helmholtz1", 18, 16),
        "random1_n16": root_case("random1", 16, 16, seed=5),
    }
    for key, c in cases.items():
        np.savez_compressed(os.path.join(OUT, key + ".npz"), **{k: np.asarray(v) for k, v in c.items()})
    # body map of test_dense_nd.cpp:175-193 (random1 n=16, load at (7, 6)): F = boundary rows of A^{-1} e_load
    c = cases["random1_n16"]
    A = O.sparse_system(c["stencil"], 16)
    s = 14
    load = (6 - 1) * s + (7 - 1)
    rhs = np.zeros(A.shape[0])
    rhs[load] = 1.0
    F = spla.spsolve(A.tocsc(), rhs)[c["boundary"]]
    np.savez_compressed(os.path.join(OUT, "random1_n16_load.npz"), load_ids=np.array([load]), F=F)


if __name__ == "__main__":
    main()
