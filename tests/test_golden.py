"""Golden fixtures (tests/golden/, generator make_golden.py): the oracle must
keep reproducing them (CPU) and the GPU engine must match them (GPU)."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
import paper_1302_5995_b200 as dtn  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")
CASES = ["laplace_n10", "helmholtz1_n18", "random1_n16"]


def _load(key):
    z = np.load(os.path.join(GOLD, key + ".npz"))
    return {k: z[k] for k in z.files}


def _rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("key", CASES)
def test_oracle_reproduces_golden(key):
    g = _load(key)
    name, n, n_leaf = str(g["name"]), int(g["n"]), int(g["n_leaf"])
    param, seed = float(g["param"]), int(g["seed"])
    pr = O.Problem(name, n, param, seed) if param or seed else O.Problem(name, n)
    assert np.array_equal(pr.stencil(), g["stencil"])
    res = O.build_root_dense(pr, O.Tree(n, n_leaf))
    assert np.array_equal(res.boundary, g["boundary"])
    assert _rel(res.S, g["S"]) <= 1e-13 and _rel(res.G, g["G"]) <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("key", CASES)
def test_gpu_matches_golden(key):
    g = _load(key)
    name, n, n_leaf, seed = str(g["name"]), int(g["n"]), int(g["n_leaf"]), int(g["seed"])
    op = dtn.discretize(dtn.catalog(name, n, seed))
    assert np.array_equal(op.stencil, g["stencil"])
    sol = dtn.build_root_gpu(op, dtn.build_tree(n, n_leaf))
    assert np.array_equal(sol.boundary, g["boundary"])
    assert _rel(sol.S_dense, g["S"]) <= 1e-10 and _rel(sol.G_dense, g["G"]) <= 1e-10


@pytest.mark.gpu
def test_gpu_body_map_matches_golden():
    g = _load("random1_n16")
    gl = _load("random1_n16_load")
    op = dtn.discretize(dtn.catalog("random1", 16, 5))
    sol = dtn.build_root_gpu(op, dtn.build_tree(16, 16), load_ids=gl["load_ids"])
    assert _rel(sol.body_map[:, 0], gl["F"]) <= 1e-10
    assert np.array_equal(sol.boundary, g["boundary"])
