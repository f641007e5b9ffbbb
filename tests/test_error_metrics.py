"""SURVEY f-4 / reference.cpp:80-177: e1/e2 error metrics (probe vectors of the
reference, exact answer from a sparse direct solve of the full system) and the
acceptance criteria that use them (acceptance.cpp:148-157 error reproduction,
:381-404 resonance behaviour) -- on the oracle (CPU) and on the GPU engine."""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle.oracle as O  # noqa: E402
import paper_1302_5995_b200 as dtn  # noqa: E402


def test_probe_vectors():
    r = O.random_unit_boundary(1021, 1)
    assert abs(np.linalg.norm(r) - 1.0) < 1e-14 and len(r) == 1021
    assert not np.array_equal(r, O.random_unit_boundary(1021, 2))
    s = O.smooth_boundary(64)
    assert abs(np.linalg.norm(s) - 1.0) < 1e-14 and abs(s[0]) == 0.0


def test_oracle_error_metrics_small():
    n = 66
    pr = O.Problem("laplace", n)
    res = O.build_root_dense(pr, O.Tree(n, 64))
    e1, e2 = O.error_metrics(lambda r: res.G @ r, pr.stencil(), n, res.boundary, 1)
    assert e1 <= 1e-10 and e2 <= 1e-10


@pytest.mark.gpu
def test_gpu_error_reproduction_criterion3():
    # acceptance criterion 3 (laplace n=256: e1, e2 <= 1e-5), dense GPU engine
    n = 256
    op = dtn.discretize(dtn.catalog("laplace", n))
    sol = dtn.build_root_gpu(op, dtn.build_tree(n, 1024))
    e1, e2 = O.error_metrics(lambda r: dtn.apply_dtn(sol, r), op.stencil, n, sol.boundary, 1)
    assert e1 <= 1e-5 and e2 <= 1e-5
    assert e1 <= 1e-10 and e2 <= 1e-10  # dense: no compression error at all


@pytest.mark.gpu
def test_gpu_resonance_criterion8():
    # acceptance criterion 8: near-resonant helmholtz3 builds, and its e2 is
    # at least 10x the Laplace e2 (condition-limited accuracy)
    n = 256
    tree = dtn.build_tree(n, 1024)
    errs = {}
    for name in ("helmholtz3", "laplace"):
        op = dtn.discretize(dtn.catalog(name, n))
        sol = dtn.build_root_gpu(op, tree)
        errs[name] = O.error_metrics(lambda r: dtn.apply_dtn(sol, r), op.stencil, n, sol.boundary, 1)[1]
    assert errs["helmholtz3"] >= 10.0 * errs["laplace"]
