"""Oracle pins against the reference's dense-engine tests
(proj/tests/test_dense_nd.cpp, proj/tests/acceptance.cpp:74-114)."""
import numpy as np
import pytest

from oracle import oracle as O


def test_leaf_without_interior_is_abb():  # test_dense_nd.cpp:62-70
    p = O.Problem("laplace", 8)
    A = p.dense_A()
    S = O.leaf_rect(p, 2, 3, 2, 5)
    b, i = O.rect_sets(8, 2, 3, 2, 5)
    assert len(i) == 0
    assert O.rel_fro(S, O.brute_schur(A, b, i)) <= 1e-14


def test_single_interior_node_by_hand():  # test_dense_nd.cpp:72-90
    p = O.Problem("uniform", 8)  # unit-spacing network, center coefficient 4
    A = p.dense_A()
    b, i = O.rect_sets(8, 2, 4, 2, 4)
    assert len(i) == 1 and A[i[0], i[0]] == 4.0
    a = A[np.ix_(b, i)][:, 0]
    expect = A[np.ix_(b, b)] - np.outer(a, a) / 4.0
    assert O.rel_fro(O.leaf_rect(p, 2, 4, 2, 4), expect) <= 1e-14


def test_leaf_vs_brute():  # test_dense_nd.cpp:92-100
    p = O.Problem("diffconv3", 16)
    A = p.dense_A()
    t = O.Tree(16, 64)
    for bid in t.levels[t.depth]:
        bx = t.boxes[bid]
        S = O.leaf_rect(p, bx["x0"], bx["x1"], bx["y0"], bx["y1"])
        assert O.rel_fro(S, O.brute_schur(A, bx["boundary"], bx["interior"])) <= 1e-12


def test_empty_interface_merge():  # test_dense_nd.cpp:102-110
    p = O.Problem("laplace", 8)
    A = p.dense_A()
    S = O.merge_rects(p, (2, 2, 2, 5), (3, 3, 2, 5))
    b, _ = O.rect_sets(8, 2, 3, 2, 5)
    assert O.rel_fro(S, O.brute_schur(A, b, [])) <= 1e-14


def test_merge_equals_union_leaf():  # test_dense_nd.cpp:112-121
    p = O.Problem("laplace", 8)
    S = O.merge_rects(p, (1, 3, 1, 6), (4, 6, 1, 6))
    assert O.rel_fro(S, O.leaf_rect(p, 1, 6, 1, 6)) <= 1e-12


@pytest.mark.parametrize("n", [8, 16, 24, 32])
@pytest.mark.parametrize("name", ["laplace", "diffconv1", "random1"])
def test_root_vs_brute(n, name):  # test_dense_nd.cpp:123-132
    p = O.Problem(name, n, seed=3)
    t = O.Tree(n, 16)
    r = O.build_root_dense(p, t)
    rb = t.root()
    assert np.array_equal(r.boundary, rb["boundary"])
    assert O.rel_fro(r.S, O.brute_schur(p.dense_A(), rb["boundary"], rb["interior"])) <= 1e-10


def test_symmetric_problem_symmetric_S():  # test_dense_nd.cpp:150-156
    p = O.Problem("random2", 16, seed=9)
    r = O.build_root_dense(p, O.Tree(16, 16))
    assert np.max(np.abs(r.S - r.S.T)) <= 1e-10 * np.linalg.norm(r.S)


def test_GS_is_identity():  # test_dense_nd.cpp:158-164
    r = O.build_root_dense(O.Problem("laplace", 16), O.Tree(16, 16))
    assert np.max(np.abs(r.G @ r.S - np.eye(len(r.S)))) <= 1e-10


def test_G_r_matches_full_solve():  # test_dense_nd.cpp:166-173
    n = 32
    p = O.Problem("laplace", n)
    t = O.Tree(n, 64)
    r = O.build_root_dense(p, t)
    rng = np.random.default_rng(17)
    g = rng.standard_normal(len(r.boundary))
    g /= np.linalg.norm(g)
    A = p.dense_A()
    rhs = np.zeros(A.shape[0])
    rhs[r.boundary] = g
    ref = np.linalg.solve(A, rhs)[r.boundary]
    assert np.linalg.norm(r.G @ g - ref) / np.linalg.norm(ref) <= 1e-10


def test_near_resonant_condition():  # test_dense_nd.cpp:195-201
    h3 = O.build_root_dense(O.Problem("helmholtz3", 32), O.Tree(32, 64))
    lap = O.build_root_dense(O.Problem("laplace", 32), O.Tree(32, 64))
    assert h3.cond > 100.0 * lap.cond


@pytest.mark.parametrize("n", [8, 16, 32])
def test_acceptance_criterion1(n):  # acceptance.cpp:74-114
    worst = 0.0
    for name in O.CATALOG:
        p = O.Problem(name, n, seed=1)
        t = O.Tree(n, 16)
        r = O.build_root_dense(p, t)
        rb = t.root()
        worst = max(worst, O.rel_fro(r.S, O.brute_schur(p.dense_A(), rb["boundary"], rb["interior"])))
    assert worst <= 1e-10


def test_threading_modes_agree():
    # reference-faithful (boxes over threads, 1 BLAS thread) vs all-core BLAS
    p = O.Problem("helmholtz1", 66)
    t = O.Tree(66, 64)
    a = O.build_root_dense(p, t, threads=4, mode=0)
    b = O.build_root_dense(p, t, threads=4, mode=1)
    assert O.rel_fro(a.S, b.S) <= 1e-13


def test_uniform_tree_root_matches_reference_tree():
    # the root S does not depend on the partition
    p = O.Problem("helmholtz", 66, param=10.0)
    a = O.build_root_dense(p, O.Tree(66, 289))
    b = O.build_root_dense(p, O.Tree(66, uniform_side=16))
    assert O.rel_fro(a.S, b.S) <= 1e-12


def test_keep_all_levels_vs_brute():
    p = O.Problem("diffconv1", 34)
    A = p.dense_A()
    t = O.Tree(34, uniform_side=8)
    r = O.build_root_dense(p, t, keep_all=True)
    for lev in range(t.depth + 1):
        for bid in t.levels[lev][:3]:
            bx = t.boxes[bid]
            assert O.rel_fro(r.box_S(bid), O.brute_schur(A, bx["boundary"], bx["interior"])) <= 1e-11
