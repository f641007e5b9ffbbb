"""SURVEY f-2: body loads carried through the merges as extra right-hand-side
columns (dense_nd.cpp:98-101, 136-147, 182-184), body map F = G rhs_root
(accel_nd.cpp:872-875), solve_with_load (bodyload.cpp:68-77). The reference's
own tests (test_dense_nd.cpp:175-193, test_bodyload.cpp:73-115) restated on the
GPU engine, with the exact answer from a sparse direct solve of the full system."""
import os
import sys

import numpy as np
import pytest
import scipy.sparse.linalg as spla

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle.oracle as O  # noqa: E402
import paper_1302_5995_b200 as dtn  # noqa: E402


def _reference_with_load(op, boundary, g, load_ids, fhat):
    """reference_with_load: x = A^{-1}(boundary forcing g + loads fhat), x on the boundary."""
    A = O.sparse_system(op.stencil, op.n)
    rhs = np.zeros(A.shape[0])
    rhs[boundary] += g
    rhs[load_ids] += fhat
    return spla.spsolve(A.tocsc(), rhs)[boundary]


def test_make_load_set_validation():
    lat = dtn.Lattice(32)
    ids = dtn.make_load_set(lat, [(16, 16), (3, 4)])
    assert ids.tolist() == [lat.unknown_id(16, 16), lat.unknown_id(3, 4)]
    with pytest.raises(ValueError):
        dtn.make_load_set(lat, [(1, 5)])  # on the root boundary ring of unknowns
    with pytest.raises(ValueError):
        dtn.make_load_set(lat, [(5, 5), (5, 5)])


@pytest.mark.gpu
def test_point_load_propagates_to_root_rhs():
    # test_dense_nd.cpp:175-193 (random1 network problem, n=16, n_leaf=16)
    op = dtn.discretize(dtn.catalog("random1", 16, 5))
    lat = dtn.Lattice(16)
    ids = [lat.unknown_id(7, 6)]
    sol = dtn.build_root_gpu(op, dtn.build_tree(16, 16), load_ids=ids)
    assert sol.body_map.shape == (sol.boundary_size(), 1)
    ref = _reference_with_load(op, sol.boundary, np.zeros(sol.boundary_size()), ids, np.ones(1))
    assert np.linalg.norm(sol.body_map[:, 0] - ref) <= 1e-10 * np.linalg.norm(ref)


@pytest.mark.gpu
def test_unit_center_load():
    # test_bodyload.cpp:73-95 (laplace n=32, n_leaf=64, dense bound 1e-8)
    n = 32
    op = dtn.discretize(dtn.catalog("laplace", n))
    ids = dtn.make_load_set(dtn.Lattice(n), [(n // 2, n // 2)])
    sol = dtn.build_with_loads(op, dtn.build_tree(n, 64), ids, dtn.Engine.gpu)
    v = dtn.solve_with_load(sol, np.zeros(sol.boundary_size()), np.ones(1))
    ref = _reference_with_load(op, sol.boundary, np.zeros(sol.boundary_size()), ids, np.ones(1))
    assert np.linalg.norm(v - ref) <= 1e-8 * np.linalg.norm(ref)


@pytest.mark.gpu
def test_clustered_loads_network():
    # test_bodyload.cpp:97-115 (random1 n=64, 10 clustered loads; compressed bound 1e-5, dense exact)
    n = 64
    op = dtn.discretize(dtn.catalog("random1", n, 11))
    pts = [(n // 2 + k % 4, n // 2 + k // 4) for k in range(10)]
    ids = dtn.make_load_set(dtn.Lattice(n), pts)
    sol = dtn.build_with_loads(op, dtn.build_tree(n, 256), ids, dtn.Engine.gpu)
    g = O.random_unit_boundary(sol.boundary_size(), 2)
    fhat = O.random_unit_boundary(len(ids), 3)
    v = dtn.solve_with_load(sol, g, fhat)
    ref = _reference_with_load(op, sol.boundary, g, ids, fhat)
    assert np.linalg.norm(v - ref) <= 1e-10 * np.linalg.norm(ref)


@pytest.mark.gpu
@pytest.mark.parametrize("nloads", [1, 7, 40])
def test_loads_through_blocked_merges(nloads):
    # the config-2 operator at n=130 (blocked merges and the root LU), loads
    # scattered over the domain, and a build without loads right after
    n = 130
    op = dtn.discretize(dtn.baseline_problem(2, n - 2))
    tree = dtn.build_tree_uniform(n, 16)
    rng = np.random.default_rng(nloads)
    pts = set()
    while len(pts) < nloads:
        pts.add((int(rng.integers(2, n - 3)), int(rng.integers(2, n - 3))))
    ids = dtn.make_load_set(dtn.Lattice(n), sorted(pts))
    sol = dtn.build_root_gpu(op, tree, load_ids=ids)
    g = rng.uniform(-1, 1, sol.boundary_size())
    fhat = rng.uniform(-1, 1, nloads)
    v = dtn.solve_with_load(sol, g, fhat)
    ref = _reference_with_load(op, sol.boundary, g, ids, fhat)
    assert np.linalg.norm(v - ref) <= 1e-9 * np.linalg.norm(ref)  # condition-limited (Helmholtz)
    plain = dtn.build_root_gpu(op, tree)
    assert np.linalg.norm(plain.S_dense - sol.S_dense) <= 1e-13 * np.linalg.norm(plain.S_dense)


@pytest.mark.gpu
def test_load_errors():
    n = 32
    op = dtn.discretize(dtn.catalog("laplace", n))
    lat = dtn.Lattice(n)
    tree = dtn.build_tree(n, 64)
    with pytest.raises(ValueError):
        dtn.build_root_gpu(op, tree, load_ids=[lat.unknown_id(1, 5)])
    with pytest.raises(ValueError):
        dtn.build_root_gpu(op, tree, load_ids=[lat.unknown_id(5, 5)] * 2)
    with pytest.raises(ValueError):
        dtn.build_root_gpu(op, tree, want_G=False, load_ids=[lat.unknown_id(5, 5)])


@pytest.mark.gpu
@pytest.mark.parametrize("crossover", [128, 1024])
def test_clustered_loads_network_accel(crossover):
    # test_bodyload.cpp:97-115 with Engine::accel (compressed bound 1e-5): crossover 128
    # compresses the root (body map = G_hbs rhs_root), 1024 keeps it dense (accel_nd.cpp:796-818)
    n = 64
    op = dtn.discretize(dtn.catalog("random1", n, 11))
    pts = [(n // 2 + k % 4, n // 2 + k // 4) for k in range(10)]
    ids = dtn.make_load_set(dtn.Lattice(n), pts)
    sol = dtn.build_with_loads(op, dtn.build_tree(n, 256), ids, dtn.Engine.accel,
                               dtn.AccelOptions(epsilon=1e-10, crossover=crossover, hbs_leaf=32))
    assert (getattr(sol, "G_hbs", None) is not None) == (crossover == 128)
    g = O.random_unit_boundary(sol.boundary_size(), 2)
    fhat = O.random_unit_boundary(len(ids), 3)
    v = dtn.solve_with_load(sol, g, fhat)
    ref = _reference_with_load(op, sol.boundary, g, ids, fhat)
    assert np.linalg.norm(v - ref) <= 1e-8 * np.linalg.norm(ref)
    assert sol.memory_bytes() > 8 * sol.body_map.size


@pytest.mark.gpu
def test_loads_accel_matches_dense_engine():
    n = 130
    op = dtn.discretize(dtn.baseline_problem(2, n - 2))
    tree = dtn.build_tree_uniform(n, 16)
    rng = np.random.default_rng(5)
    ids = dtn.make_load_set(dtn.Lattice(n), [(20, 30), (64, 64), (100, 40), (33, 99)])
    acc = dtn.build_with_loads(op, tree, ids, dtn.Engine.accel, dtn.AccelOptions(epsilon=1e-10, crossover=256))
    dense = dtn.build_with_loads(op, tree, ids, dtn.Engine.gpu)
    assert acc.G_hbs is not None
    assert np.linalg.norm(acc.body_map - dense.body_map) <= 1e-9 * dense.cond_estimate * np.linalg.norm(dense.body_map)
    g = rng.uniform(-1, 1, dense.boundary_size())
    fhat = rng.uniform(-1, 1, len(ids))
    ref = _reference_with_load(op, dense.boundary, g, ids, fhat)
    v = dtn.solve_with_load(acc, g, fhat)
    assert np.linalg.norm(v - ref) <= 1e-7 * np.linalg.norm(ref)
