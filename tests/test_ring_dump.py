"""SURVEY f-1 (Dirichlet-ring DtN adapter) and f-3 (dense dump/load format).

CPU: the oracle's T = (1/h)(I + P G D_b) against the one-sided derivative of a
direct sparse solve A u = -D g (grid.hpp:88-90), the ring geometry of the
product's adapter against the oracle's, and the dense_nd.cpp:227-251 file
format. GPU: the adapter computed from the resident G against the oracle."""
import os
import sys

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle.oracle as O  # noqa: E402
import paper_1302_5995_b200 as dtn  # noqa: E402


def _assemble(problem: O.Problem):
    """A (unknowns) and D (unknowns x ring) from the stencil (grid.cpp:128-166)."""
    n = problem.n
    s, m = n - 2, n - 1
    st = problem.stencil()

    def ring_id(x, y):
        if y == 0:
            return x
        if x == m:
            return m + y
        if y == m:
            return 2 * m + (m - x)
        return 3 * m + (m - y)

    ra, ca, va, rd, cd, vd = [], [], [], [], [], []
    for k in range(s * s):
        x, y = k % s + 1, k // s + 1
        ra.append(k); ca.append(k); va.append(st[0, k])
        for r, (dx, dy) in enumerate([(1, 0), (-1, 0), (0, 1), (0, -1)], start=1):
            qx, qy = x + dx, y + dy
            if 1 <= qx <= s and 1 <= qy <= s:
                ra.append(k); ca.append((qy - 1) * s + qx - 1); va.append(st[r, k])
            else:
                rd.append(k); cd.append(ring_id(qx, qy)); vd.append(st[r, k])
    A = sp.csc_matrix((va, (ra, ca)), shape=(s * s, s * s))
    D = sp.csc_matrix((vd, (rd, cd)), shape=(s * s, 4 * m))
    return A, D


@pytest.mark.parametrize("name,param,n", [("laplace", 0.0, 14), ("helmholtz", 7.0, 18), ("diffconv1", 0.0, 16)])
def test_oracle_ring_dtn_matches_direct_solve(name, param, n):
    pr = O.Problem(name, n, param) if param else O.Problem(name, n)
    res = O.build_root_dense(pr, O.Tree(n, 16))
    T = O.ring_dtn(pr, res)
    A, D = _assemble(pr)
    m, s, h = n - 1, n - 2, 1.0 / (n - 1)
    rng = np.random.default_rng(n)
    g_full = rng.uniform(-1, 1, 4 * m)
    g_full[::m] = 0.0  # corners (never coupled)
    u = spla.spsolve(A, -(D @ g_full))
    noncorner = np.array([r for r in range(4 * m) if r % m != 0])
    _, _, adj_uid, _ = dtn.ring_nodes(n)
    neumann = (g_full[noncorner] - u[adj_uid]) / h
    assert np.linalg.norm(T @ g_full[noncorner] - neumann) <= 1e-9 * np.linalg.norm(neumann)


def test_ring_nodes_geometry():
    n = 10
    ids, pos, adj, dirs = dtn.ring_nodes(n)
    s = n - 2
    assert len(ids) == 4 * s and len(set(adj.tolist())) == 4 * s - 4  # corner unknowns serve two ring nodes
    step = {1: (1, 0), 2: (-1, 0), 3: (0, 1), 4: (0, -1)}
    for (x, y), a, d in zip(pos, adj, dirs):
        ax, ay = a % s + 1, a // s + 1
        assert (ax + step[d][0], ay + step[d][1]) == (x, y)


def test_dump_load_schur_format(tmp_path):
    rng = np.random.default_rng(0)
    S = np.asfortranarray(rng.standard_normal((7, 5)))
    p = tmp_path / "s.bin"
    dtn.dump_schur(S, str(p))
    raw = p.read_bytes()
    assert len(raw) == 16 + 8 * 35
    assert np.frombuffer(raw[:16], dtype="<i8").tolist() == [7, 5]
    assert np.array_equal(np.frombuffer(raw[16:], dtype="<f8").reshape(7, 5), S)  # row-major payload
    assert np.array_equal(dtn.load_schur(str(p)), S)
    (tmp_path / "t.bin").write_bytes(raw[:-8])
    with pytest.raises(RuntimeError):
        dtn.load_schur(str(tmp_path / "t.bin"))


@pytest.mark.gpu
@pytest.mark.parametrize("name,cfg,n,leaf", [("laplace", 1, 66, 16), ("helmholtz", 2, 130, 16)])
def test_gpu_ring_dtn_vs_oracle(name, cfg, n, leaf):
    op = dtn.discretize(dtn.baseline_problem(cfg, n - 2))
    sol = dtn.build_root_gpu(op, dtn.build_tree_uniform(n, leaf))
    T = dtn.ring_dtn(sol, op)
    pr = O.Problem("laplace", n) if name == "laplace" else O.Problem("helmholtz", n, 40.0)
    ref = O.build_root_dense(pr, O.Tree(n, uniform_side=leaf), threads=8, mode=2)
    Tref = O.ring_dtn(pr, ref)
    # G parity is condition-limited for Helmholtz; T inherits it
    tol = 1e-10 if name == "laplace" else 1e-9
    assert np.linalg.norm(T - Tref) <= tol * np.linalg.norm(Tref)
    Td = dtn.ring_dtn(sol, op, device=True)
    assert np.array_equal(Td.cpu().numpy(), T)
