"""GPU HBS compression / apply / DTNHBS01 (csrc/hbs.cu, csrc/k_hbs.cu through
the C ABI) against the oracle restatement of hbs.cpp and the reference's own
HBS test properties (proj/tests/test_hbs.cpp)."""
import numpy as np
import pytest

from oracle import hbs_oracle as HO
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def rel_fro(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.fixture(scope="module")
def H():
    from paper_1302_5995_b200 import hbs
    return hbs


def test_identity_rank_zero(H):  # test_hbs.cpp:88-100
    c = H.compress(np.eye(96), 1e-10, 16)
    assert c.max_rank() == 0
    for t in range(c.tree.num_nodes()):
        if c.tree.is_leaf(t):
            assert np.abs(c.factor(t, "D") - np.eye(c.tree.node_size(t))).max() == 0.0
    assert rel_fro(H.reconstruct(c), np.eye(96)) <= 1e-14


def test_rank_one(H):  # test_hbs.cpp:102-108
    rng = np.random.default_rng(1)
    A = rng.standard_normal((80, 1)) @ rng.standard_normal((1, 80))
    c = H.compress(A, 1e-10, 16)
    assert c.max_rank() <= 1
    assert rel_fro(H.reconstruct(c), A) <= 1e-12


def test_laplace_root_schur(H):  # test_hbs.cpp:110-116
    S = O.build_root_dense(O.Problem("laplace", 64), O.Tree(64, 4096)).S
    c = H.compress(S, 1e-7, 64)
    assert rel_fro(H.reconstruct(c), S) <= 1e-6
    assert c.max_rank() < S.shape[0] / 4
    assert H.basis_orthonormality_defect(c) <= 1e-12


def test_apply_matches_dense(H):  # test_hbs.cpp:118-125
    A = HO.kernel_matrix(150, 3)
    c = H.compress(A, 1e-9, 32)
    x = np.random.default_rng(4).standard_normal((150, 3))
    assert rel_fro(H.apply(c, x), A @ x) <= 1e-8
    assert np.linalg.norm(H.apply(c, np.zeros((150, 2)))) == 0.0
    with pytest.raises(ValueError):
        H.apply(c, np.zeros((10, 1)))


@pytest.mark.parametrize("eps", [1e-4, 1e-7, 1e-10])
@pytest.mark.parametrize("seed", [11, 12, 13])
def test_roundtrip_budget(H, eps, seed):  # test_hbs.cpp:127-136
    A = HO.kernel_matrix(130, seed)
    c = H.compress(A, eps, 16)
    assert rel_fro(H.reconstruct(c), A) <= 10.0 * eps * (c.tree.depth + 1)
    assert H.basis_orthonormality_defect(c) <= 1e-12


def test_ranks_monotone_and_match_oracle(H):  # test_hbs.cpp:138-146
    A = HO.kernel_matrix(128, 5)
    loose, tight = H.compress(A, 1e-4, 16), H.compress(A, 1e-9, 16)
    assert all(loose.rank(t) <= tight.rank(t) for t in range(1, loose.tree.num_nodes()))
    ref = HO.compress(A, 1e-9, 16)
    for t in range(1, ref.tree.num_nodes()):
        if ref.tree.is_leaf(t):
            assert tight.rank(t) == ref.rank(t), t  # identical block rows: identical eps-ranks
        else:
            assert abs(tight.rank(t) - ref.rank(t)) <= 2, t


def test_serialization(H, tmp_path):  # test_hbs.cpp:177-196
    A = HO.kernel_matrix(90, 9)
    c = H.compress(A, 1e-8, 16)
    b1, b2 = H.serialize(c), H.serialize(H.compress(A, 1e-8, 16))
    assert b1 == b2  # byte-for-byte stable for a fixed input
    ho = HO.deserialize(b1)  # the reference layout, read by the oracle
    assert rel_fro(HO.reconstruct(ho), H.reconstruct(c)) <= 1e-14
    back = H.deserialize(b1)
    assert back.tree == c.tree
    assert rel_fro(H.reconstruct(back), H.reconstruct(c)) == 0.0
    p = str(tmp_path / "hbs_io.tmp")
    H.write_hbs(c, p)
    assert H.serialize(H.read_hbs(p)) == b1
    # an oracle-made operator uploads and applies like the oracle
    oc = HO.compress(A, 1e-8, 16)
    g = H.deserialize(HO.serialize(oc))
    x = np.random.default_rng(2).standard_normal((90, 4))
    assert rel_fro(H.apply(g, x), HO.apply(oc, x)) <= 1e-13
    with pytest.raises(ValueError):
        H.deserialize(bytes([1, 2, 3]))


def test_single_node(H):
    A = HO.kernel_matrix(40, 1)
    c = H.compress(A, 1e-10, 64)
    assert c.tree.num_nodes() == 1
    x = np.random.default_rng(0).standard_normal(40)
    assert rel_fro(H.apply(c, x), A @ x) <= 1e-14


@pytest.mark.parametrize("name,param", [("laplace", 0.0), ("helmholtz", 40.0)])
def test_root_operators_within_10eps(H, name, param):
    """The compressed root operators (S_hbs, G_hbs of build_root_accel's
    result) against the dense oracle: within 10 eps relative Frobenius at
    eps = 1e-10, on the reference-size boundary M = 1020."""
    import paper_1302_5995_b200 as dtn
    n = 258
    ref = O.build_root_dense(O.Problem(name, n, param), O.Tree(n, uniform_side=16))
    spec = dtn.catalog(name, n) if param == 0.0 else dtn.ProblemSpec.continuum(
        "h", n, None, None, lambda x, y: np.full_like(x, -param * param))
    sol = dtn.build_root_gpu(dtn.discretize(spec), dtn.build_tree_uniform(n, 16))
    eps = 1e-10
    for which, dense in (("S", ref.S), ("G", ref.G)):
        c = H.compress_operator(sol, which, eps, 64)
        assert rel_fro(H.reconstruct(c), dense) <= 10 * eps, which
        g = np.random.default_rng(1).uniform(-1, 1, (dense.shape[0], 16))
        assert rel_fro(H.apply(c, g), dense @ g) <= 10 * eps, which
        assert c.max_rank() < dense.shape[0] / 4
        # leaf ranks as the oracle's compress of the same operator
        oc = HO.compress(dense, eps, 64)
        for t in range(1, oc.tree.num_nodes()):
            if oc.tree.is_leaf(t):
                assert abs(c.rank(t) - oc.rank(t)) <= 1, (which, t)


def test_torch_device_apply(H):
    import torch
    A = HO.kernel_matrix(200, 7)
    c = H.compress(torch.tensor(A, device="cuda"), 1e-10, 32)
    x = torch.randn(200, 5, dtype=torch.float64, device="cuda")
    y = H.apply(c, x)
    assert y.is_cuda
    assert rel_fro(y.cpu().numpy(), A @ x.cpu().numpy()) <= 1e-9


# ---- invert_hbs on the device (hbs_ops.cpp:148-205), test_hbs_ops.cpp:164-216 ----

def test_invert_diagonal(H):  # test_hbs_ops.cpp:164-172
    d = 1.0 + (np.arange(64) % 7)
    inv = H.invert_hbs(H.compress(np.diag(d), 1e-12, 16))
    x = np.linspace(-1.0, 2.0, 64)
    assert np.linalg.norm(H.apply_inverse(inv, x) - x / d) <= 1e-12


def test_invert_two_level_synthetic_matches_oracle(H):  # test_hbs_ops.cpp:174-180
    h = HO.synthetic_hbs(16, 4, 2, 6)
    g = H.deserialize(HO.serialize(h))
    inv = H.invert_hbs(g)
    dense = HO.reconstruct(h)
    G = H.apply_inverse(inv, np.eye(16))
    assert rel_fro(G, np.linalg.inv(dense)) <= 1e-9
    # factor by factor against the oracle's inversion of the same matrix
    ref = HO.invert_hbs(h)
    for t in range(1, h.tree.num_nodes()):
        assert rel_fro(inv.E(t), ref.U[t]) <= 1e-12, t
        assert rel_fro(inv.F(t), ref.V[t]) <= 1e-12, t
        assert rel_fro(inv.G(t), ref.D[t] if h.tree.is_leaf(t) else ref.B[t]) <= 1e-12, t
    assert rel_fro(inv.factor(0, "B"), ref.B[0]) <= 1e-12


@pytest.mark.parametrize("m,leaf,k,seed", [(200, 16, 5, 1), (1000, 64, 12, 2), (777, 40, 30, 3)])
def test_invert_synthetic_sizes(H, m, leaf, k, seed):
    h = HO.synthetic_hbs(m, leaf, k, seed)
    inv = H.invert_hbs(H.deserialize(HO.serialize(h)))
    x = np.random.default_rng(seed).standard_normal((m, 3))
    ref = HO.apply(HO.invert_hbs(h), x)
    assert rel_fro(H.apply_inverse(inv, x), ref) <= 1e-10
    assert rel_fro(HO.apply(h, H.apply_inverse(inv, x)), x) <= 1e-10


def test_invert_laplace_schur_residual(H):  # test_hbs_ops.cpp:182-190
    S = O.build_root_dense(O.Problem("laplace", 64), O.Tree(64, 4096)).S
    c = H.compress(S, 1e-7, 64)
    x = np.random.default_rng(7).standard_normal((S.shape[0], 2))
    back = H.apply(c, H.apply_inverse(H.invert_hbs(c), x))
    assert np.linalg.norm(back - x) / np.linalg.norm(x) <= 1e-5


@pytest.mark.parametrize("n", [32, 64])
def test_invert_residual_100eps(H, n):  # test_hbs_ops.cpp:192-203
    eps = 1e-7
    S = O.build_root_dense(O.Problem("laplace", n), O.Tree(n, 4096)).S
    c = H.compress(S, eps, 32)
    x = np.random.default_rng(8).standard_normal((S.shape[0], 1))
    back = H.apply(c, H.apply_inverse(H.invert_hbs(c), x))
    assert np.linalg.norm(back - x) / np.linalg.norm(x) <= 100 * eps


def test_invert_names_failing_node(H):  # test_hbs_ops.cpp:205-216
    import paper_1302_5995_b200 as dtn
    h = HO.synthetic_hbs(16, 4, 2, 9)
    for t in range(h.tree.num_nodes()):
        if h.tree.is_leaf(t):
            h.D[t][:] = 0.0
            break
    with pytest.raises(dtn.FactorizationError, match=r"Dtilde is singular \[node \d+ level \d+\]"):
        H.invert_hbs(H.deserialize(HO.serialize(h)))


def test_invert_single_node(H):
    A = HO.kernel_matrix(40, 1)
    inv = H.invert_hbs(H.compress(A, 1e-10, 64))
    assert rel_fro(H.apply_inverse(inv, np.eye(40)), np.linalg.inv(A)) <= 1e-13


def test_invert_serializes(H):
    """memory_bytes of the compressed engine serializes G_hbs.rep (solution_operator.cpp:9-11)."""
    A = HO.kernel_matrix(300, 4)
    inv = H.invert_hbs(H.compress(A, 1e-10, 32))
    back = H.deserialize(H.serialize(inv))
    x = np.random.default_rng(3).standard_normal((300, 2))
    assert rel_fro(H.apply(back, x), np.linalg.solve(A, x)) <= 1e-9


# ---- the compressed engine (build_root_accel, accel_nd.cpp:707-859) ----

@pytest.mark.parametrize("name,param", [("laplace", 0.0), ("helmholtz", 40.0)])
def test_build_root_accel_vs_dense_oracle(H, name, param):
    """S_hbs and G_hbs of the compressed engine against the dense oracle at
    eps = 1e-10 (M = 1020): S and the Neumann data S g within 10 eps; G g
    within 10 eps x cond(S) (G_hbs is the exact inverse of S_hbs, so its
    error is S_hbs's relative error amplified by the conditioning); residual
    S (G_hbs g) = g."""
    import paper_1302_5995_b200 as dtn
    n = 258
    ref = O.build_root_dense(O.Problem(name, n, param), O.Tree(n, uniform_side=16))
    spec = dtn.catalog(name, n) if param == 0.0 else dtn.ProblemSpec.continuum(
        "h", n, None, None, lambda x, y: np.full_like(x, -param * param))
    eps = 1e-10
    sol = dtn.build_root_accel(dtn.discretize(spec), dtn.build_tree_uniform(n, 16),
                               dtn.AccelOptions(epsilon=eps, crossover=256, hbs_leaf=64))
    assert sol.engine == dtn.Engine.accel and sol.G_hbs is not None
    assert np.array_equal(sol.boundary, ref.boundary)
    g = np.random.default_rng(1).uniform(-1, 1, (len(ref.boundary), 16))
    assert rel_fro(dtn.apply_schur(sol, g), ref.S @ g) <= 10 * eps
    assert rel_fro(H.reconstruct(sol.S_hbs), ref.S) <= 10 * eps
    cond = np.linalg.cond(ref.S, 1)
    assert rel_fro(dtn.apply_dtn(sol, g), ref.G @ g) <= 10 * eps * cond
    assert rel_fro(ref.S @ dtn.apply_dtn(sol, g), g) <= 10 * eps * cond
    # the reference's probe estimate (accel_nd.cpp:834-841) evaluated on the oracle's S and G
    m = len(ref.boundary)
    one = np.ones(m)
    est = (np.abs(ref.S @ one).sum() / m) * (np.abs(ref.G @ one).sum() / m) * m
    assert abs(sol.cond_estimate - est) <= 1e-6 * est
    assert sol.memory_bytes() < 2 * 8 * len(ref.boundary) ** 2


def test_build_root_accel_below_crossover_is_dense(H):  # accel_nd.cpp:796-818
    import paper_1302_5995_b200 as dtn
    n = 66
    ref = O.build_root_dense(O.Problem("laplace", n), O.Tree(n, uniform_side=16))
    sol = dtn.build_root_accel(dtn.discretize(dtn.catalog("laplace", n)), dtn.build_tree_uniform(n, 16),
                               dtn.AccelOptions(epsilon=1e-10, crossover=1024))
    assert sol.engine == dtn.Engine.accel and getattr(sol, "G_hbs", None) is None
    assert rel_fro(sol.G_dense, ref.G) <= 1e-10
    assert rel_fro(dtn.densify_dtn(sol), ref.G) <= 1e-10


def test_build_with_loads_accel_dispatch(H):  # bodyload.cpp:47-57
    import paper_1302_5995_b200 as dtn
    n = 130
    op = dtn.discretize(dtn.catalog("laplace", n))
    tree = dtn.build_tree_uniform(n, 16)
    sol = dtn.build_with_loads(op, tree, None, dtn.Engine.accel, dtn.AccelOptions(epsilon=1e-10, crossover=256))
    dense = dtn.build_root_gpu(op, tree)
    g = np.random.default_rng(5).uniform(-1, 1, len(dense.boundary))
    assert rel_fro(dtn.apply_schur(sol, g), dtn.apply_schur(dense, g)) <= 1e-9
    G = dtn.densify_dtn(sol)
    assert rel_fro(G, dense.G_dense) <= 1e-9 * dense.cond_estimate


def test_torch_column_major_batch(H):
    """Column-major (Fortran-order) device batches are applied in place."""
    import torch
    A = HO.kernel_matrix(120, 2)
    c = H.compress(A, 1e-10, 32)
    Xh = np.asfortranarray(np.random.default_rng(1).standard_normal((120, 7)))
    X = torch.from_numpy(Xh).cuda().t().contiguous().t()
    assert X.stride(0) == 1
    y = H.apply(c, X).cpu().numpy()
    assert rel_fro(y, A @ Xh) <= 1e-9
    y2 = H.apply(c, torch.from_numpy(np.ascontiguousarray(Xh)).cuda()).cpu().numpy()
    assert rel_fro(y2, A @ Xh) <= 1e-9


@pytest.mark.parametrize("cfg,n_int,leaf", [(3, 1024, 32), (5, 2048, 32)])
def test_baseline_compressed_configs_full_size(H, cfg, n_int, leaf):
    """BASELINE configs 3 and 5 at full size through the compressed engine:
    S_hbs (and the Neumann data S g) within 10 eps = 1e-9 of the dense GPU
    operator of the same build (the dense engine is itself pinned to the
    oracle, tests/test_gpu_parity.py), and G_hbs the inverse of S_hbs
    (residual of S G_hbs g at the conditioning level)."""
    import torch
    import paper_1302_5995_b200 as dtn
    op = dtn.discretize(dtn.baseline_problem(cfg, n_int))
    tree = dtn.build_tree_uniform(n_int + 2, leaf)
    eps = 1e-10
    sol = dtn.build_root_accel(op, tree, dtn.AccelOptions(epsilon=eps, crossover=256, hbs_leaf=64), keep_dense=True)
    nb = sol.boundary_size()
    g = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, (nb, 16))).cuda()
    Sg = dtn.apply_schur(sol.dense_op, g)
    rel = lambda a, b: float(torch.linalg.norm(a - b) / torch.linalg.norm(b))
    assert rel(dtn.apply_schur(sol, g), Sg) <= 10 * eps
    # the whole operator: S_hbs applied to the identity against the dense S
    E = torch.eye(nb, dtype=torch.float64, device="cuda")
    S_rec = dtn.apply_schur(sol, E)
    S_dense = dtn.apply_schur(sol.dense_op, E)
    assert rel(S_rec, S_dense) <= 10 * eps
    res = rel(dtn.apply_dtn(sol, Sg), g)
    assert res <= 10 * eps * sol.cond_estimate, (res, sol.cond_estimate)
    assert sol.S_hbs.max_rank() < nb / 8
    sol.dense_op.free()


def test_repeated_compressed_builds_keep_memory_flat(H):
    """Plans are cached per context, the compression scratch and the caching pool are
    reused and the factors are freed with their operators: device memory in use is
    flat over repeated build_root_accel + apply rounds."""
    import torch
    import paper_1302_5995_b200 as dtn
    op = dtn.discretize(dtn.baseline_problem(3, 1024))
    tree = dtn.build_tree_uniform(1026, 32)
    marks = []
    for _ in range(4):
        acc = dtn.build_root_accel(op, tree, dtn.AccelOptions(epsilon=1e-10, crossover=256))
        X = torch.randn(acc.boundary_size(), 64, dtype=torch.float64, device="cuda")
        dtn.apply_dtn(acc, X)
        del acc, X
        torch.cuda.synchronize()
        free, total = torch.cuda.mem_get_info()
        marks.append(total - free)
    assert marks[-1] <= marks[1] + (64 << 20), marks


@pytest.mark.parametrize("crossover,compressed", [(188, True), (189, False), (252, False)])
def test_crossover_gate_is_size_at_least(H, crossover, compressed):
    """The reference compresses a merged box whose boundary size is >= crossover
    only when it has a next merge (merge_pair, accel_nd.cpp:667-689); the root's
    W|E merge has none (:771-779), so the root is structured exactly when both
    halves are. n_int = 64 with 16 x 16 leaves: the W / E halves are 32 x 64 boxes
    with boundary 2 (32 + 64) - 4 = 188; the root boundary 252 does not matter."""
    import paper_1302_5995_b200 as dtn
    n = 66
    sol = dtn.build_root_accel(dtn.discretize(dtn.catalog("laplace", n)), dtn.build_tree_uniform(n, 16),
                               dtn.AccelOptions(epsilon=1e-10, crossover=crossover, hbs_leaf=32))
    assert (getattr(sol, "G_hbs", None) is not None) == compressed
    assert sol.boundary_size() == 252
