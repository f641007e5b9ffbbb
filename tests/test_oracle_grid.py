"""Oracle pins against the reference's grid tests (proj/tests/test_grid.cpp)."""
import numpy as np
import pytest

from oracle import oracle as O


def test_five_point_stencil_n5():  # test_grid.cpp:12-26
    p = O.Problem("laplace", 5)
    s = 3
    uid = lambda x, y: (y - 1) * s + (x - 1)
    k = uid(2, 2)
    assert p.coeff(k, k) == pytest.approx(64.0)
    for q in [uid(3, 2), uid(1, 2), uid(2, 3), uid(2, 1)]:
        assert p.coeff(k, q) == pytest.approx(-16.0)


def test_boundary_row_sums_vanish():  # test_grid.cpp:28-39
    p = O.Problem("laplace", 5)
    st = p.stencil()
    k = 0  # (1,1): two ring neighbours (west, south) go to the forcing map
    assert st[:, k].sum() == pytest.approx(0.0, abs=1e-12)


def test_unit_spacing_scaling():  # test_grid.cpp:41-53
    n = 8
    p = O.Problem("laplace", n)
    h = 1.0 / (n - 1)
    s = n - 2
    uid = lambda x, y: (y - 1) * s + (x - 1)
    k = uid(3, 3)
    assert p.coeff(k, k) * h * h == pytest.approx(4.0)
    assert p.coeff(k, uid(4, 3)) * h * h == pytest.approx(-1.0)
    assert p.coeff(k, uid(3, 2)) * h * h == pytest.approx(-1.0)
    assert p.coeff(k, uid(4, 4)) == 0.0


def test_network_seed_and_range():  # test_grid.cpp:55-82
    a = O.Problem("random1", 17, seed=42).stencil()
    b = O.Problem("random1", 17, seed=42).stencil()
    c = O.Problem("random1", 17, seed=43).stencil()
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    assert np.all(-a[1:] >= 1.0) and np.all(-a[1:] < 2.0)


def test_symmetry_when_no_convection():  # test_grid.cpp:84-91
    for name in ["laplace", "helmholtz1", "random2"]:
        A = O.Problem(name, 12, seed=3).dense_A()
        assert np.max(np.abs(A - A.T)) == 0.0


def test_discretize_rejects_small_n():  # test_grid.cpp:93-98
    with pytest.raises(O.OracleError) as e:
        O.Problem("laplace", 3)
    assert e.value.code == 2


def test_tree_depth_rule():  # test_grid.cpp:100-104
    assert O.Tree(16, 64).depth == 1
    assert O.Tree(64, 4096).depth == 0
    assert O.Tree(128, 4096).depth == 1


def test_four_leaves_of_64():  # test_grid.cpp:106-116
    t = O.Tree(16, 64)
    assert len(t.levels[1]) == 4
    tot = 0
    for bid in t.levels[1]:
        b = t.boxes[bid]
        assert (b["gx1"] - b["gx0"]) * (b["gy1"] - b["gy0"]) == 64
        tot += len(b["boundary"]) + len(b["interior"])
    assert tot == 14 * 14


@pytest.mark.parametrize("n", [8, 11, 16, 21])
def test_partition_and_nesting(n):  # test_grid.cpp:118-153
    t = O.Tree(n, 16)
    s = n - 2
    for b in t.boxes:
        p = set(b["boundary"].tolist())
        assert len(p) == len(b["boundary"])
        for i in b["interior"].tolist():
            assert i not in p
            p.add(i)
        for i in b["interior"].tolist():
            x, y = i % s + 1, i // s + 1
            for qx, qy in [(x + 1, y), (x - 1, y), (x, y + 1), (x, y - 1)]:
                assert 1 <= qx <= n - 2 and 1 <= qy <= n - 2
                assert (qy - 1) * s + qx - 1 in p
        if b["children"][0] >= 0:
            kids = set()
            for c in b["children"]:
                kids |= set(t.boxes[c]["boundary"].tolist()) | set(t.boxes[c]["interior"].tolist())
            assert kids == p
    for level in t.levels:
        assert sum(len(t.boxes[i]["boundary"]) + len(t.boxes[i]["interior"]) for i in level) == s * s


def test_ccw_order():  # test_grid.cpp:155-172
    t = O.Tree(16, 64)
    s = 14
    pt = lambda i: (i % s + 1, i // s + 1)
    for b in t.boxes:
        bd = b["boundary"].tolist()
        assert pt(bd[0]) == (b["x0"], b["y0"])
        for i in range(len(bd)):
            p, q = pt(bd[i]), pt(bd[(i + 1) % len(bd)])
            assert abs(p[0] - q[0]) + abs(p[1] - q[1]) == 1
        if b["x1"] > b["x0"]:
            assert pt(bd[1])[0] == b["x0"] + 1


def test_tree_rejects_bad_params():  # test_grid.cpp:174-177
    for args in [(3, 64), (16, 8)]:
        with pytest.raises(O.OracleError):
            O.Tree(*args)


def test_reference_partition_at_baseline_size():
    # n_int=256 (ref n=258) with nleaf=289 -> depth 4, leaves 15/16/17 wide
    t = O.Tree(258, 289)
    assert t.depth == 4
    widths = {t.boxes[i]["x1"] - t.boxes[i]["x0"] + 1 for i in t.levels[4]}
    assert widths == {15, 16, 17}


def test_uniform_tree():
    t = O.Tree(66, uniform_side=16)
    assert t.depth == 2
    for i in t.levels[2]:
        b = t.boxes[i]
        assert b["x1"] - b["x0"] + 1 == 16 and b["y1"] - b["y0"] + 1 == 16
