"""Deferred boundary columns (engine.cu NodeDev::defer): the LU of a heavy merge
wave skips the boundary columns, which are formed afterwards as
Y = L^{-1} P M_ib by blocked forward substitution. Forced on every merge with
ni >= 256 (DTN_DEFER_MIN_WORK=1, read once per process: subprocesses), the
operator, G and the body map must equal the default schedule's (same
arithmetic in the same order; pivoting problems exercise the permutation)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import json, sys
sys.path.insert(0, sys.argv[1])
import numpy as np
import paper_1302_5995_b200 as dtn
cfg, n_int, out = int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
op = dtn.discretize(dtn.baseline_problem(cfg, n_int))
tree = dtn.build_tree_uniform(n_int + 2, 16)
ids = dtn.make_load_set(dtn.Lattice(n_int + 2), [(40, 50), (n_int // 2, n_int // 3), (n_int - 9, 12)])
sol = dtn.build_root_gpu(op, tree, load_ids=ids)
np.savez(out, S=sol.S_dense, G=sol.G_dense, F=sol.body_map)
'''


def _run(tmp_path, cfg, n_int, env):
    out = str(tmp_path / f"r_{cfg}_{env.get('DTN_DEFER_MIN_WORK', 'd')}.npz")
    r = subprocess.run([sys.executable, "-c", CHILD, ROOT, str(cfg), str(n_int), out],
                       env=dict(os.environ, **env), capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return np.load(out)


@pytest.mark.parametrize("cfg,n_int", [(2, 512), (3, 512)])
def test_deferred_columns_match_default(tmp_path, cfg, n_int):
    a = _run(tmp_path, cfg, n_int, {"DTN_DEFER_MIN_WORK": "1"})
    b = _run(tmp_path, cfg, n_int, {"DTN_DEFER_MIN_WORK": "0"})
    for k in ("S", "G", "F"):
        assert np.linalg.norm(a[k] - b[k]) <= 1e-12 * np.linalg.norm(b[k]), k
