"""GPU accuracy of G g on the n=1024 config-3 operator (the parity test's check), per env toggle."""
import os, sys, subprocess, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

def run(micro):
    import scipy.sparse as sp
    import scipy.sparse.linalg as spla
    import paper_1302_5995_b200 as dtn
    n, s = 1026, 1024
    op = dtn.discretize(dtn.baseline_problem(3, s))
    sol = dtn.build_root_gpu(op, dtn.build_tree_uniform(n, 32), micro_max=micro)
    st = op.stencil
    idx = np.arange(s * s); x, y = idx % s, idx // s
    rows, cols, vals = [idx], [idx], [st[0]]
    for r, (dx, dy) in enumerate([(1, 0), (-1, 0), (0, 1), (0, -1)], start=1):
        ok = (x + dx >= 0) & (x + dx < s) & (y + dy >= 0) & (y + dy < s)
        rows.append(idx[ok]); cols.append((idx + dx + dy * s)[ok]); vals.append(st[r][ok])
    A = sp.csc_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(s * s, s * s))
    b = sol.boundary
    g = np.random.default_rng(3).standard_normal(len(b))
    rhs = np.zeros(s * s); rhs[b] = g
    ub = spla.splu(A).solve(rhs)[b]
    return [np.linalg.norm(dtn.apply_dtn(sol, g) - ub) / np.linalg.norm(ub),
            np.linalg.norm(sol.S_dense @ ub - g) / np.linalg.norm(g)]

if __name__ == "__main__":
    if len(sys.argv) > 1:
        print(json.dumps(run(int(sys.argv[1]))))
        sys.exit(0)
    envs = [{}, {"DTN_SUBST_REF": "1"}]
    for env in envs:
        out = subprocess.run([sys.executable, __file__, "128"], env=dict(os.environ, **env), capture_output=True, text=True)
        print(env, out.stdout.strip() or out.stderr[-300:], flush=True)
