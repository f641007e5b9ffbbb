"""A/B accuracy experiments: GPU S and G*g vs an independent sparse LU, per toggle."""
import os, sys, subprocess, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

def run(nint, micro, cfg):
    import paper_1302_5995_b200 as dtn
    n = nint + 2
    op = dtn.discretize(dtn.baseline_problem(cfg, nint))
    st = op.stencil; s = nint
    idx = np.arange(s * s); x = idx % s; y = idx // s
    rows = [idx]; cols = [idx]; vals = [st[0]]
    for r, (dx, dy) in enumerate([(1, 0), (-1, 0), (0, 1), (0, -1)], start=1):
        ok = (x + dx >= 0) & (x + dx < s) & (y + dy >= 0) & (y + dy < s)
        rows.append(idx[ok]); cols.append((idx + dx + dy * s)[ok]); vals.append(st[r][ok])
    A = sp.csc_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(s * s, s * s))
    lu = spla.splu(A)
    sol = dtn.build_root_gpu(op, dtn.build_tree_uniform(n, 32 if nint >= 1024 else 16), micro_max=micro)
    b = sol.boundary
    g = np.random.default_rng(3).standard_normal(len(b))
    rhs = np.zeros(s * s); rhs[b] = g
    ub = lu.solve(rhs)[b]
    return (np.linalg.norm(sol.G_dense @ g - ub) / np.linalg.norm(ub), np.linalg.norm(sol.S_dense @ ub - g) / np.linalg.norm(g))

if __name__ == "__main__":
    if len(sys.argv) > 1:
        nint, micro, cfg = map(int, sys.argv[1:4])
        print(json.dumps(run(nint, micro, cfg)))
        sys.exit(0)
    exps = [({}, 512, 0, 3), ({"DTN_NO_LOOKAHEAD": "1", "DTN_NO_GRAPH": "1"}, 512, 0, 3),
            ({}, 512, 16, 3), ({}, 512, 160, 3), ({}, 512, 0, 2), ({}, 256, 0, 3)]
    if os.environ.get("AB_SET") == "backsub":
        exps = [(e, nint, 0, cfg) for nint, cfg in ((512, 2), (512, 3), (1024, 3))
                for e in ({}, {"DTN_BACKSUB_SUBST": "0"}, {"DTN_NO_FUSED": "1"})]
    for env, nint, micro, cfg in exps:
        e = dict(os.environ); e.update(env)
        out = subprocess.run([sys.executable, __file__, str(nint), str(micro), str(cfg)], env=e, capture_output=True, text=True)
        print(env, nint, micro, cfg, out.stdout.strip() or out.stderr[-300:], flush=True)
