"""Config-4 dense build with G = S^{-1} (root LU of 16380 rows on the tall panel): build time
and the manufactured-solution check. python tools/cfg4_dense_g.py [n_int]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1302_5995_b200 as dtn

n_int = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
op = dtn.discretize(dtn.baseline_problem(4, n_int))
tree = dtn.build_tree_uniform(n_int + 2, 32)
st = torch.from_numpy(op.stencil).cuda()
out = {"n_int": n_int}
for want_G in (False, True, True):
    s = dtn.build_root_gpu(None, tree, want_G=want_G, stencil_device_ptr=st.data_ptr())
    out[f"build_ms_G{int(want_G)}"] = s.build_stats["build_ms"]
    if want_G:
        b = dtn.root_boundary(tree)
        h = 1.0 / (n_int + 1)
        x, y = b % n_int + 1, b // n_int + 1
        ub = (x * h) * (y * h)
        out["G_S_ub_rel"] = float(np.linalg.norm(dtn.apply_dtn(s, dtn.apply_schur(s, ub)) - ub) / np.linalg.norm(ub))
        out["cond_estimate"] = s.cond_estimate
    s.free()
print(json.dumps(out), flush=True)
