"""One compressed-engine build (build_root_accel) + one G_hbs solve of a
BASELINE config, for ncu launch lists: python tools/prof_compressed.py 5"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1302_5995_b200 as dtn

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
n_int = {3: 1024, 4: 4096, 5: 2048}[cfg]
dev = torch.device("cuda", 0)
op = dtn.discretize(dtn.baseline_problem(cfg, n_int))
tree = dtn.build_tree_uniform(n_int + 2, 32)
st = torch.from_numpy(op.stencil).to(dev)
sol = dtn.build_root_accel(None, tree, dtn.AccelOptions(epsilon=1e-10, crossover=256, hbs_leaf=64),
                           stencil_device_ptr=st.data_ptr())
nb = sol.boundary_size()
X = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, (4096, nb))).to(dev).t()
Y = dtn.apply_dtn(sol, X)
torch.cuda.synchronize()
print("ok", nb, sol.S_hbs.max_rank(), float(Y.abs().sum()))
