"""Repeated builds (dense + compressed, configs 5 and 4) on one context: device memory in use
must stay flat after the first round (plans cached per context, compression scratch and the
caching pool reused, factors freed with their operators)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1302_5995_b200 as dtn

def used_gb():
    free, total = torch.cuda.mem_get_info()
    return (total - free) / 1e9

for cfg, n_int in ((5, 2048), (4, 4096)):
    op = dtn.discretize(dtn.baseline_problem(cfg, n_int))
    tree = dtn.build_tree_uniform(n_int + 2, 32)
    st = torch.from_numpy(op.stencil).cuda()
    marks = []
    for it in range(4):
        acc = dtn.build_root_accel(None, tree, dtn.AccelOptions(epsilon=1e-10, crossover=256),
                                   stencil_device_ptr=st.data_ptr())
        X = torch.randn(len(acc.boundary), 256, dtype=torch.float64, device="cuda")
        Y = dtn.apply_dtn(acc, X)
        del acc, X, Y
        torch.cuda.synchronize()
        marks.append(round(used_gb(), 2))
    print(f"config {cfg}: device memory in use after each round (GB): {marks}")
    assert marks[-1] <= marks[1] + 0.5, marks
print("ok")
