"""One structured build of a BASELINE operator (for ncu): python tools/k5_one.py CFG [reps]"""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_1302_5995_b200 as dtn

c = int(sys.argv[1]) if len(sys.argv) > 1 else 3
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
n_int, leaf = {3: (1024, 32), 5: (2048, 32), 4: (4096, 32), 2: (512, 16)}[c]
op = dtn.discretize(dtn.baseline_problem(c, n_int))
tree = dtn.build_tree_uniform(n_int + 2, leaf)
st = torch.from_numpy(op.stencil).cuda()
opt = dtn.AccelOptions(epsilon=1e-10, crossover=256)
for _ in range(reps):
    dtn.build_root_accel(None, tree, opt, stencil_device_ptr=st.data_ptr())
torch.cuda.synchronize()
print("done")
