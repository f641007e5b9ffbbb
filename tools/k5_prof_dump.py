"""Per-launch timeline of one profiled structured build (DTN_PROF_DUMP=1 prints it on stderr)."""
import os
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_1302_5995_b200 as dtn

c = int(sys.argv[1]) if len(sys.argv) > 1 else 4
n_int, leaf = {3: (1024, 32), 5: (2048, 32), 4: (4096, 32), 2: (512, 16)}[c]
op = dtn.discretize(dtn.baseline_problem(c, n_int))
tree = dtn.build_tree_uniform(n_int + 2, leaf)
st = torch.from_numpy(op.stencil).cuda()
opt = dtn.AccelOptions(epsilon=1e-10, crossover=256)
dtn.build_root_gpu(None, tree, want_G=False, accel=opt, stencil_device_ptr=st.data_ptr()).free()
os.environ["DTN_PROF_DUMP"] = "1"
dtn.build_root_gpu(None, tree, want_G=False, accel=opt, stencil_device_ptr=st.data_ptr(), profile=True).free()
