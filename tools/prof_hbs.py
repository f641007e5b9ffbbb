"""The root compression (compress of the dense root S) and invert_hbs of a BASELINE config,
bracketed by cudaProfilerStart/Stop for `ncu --profile-from-start off`: python tools/prof_hbs.py 3"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1302_5995_b200 as dtn
from paper_1302_5995_b200 import hbs as H

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n_int = {3: 1024, 5: 2048, 4: 4096}[cfg]
op = dtn.discretize(dtn.baseline_problem(cfg, n_int))
tree = dtn.build_tree_uniform(n_int + 2, 32)
st = torch.from_numpy(op.stencil).cuda()
sol = dtn.build_root_gpu(None, tree, want_G=False, stencil_device_ptr=st.data_ptr(),
                         accel=dtn.AccelOptions(epsilon=1e-10, crossover=256))
for it in range(3):
    if it == 2:
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
    Sh = H.compress_operator(sol, "S", 1e-10, 64)
    Gh = H.invert_hbs(Sh)
    torch.cuda.synchronize()
    if it == 2:
        torch.cuda.profiler.stop()
print("ok", Sh.max_rank(), Gh.max_rank())
