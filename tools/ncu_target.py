"""Short target for ncu captures: config-2 build (warm-up + one measured build)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1302_5995_b200 as dtn

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n_int = {1: 256, 2: 512}[cfg]
op = dtn.discretize(dtn.baseline_problem(cfg, n_int))
tree = dtn.build_tree_uniform(n_int + 2, 16)
st = torch.from_numpy(op.stencil).cuda()
for _ in range(2):
    s = dtn.build_root_gpu(None, tree, stencil_device_ptr=st.data_ptr())
    print("build_ms", s.build_stats["build_ms"], "launches", s.build_stats["launches"])
    s.free()
