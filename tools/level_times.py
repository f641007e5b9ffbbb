"""Per-level device time of a (non-graph) build: where the critical path goes (GPU)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("DTN_NO_GRAPH", "1")
import torch
import paper_1302_5995_b200 as dtn

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n_int = {1: 256, 2: 512}[cfg]
op = dtn.discretize(dtn.baseline_problem(cfg, n_int))
tree = dtn.build_tree_uniform(n_int + 2, 16)
st = torch.from_numpy(op.stencil).cuda()
for it in range(3):
    s = dtn.build_root_gpu(None, tree, stencil_device_ptr=st.data_ptr())
    if it == 2:
        b = s.build_stats
        print("build_ms %.3f leaf_ms %.3f merge_ms %.3f inverse_ms %.3f" % (b["build_ms"], b["leaf_ms"], b["merge_ms"],
                                                                          b["inverse_ms"]))
        for ls in s.level_stats:
            print(ls)
    s.free()
