"""Config-4 operator (Laplace, n_int=4096, 32x32 leaves) on the dense engine, one GPU, no G (GPU)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1302_5995_b200 as dtn

n_int = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
leaf = 32
op = dtn.discretize(dtn.baseline_problem(4, n_int))
tree = dtn.build_tree_uniform(n_int + 2, leaf)
st = torch.from_numpy(op.stencil).cuda()
for it in range(2):
    t0 = time.time()
    s = dtn.build_root_gpu(None, tree, want_G=False, stencil_device_ptr=st.data_ptr())
    b = s.build_stats
    print("n_int", n_int, "build_ms %.1f" % b["build_ms"], "merge GF %.0f" % (b["merge_flops"] / 1e9),
          "TF/s %.2f" % (b["merge_flops"] / b["build_ms"] / 1e9), "wall %.2f s" % (time.time() - t0),
          "grid-pts/s %.3e" % (n_int ** 2 / (b["build_ms"] * 1e-3)),
          "mem GB %.1f" % (torch.cuda.mem_get_info()[1] / 1e9 - torch.cuda.mem_get_info()[0] / 1e9), flush=True)
    if it == 1:
        g = np.random.default_rng(1).uniform(-1, 1, s.boundary_size())
        Sg = dtn.apply_schur(s, g)
        print("S symmetric rel", float(np.linalg.norm(s.S_dense - s.S_dense.T) / np.linalg.norm(s.S_dense)))
    s.free()
