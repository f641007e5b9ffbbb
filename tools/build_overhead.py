import os, sys, time
sys.path.insert(0, '.')
import torch
import paper_1302_5995_b200 as dtn
for cfg, n_int, leaf, G in ((2, 512, 16, True), (4, 4096, 32, False)):
    op = dtn.discretize(dtn.baseline_problem(cfg, n_int))
    tree = dtn.build_tree_uniform(n_int + 2, leaf)
    st = torch.from_numpy(op.stencil).cuda()
    for i in range(3):
        t0 = time.perf_counter()
        s = dtn.build_root_gpu(None, tree, want_G=G, stencil_device_ptr=st.data_ptr())
        t1 = time.perf_counter()
        print(cfg, "host total %.3f ms, graph %.3f ms" % ((t1 - t0) * 1e3, s.build_stats["build_ms"]), file=sys.stderr)
        s.free()
