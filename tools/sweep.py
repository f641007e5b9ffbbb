"""Tuning sweep (GPU): build time vs leaf granularity (micro_max) and per-kernel split."""
import json
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1302_5995_b200 as dtn

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n_int = {1: 256, 2: 512}[cfg]
n = n_int + 2
op = dtn.discretize(dtn.baseline_problem(cfg, n_int))
tree = dtn.build_tree_uniform(n, 16)
st = torch.from_numpy(op.stencil).cuda()
for mm in [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["16", "36", "64", "100", "128", "160"])]:
    ts = []
    for it in range(8):
        s = dtn.build_root_gpu(None, tree, stencil_device_ptr=st.data_ptr(), micro_max=mm)
        ts.append(s.build_stats["build_ms"])
        s.free()
    p = dtn.build_root_gpu(None, tree, stencil_device_ptr=st.data_ptr(), micro_max=mm, profile=True)
    print(json.dumps({"micro_max": mm, "build_ms": min(ts[1:]), "leaf_ms": p.build_stats["leaf_ms"],
                      "merge_ms": p.build_stats["merge_ms"], "inverse_ms": p.build_stats["inverse_ms"],
                      "kernels": {k: (round(v["ms"], 3), v["launches"]) for k, v in p.kernel_stats.items()
                                  if v["launches"]}}))
    p.free()
