"""Per-kernel-class split of one profiled config-4 (n=4096) dense build (GPU)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1302_5995_b200 as dtn
n_int = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
op = dtn.discretize(dtn.baseline_problem(4, n_int))
tree = dtn.build_tree_uniform(n_int + 2, 32)
st = torch.from_numpy(op.stencil).cuda()
s = dtn.build_root_gpu(None, tree, want_G=False, stencil_device_ptr=st.data_ptr())
print("graph build_ms", s.build_stats["build_ms"]); s.free()
p = dtn.build_root_gpu(None, tree, want_G=False, stencil_device_ptr=st.data_ptr(), profile=True)
print("profiled build_ms", p.build_stats["build_ms"])
for k, v in sorted(p.kernel_stats.items(), key=lambda kv: -kv[1]["ms"]):
    if v["launches"]:
        print(f"{k:14s} {v['launches']:5d} {v['ms']:9.2f} ms  {v['flops'] / max(v['ms'], 1e-9) / 1e9:7.2f} TF/s")
