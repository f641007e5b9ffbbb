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

# phase clocks of the fused merge kernel (CTA 0 of the last launch of each size class)
import ctypes as _C
from paper_1302_5995_b200 import _lib as _L
_buf = (_C.c_int64 * 24)()
if hasattr(_L.lib(), "dtn_debug_fused_clocks") and _L.lib().dtn_debug_fused_clocks(_buf) == 0:
    for c in range(3):
        q = list(_buf[8 * c:8 * c + 8])
        if q[4]:
            print(f"fused class {c}: assembly {q[1]-q[0]} LU {q[2]-q[1]} subst {q[3]-q[2]} gemm {q[4]-q[3]} clk (LU: panel {q[5]} update {q[6]})")
