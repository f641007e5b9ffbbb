"""Host-side breakdown of the config-3 bench step: the device-stencil build
(DTN_HBS_TRACE / DTN_TRACE_BUILD phase laps on stderr) and the e2e step
(pinned host stencil in, both DTNHBS01 factor sets out)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1302_5995_b200 as dtn
from paper_1302_5995_b200 import hbs as H

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n_int = {3: 1024, 5: 2048, 4: 4096}[cfg]
dev = torch.device("cuda", 0)
op = dtn.discretize(dtn.baseline_problem(cfg, n_int))
tree = dtn.build_tree_uniform(n_int + 2, 32)
opt = bench.accel_opt(dtn)
st = torch.from_numpy(op.stencil).to(dev)
pin = torch.empty(op.stencil.shape, dtype=torch.float64, pin_memory=True).numpy()
pin[...] = op.stencil
op_h = dtn.DiscreteOperator(op.n, op.h, op.mode, pin)
for it in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s = dtn.build_root_accel(None, tree, opt, stencil_device_ptr=st.data_ptr())
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    del s
    t2 = time.perf_counter()
    s = dtn.build_root_accel(op_h, tree, opt)
    t3 = time.perf_counter()
    a = H.serialize(s.S_hbs)
    b = H.serialize(s.G_hbs)
    t4 = time.perf_counter()
    del s
    t5 = time.perf_counter()
    print(f"device-stencil step {1e3*(t1-t0):.3f} ms | e2e build {1e3*(t3-t2):.3f} serialize {1e3*(t4-t3):.3f} "
          f"({len(a)+len(b)} B) free {1e3*(t5-t4):.3f} total {1e3*(t5-t2):.3f} ms", flush=True)
