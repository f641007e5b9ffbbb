"""Config-5 compressed solve timing (G_hbs applied to 4096 vectors), for A/B
runs of the HBS apply: python tools/hbs_solve_time.py [n_int] [batch]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1302_5995_b200 as dtn

n_int = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
dev = torch.device("cuda", 0)
ctx = dtn.default_context(0)
stream = torch.cuda.current_stream(dev)
ctx.set_stream(stream.cuda_stream)
op = dtn.discretize(dtn.baseline_problem(5, n_int))
tree = dtn.build_tree_uniform(n_int + 2, 32)
st = torch.from_numpy(op.stencil).to(dev)
sol = dtn.build_root_accel(None, tree, dtn.AccelOptions(epsilon=1e-10, crossover=256, hbs_leaf=64),
                           keep_dense=True, stencil_device_ptr=st.data_ptr())
nb = sol.boundary_size()
X = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, (batch, nb))).to(dev).t()
for _ in range(5):
    Y = dtn.apply_dtn(sol, X)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(5):
        Y = dtn.apply_dtn(sol, X)
    e1.record(stream)
    e1.synchronize()
    ts.append(e0.elapsed_time(e1) / 5)
ms = sorted(ts)[2]
R = dtn.apply_schur(sol.dense_op, Y)
err = float(torch.linalg.norm(R - X) / torch.linalg.norm(X))
print(f"n_int {n_int} nb {nb} batch {batch}: {ms:.3f} ms  {batch / ms * 1e3 / 1e6:.3f} M vectors/s  "
      f"residual |S Y - X|/|X| {err:.2e}  env {os.environ.get('DTN_GEMM_BIG', '')}")
