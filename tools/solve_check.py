import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_1302_5995_b200 as dtn
n_int = 2048
op = dtn.discretize(dtn.baseline_problem(5, n_int))
st = torch.from_numpy(op.stencil).cuda()
sol = dtn.build_root_gpu(None, dtn.build_tree_uniform(n_int + 2, 32), stencil_device_ptr=st.data_ptr())
nb = len(sol.boundary)
G = torch.empty((nb, nb), dtype=torch.float64, device='cuda').t()
sol.export_device(None, 0, G.data_ptr(), nb)
print("G finite", bool(torch.isfinite(G).all()), "max", float(G.abs().max()), "min nonzero", float(G[G != 0].abs().min()))
X = torch.rand((4096, nb), dtype=torch.float64, device='cuda').t() * 2 - 1
X = X.t().contiguous().t()
for it in range(3):
    torch.cuda.synchronize(); t0 = time.time()
    for _ in range(5): Y = dtn.apply_dtn(sol, X)
    torch.cuda.synchronize(); dt = (time.time() - t0) / 5
    print("apply ms %.2f  TF/s %.1f" % (dt * 1e3, 2 * nb * nb * 4096 / dt / 1e12))
Gc = G.contiguous()
torch.cuda.synchronize(); t0 = time.time()
for _ in range(5): Y2 = G @ X
torch.cuda.synchronize(); dt = (time.time() - t0) / 5
print("torch matmul ms %.2f TF/s %.1f" % (dt * 1e3, 2 * nb * nb * 4096 / dt / 1e12))
Gr = torch.rand_like(G)
torch.cuda.synchronize(); t0 = time.time()
for _ in range(5): Y3 = Gr @ X
torch.cuda.synchronize(); dt = (time.time() - t0) / 5
print("torch matmul random ms %.2f TF/s %.1f" % (dt * 1e3, 2 * nb * nb * 4096 / dt / 1e12))
