"""Host-side breakdown of the bench's e2e step (config 2): build from a pinned host
stencil with S exported during the root inverse, G X for 16 pinned host vectors, S read."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1302_5995_b200 as dtn
import bench

n_int, nvec = 512, 16
op = dtn.discretize(dtn.baseline_problem(2, n_int))
tree = dtn.build_tree_uniform(n_int + 2, 16)
nb = 4 * n_int - 4
pin_st = torch.empty(op.stencil.shape, dtype=torch.float64, pin_memory=True).numpy()
pin_st[...] = op.stencil
op_h = dtn.DiscreteOperator(op.n, op.h, op.mode, pin_st)
pin_x = torch.empty((nvec, nb), dtype=torch.float64, pin_memory=True).numpy().T
pin_x[...] = bench.seeded_vectors(nb, nvec)
for it in range(6):
    t0 = time.perf_counter()
    s = dtn.build_root_gpu(op_h, tree, export_S=True)
    t1 = time.perf_counter()
    y = dtn.apply_dtn(s, pin_x)
    t2 = time.perf_counter()
    S = s.S_dense
    bms = s.build_stats["build_ms"]
    s.free()
    t3 = time.perf_counter()
    if it >= 3:
        print(f"build call {1e3 * (t1 - t0):.3f} ms (graph {bms:.3f}), apply {1e3 * (t2 - t1):.3f} ms, "
              f"S + free {1e3 * (t3 - t2):.3f} ms, total {1e3 * (t3 - t0):.3f} ms")
