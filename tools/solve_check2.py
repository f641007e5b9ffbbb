"""Bisect the config-5 solve timing: bench.solve_cfg5 alone vs inside the bench flow (GPU)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1302_5995_b200 as dtn
dev = torch.device("cuda", 0)
ctx = dtn.Context(0)
stream = torch.cuda.current_stream(dev)
ctx.set_stream(stream.cuda_stream)
for i in range(2):
    r = bench.solve_cfg5(dtn, torch, ctx, dev, stream, 0, 1, steps=5, warmup=2)
    print("bench-ctx", r["ms_per_batch"], r["tflops"], flush=True)
ctx2 = dtn.Context(0)
for i in range(2):
    r = bench.solve_cfg5(dtn, torch, ctx2, dev, stream, 0, 1, steps=5, warmup=2)
    print("own-stream ctx", r["ms_per_batch"], r["tflops"], flush=True)
