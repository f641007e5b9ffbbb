"""Run only the compressed-engine section of bench.py (one GPU)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1302_5995_b200 as dtn

dev = torch.device("cuda", 0)
ctx = dtn.default_context(0)
stream = torch.cuda.current_stream(dev)
ctx.set_stream(stream.cuda_stream)
print(json.dumps(bench.compressed_runs(dtn, torch, dev, stream, ctx), indent=1))
