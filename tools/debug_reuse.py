import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1302_5995_b200 as dtn
from oracle import oracle as O
for names in (["laplace", "diffconv1", "diffconv1", "laplace"], ["diffconv1", "laplace"]):
    ctx = dtn.Context(0)
    for name in names:
        op = dtn.discretize(dtn.catalog(name, 8))
        try:
            s = dtn.build_root_gpu(op, dtn.build_tree(8, 16), ctx=ctx)
            ref = O.build_root_dense(O.Problem(name, 8), O.Tree(8, 16))
            print(name, "ok", O.rel_fro(s.S_dense, ref.S), flush=True)
            s.free()
        except Exception as e:
            print(name, "ERR", e, flush=True)
    ctx.close()
