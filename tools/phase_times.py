"""Phase split of the graph-mode build (GPU): build time with / without the
root inverse and under the engine's schedule toggles, plus per-wave times."""
import json
import os
import subprocess
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if len(sys.argv) > 2 and sys.argv[2] == "child":
    import torch
    import paper_1302_5995_b200 as dtn
    cfg = int(sys.argv[1])
    n_int = {1: 256, 2: 512}[cfg]
    op = dtn.discretize(dtn.baseline_problem(cfg, n_int))
    tree = dtn.build_tree_uniform(n_int + 2, 16)
    st = torch.from_numpy(op.stencil).cuda()
    out = {}
    for want_G in (True, False):
        ts = []
        for _ in range(6):
            s = dtn.build_root_gpu(None, tree, want_G=want_G, stencil_device_ptr=st.data_ptr())
            ts.append(s.build_stats["build_ms"])
            s.free()
        out["G" if want_G else "noG"] = round(min(ts[1:]), 3)
    print(json.dumps(out))
    sys.exit(0)

cfg = sys.argv[1] if len(sys.argv) > 1 else "2"
for env in ({}, {"DTN_NO_FUSED": "1"}, {"DTN_NO_LOOKAHEAD": "1"}, {"DTN_BACKSUB_SUBST": "0"}):
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, __file__, cfg, "child"], env=e, capture_output=True, text=True)
    print(env, r.stdout.strip() or r.stderr[-500:])
