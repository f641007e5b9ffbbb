"""Deferred boundary columns (NodeDev::defer) A/B: S of a build with deferral against
the same build without (DTN_DEFER_MIN_WORK=0 in a child), and the build time."""
import json, os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 2 and sys.argv[1] == "child":
    import numpy as np
    import torch
    import paper_1302_5995_b200 as dtn
    cfg, n_int, leaf = [int(x) for x in sys.argv[2:5]]
    op = dtn.discretize(dtn.baseline_problem(cfg, n_int))
    tree = dtn.build_tree_uniform(n_int + 2, leaf)
    st = torch.from_numpy(op.stencil).cuda()
    ts = []
    for _ in range(3):
        s = dtn.build_root_gpu(None, tree, want_G=False, stencil_device_ptr=st.data_ptr())
        ts.append(s.build_stats["build_ms"])
        last = s
        if _ < 2:
            s.free()
    nb = last.boundary_size()
    S = torch.empty((nb, nb), dtype=torch.float64, device="cuda").t()
    last.export_device(S.data_ptr(), nb)
    torch.save(S.cpu(), sys.argv[5])
    print(json.dumps({"ms": min(ts)}))
    sys.exit(0)
cfg, n_int, leaf = sys.argv[1:4]
res = {}
for tag, env in (("defer", {}), ("nodefer", {"DTN_DEFER_MIN_WORK": "0"})):
    r = subprocess.run([sys.executable, __file__, "child", cfg, n_int, leaf, f"/tmp/S_{tag}.pt"],
                       env=dict(os.environ, **env), capture_output=True, text=True)
    res[tag] = json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else r.stderr[-2000:]
import torch
a, b = torch.load("/tmp/S_defer.pt"), torch.load("/tmp/S_nodefer.pt")
res["S_rel_diff"] = float(torch.linalg.norm(a - b) / torch.linalg.norm(b))
print(cfg, n_int, json.dumps(res))
