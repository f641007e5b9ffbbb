"""A/B of an engine knob on the structured build: python tools/ab_struct.py CFG N_INT VAR=VALUE [oracle]
Builds S through the structured merges (want_G = False) with and without the setting in child
processes; reports build time, ranks, sketch tail, |S_a - S_b| / |S_b| and optionally both vs the oracle."""
import json, os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 2 and sys.argv[1] == "child":
    import numpy as np
    import torch
    import paper_1302_5995_b200 as dtn
    cfg, n_int = int(sys.argv[2]), int(sys.argv[3])
    op = dtn.discretize(dtn.baseline_problem(cfg, n_int))
    tree = dtn.build_tree_uniform(n_int + 2, 32)
    st = torch.from_numpy(op.stencil).cuda()
    opt = dtn.AccelOptions(epsilon=1e-10, crossover=256)
    ts = []
    for i in range(4):
        s = dtn.build_root_gpu(None, tree, want_G=False, accel=opt, stencil_device_ptr=st.data_ptr())
        ts.append(s.build_stats["build_ms"])
        if i < 3:
            s.free()
    bs = s.build_stats
    np.save(sys.argv[4], s.S_dense)
    print(json.dumps({"ms": min(ts), "max_rank": bs["max_rank"], "tail": bs["sketch_tail"],
                      "merges": bs["structured_merges"]}))
    sys.exit(0)
cfg, n_int, kv = sys.argv[1:4]
var, val = kv.split("=")
res = {}
for tag, env in (("on", {var: val}), ("off", {})):
    e = dict(os.environ)
    e.pop(var, None)
    e.update(env)
    r = subprocess.run([sys.executable, __file__, "child", cfg, n_int, f"/tmp/S_{tag}.npy"], env=e,
                       capture_output=True, text=True)
    res[tag] = json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else r.stderr[-1500:]
import numpy as np
a, b = np.load("/tmp/S_on.npy"), np.load("/tmp/S_off.npy")
res["S_rel_diff"] = float(np.linalg.norm(a - b) / np.linalg.norm(b))
if len(sys.argv) > 4 and sys.argv[4] == "oracle":
    from oracle import oracle as O
    p = {2: ("helmholtz", 40.0), 3: ("varcoef", 60.0), 1: ("laplace", 0.0), 5: ("helmholtz", 100.0)}[int(cfg)]
    n = int(n_int) + 2
    ref = O.build_root_dense(O.Problem(p[0], n, p[1]), O.Tree(n, uniform_side=32), threads=os.cpu_count(), mode=2)
    res["on_vs_oracle"] = O.rel_fro(a, ref.S)
    res["off_vs_oracle"] = O.rel_fro(b, ref.S)
print(cfg, n_int, kv, json.dumps(res), flush=True)
