"""Launch timeline of one profiled build (GPU): per-wave sums by kernel class."""
import os
import sys
import subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 2 and sys.argv[2] == "child":
    import torch
    import paper_1302_5995_b200 as dtn
    cfg = int(sys.argv[1])
    n_int = {1: 256, 2: 512}[cfg]
    op = dtn.discretize(dtn.baseline_problem(cfg, n_int))
    tree = dtn.build_tree_uniform(n_int + 2, 16)
    st = torch.from_numpy(op.stencil).cuda()
    for prof in (False, False, True):  # warm (lazy module loading), then the profiled build
        s = dtn.build_root_gpu(None, tree, stencil_device_ptr=st.data_ptr(), profile=prof)
        s.free()
    sys.exit(0)
cfg = sys.argv[1] if len(sys.argv) > 1 else "2"
r = subprocess.run([sys.executable, __file__, cfg, "child"], env=dict(os.environ, DTN_PROF_DUMP="1"),
                   capture_output=True, text=True)
from collections import defaultdict
agg = defaultdict(lambda: defaultdict(lambda: [0, 0.0, 0.0]))
span = {}
for line in r.stderr.splitlines():
    if line.startswith("prof panel fallbacks") or "pivoting panels" in line:
        print(line)
        continue
    if not line.startswith("prof wave"):
        continue
    f = line.split()
    w, k, start, dur, gf = int(f[2]), f[3], float(f[5]), float(f[8]), float(f[11])
    a = agg[w][k]
    a[0] += 1; a[1] += dur; a[2] += gf
    s0, s1 = span.get(w, (1e9, 0))
    span[w] = (min(s0, start), max(s1, start + dur))
for w in sorted(agg):
    s0, s1 = span[w]
    print(f"wave {w:3d} span {s1 - s0:8.3f} ms: " + ", ".join(
        f"{k} {v[0]}x {v[1]:.3f}ms {v[2] / max(v[1], 1e-9):.1f}TF" for k, v in sorted(agg[w].items(), key=lambda x: -x[1][1])))
if not agg:
    print(r.stderr[-2000:])
