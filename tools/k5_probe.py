"""Structured-merge (K5) probe: build time, statistics and agreement with the dense
engine on the BASELINE operators. Usage: python tools/k5_probe.py [cfg ...]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_1302_5995_b200 as dtn

CFG = {3: (1024, 32), 5: (2048, 32), 4: (4096, 32), 2: (512, 16)}


def main():
    cfgs = [int(a) for a in sys.argv[1:] if a.isdigit()] or [3, 5, 4]
    for c in cfgs:
        n_int, leaf = CFG[c]
        n = n_int + 2
        op = dtn.discretize(dtn.baseline_problem(c, n_int))
        tree = dtn.build_tree_uniform(n, leaf)
        st = torch.from_numpy(op.stencil).cuda()
        opt = dtn.AccelOptions(epsilon=1e-10, crossover=256)
        ts = []
        for rep in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            sol = dtn.build_root_gpu(None, tree, want_G=False, accel=opt, stencil_device_ptr=st.data_ptr())
            torch.cuda.synchronize()
            ts.append((time.perf_counter() - t0) * 1e3)
            bs = sol.build_stats
            if rep < 2:
                sol.free()
        print(f"cfg{c} structured: wall {ts} ms, device {bs['build_ms']:.2f} ms, merges {bs['structured_merges']}, "
              f"max_rank {bs['max_rank']}, tail {bs['sketch_tail']:.2e}, arena {bs['arena_bytes']/1e9:.2f} GB "
              f"(sum {bs['arena_sum_bytes']/1e9:.2f}), exec {bs['exec_flops']/1e12:.3f} TF", flush=True)
        print(f"   rank attempts {bs['rank_attempts']}", flush=True)
        if "--prof" in sys.argv or True:
            pr = dtn.build_root_gpu(None, tree, want_G=False, accel=opt, stencil_device_ptr=st.data_ptr(), profile=True)
            ks = sorted(pr.kernel_stats.items(), key=lambda kv: -kv[1]["ms"])
            tot = sum(v["ms"] for _, v in ks)
            print("   profile (summed launch ms): " + ", ".join(f"{k} {v['ms']:.1f} ({v['launches']})" for k, v in ks
                                                             if v["launches"]) + f"; total {tot:.1f}", flush=True)
            pr.free()
        for lv in sol.level_stats:
            print(f"   level {lv.level}: boxes {lv.boxes} max_rank {lv.max_rank} bytes {lv.bytes/1e6:.1f} MB", flush=True)
        nb = len(sol.boundary)
        S = torch.empty((nb, nb), dtype=torch.float64, device="cuda").t()
        sol.export_device(S.data_ptr(), nb)
        sol.free()
        d = dtn.build_root_gpu(None, tree, want_G=False, stencil_device_ptr=st.data_ptr())
        Sd = torch.empty((nb, nb), dtype=torch.float64, device="cuda").t()
        d.export_device(Sd.data_ptr(), nb)
        print(f"   dense build {d.build_stats['build_ms']:.2f} ms, arena {d.build_stats['arena_bytes']/1e9:.2f} GB; "
              f"|S_struct - S_dense| / |S_dense| = {float(torch.linalg.norm(S - Sd) / torch.linalg.norm(Sd)):.3e}",
              flush=True)
        d.free()
        del S, Sd, st
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
