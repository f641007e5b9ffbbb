#!/usr/bin/env python
"""Benchmark of the build stage (leaf elimination + hierarchical merges +
root inverse) and the solve stage on B200.

A step = one full build of the BASELINE workload (default configs[1]:
Helmholtz kappa=40, n=512 interior, 16x16 leaves, dense FP64 merges) from a
stencil resident in HBM, plus G applied to the config's Dirichlet vectors
(16 for configs[1]). value = grid points/s over all ranks. e2e = the same
metric through the public API with host buffers (stencil H2D, vectors H2D,
DtN matrix S and the solution D2H inside the timed region).

--impl reference: the reference's CPU path (restated C++ port of
proj/src/dense_nd.cpp with OpenBLAS; the reference itself needs Eigen, which
is not in this image) on all host cores, same metric and workload.

Multi-GPU (torchrun): one build per step, subtree-sharded over the GPUs
(paper_1302_5995_b200/shard.py) — strong scaling.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    1: dict(name="laplace", n_int=256, leaf=16, nvec=1, oracle=("laplace", 0.0)),
    2: dict(name="helmholtz_k40", n_int=512, leaf=16, nvec=16, oracle=("helmholtz", 40.0)),
}
METRIC = "build grid-points/s"


def fp64_peak():
    """Measured FP64 peak (cuBLAS DGEMM 8192^3 on this pool, tools/probe/fp64_peak.py);
    MEASURED_PEAKS.json carries no FP64 entry."""
    try:
        with open(os.path.join(ROOT, "profiles", "r01_fp64_peak.json")) as f:
            d = json.load(f)
        return float(d["dgemm_tflops"]), "measured (profiles/r01_fp64_peak.json, cuBLAS DGEMM burst)"
    except Exception:
        return 37.0, "fallback (DMMA instruction-rate probe)"


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu, self.lines, self.proc = gpu, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                pass

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def seeded_vectors(nb: int, nvec: int, seed: int = 1) -> np.ndarray:
    rng = np.random.Generator(np.random.MT19937(seed))
    return np.asfortranarray(rng.uniform(-1.0, 1.0, (nb, nvec)))


# ------------------------------------------------------------------ reference arm
def cpu_oracle_step(cfg, threads):
    from oracle import oracle as O
    n = cfg["n_int"] + 2
    p = O.Problem(cfg["oracle"][0], n, cfg["oracle"][1])
    t = O.Tree(n, uniform_side=cfg["leaf"])
    t0 = time.perf_counter()
    r = O.build_root_dense(p, t, threads=threads, mode=2)
    X = seeded_vectors(len(r.boundary), cfg["nvec"])
    Y = r.G @ X  # numpy/OpenBLAS DGEMM on the same cores
    dt = time.perf_counter() - t0
    return dt, float(np.linalg.norm(Y))


def run_reference(args, cfg, rank, world):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_oracle_step(cfg, threads)
    times = [cpu_oracle_step(cfg, threads)[0] for _ in range(args.steps)]
    total = sum(times)
    value = args.steps * cfg["n_int"] ** 2 / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "grid-points/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"config{args.config}: {cfg['name']} n={cfg['n_int']} interior, "
                               f"{cfg['leaf']}x{cfg['leaf']} leaves, dense, {cfg['nvec']} vectors"},
        "cpu_baseline": {"value": value, "unit": "grid-points/s", "cores": threads, "kind": "port",
                         "sample": f"{args.steps} full builds + G*X ({cfg['nvec']} vectors), C++ restatement of "
                                   "dense_nd.cpp with OpenBLAS (Eigen absent; reference not buildable)"},
        "e2e": {"value": value, "unit": "grid-points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ B200 arm
def build_cfg3_dense(dtn, torch, dev, reps=3):
    """configs[2]'s operator (variable-coefficient convection-diffusion-reaction,
    kappa=60, n=1024 interior, 32x32 leaves) on the DENSE engine with G (the
    reference compresses above boundary 256; dense is exact). Device time of
    the build from its events, inputs resident in HBM."""
    n_int = 1024
    op = dtn.discretize(dtn.baseline_problem(3, n_int))
    tree = dtn.build_tree_uniform(n_int + 2, 32)
    st = torch.from_numpy(op.stencil).to(dev)
    best = None
    for _ in range(reps + 1):
        s = dtn.build_root_gpu(None, tree, stencil_device_ptr=st.data_ptr())
        b = s.build_stats
        s.free()
        best = b if best is None or b["build_ms"] < best["build_ms"] else best
    peak_tf, _ = fp64_peak()
    flops = best["merge_flops"] + best["inverse_flops"]
    return {"workload": "config3 operator: varcoef kappa=60 n=1024 interior, 32x32 leaves, dense FP64 merges + G, 1 GPU",
            "build_ms": best["build_ms"], "grid_points_per_s": n_int ** 2 / (best["build_ms"] * 1e-3),
            "tflops_algorithmic": flops / (best["build_ms"] * 1e-3) / 1e12,
            "frac_fp64_peak": flops / (best["build_ms"] * 1e-3) / 1e12 / peak_tf}


def build_cfg4_dense(dtn, torch, dev, reps=2):
    """configs[3]'s operator (Laplace, n=4096 interior, 32x32 leaves; 16.8M
    unknowns) on the DENSE engine on one GPU (the reference compresses these
    merges; dense is exact): S only (the root inverse needs a > 8192-row
    panel). Inputs resident in HBM; device time of the build from its events."""
    n_int = 4096
    op = dtn.discretize(dtn.baseline_problem(4, n_int))
    tree = dtn.build_tree_uniform(n_int + 2, 32)
    st = torch.from_numpy(op.stencil).to(dev)
    best = None
    for _ in range(reps + 1):  # first build: plan + graph capture (untimed)
        s = dtn.build_root_gpu(None, tree, want_G=False, stencil_device_ptr=st.data_ptr())
        b = s.build_stats
        s.free()
        best = b if best is None or b["build_ms"] < best["build_ms"] else best
    peak_tf, _ = fp64_peak()
    del st
    torch.cuda.empty_cache()
    return {"workload": "config4 operator: laplace n=4096 interior, 32x32 leaves, dense FP64 merges (S only), 1 GPU",
            "build_ms": best["build_ms"], "grid_points_per_s": n_int ** 2 / (best["build_ms"] * 1e-3),
            "merge_tflops": best["merge_flops"] / (best["build_ms"] * 1e-3) / 1e12,
            "merge_frac_fp64_peak": best["merge_flops"] / (best["build_ms"] * 1e-3) / 1e12 / peak_tf,
            "merge_gflop": best["merge_flops"] / 1e9, "launches": best["launches"]}


def compressed_runs(dtn, torch, dev, stream, ctx=None):
    """The compressed engine (build_root_accel: S from the exact dense merges,
    S_hbs = compress(S, 1e-10), G_hbs = invert_hbs(S_hbs)) on configs[2]-[4]'s
    operators, one GPU, and configs[4]'s solve through G_hbs. Device time of the
    whole call (CUDA events on the context stream; the dense build's own share
    from its events). Parity: S_hbs g against the dense S g of the same build
    (the dense engine is itself pinned to the oracle), and G_hbs (S g) = g."""
    peak_tf, _ = fp64_peak()
    out = {}
    if ctx is None:  # the default context: its cached plans (config-3/4 dense runs) are reused
        ctx = dtn.default_context(dev.index or 0)
        ctx.set_stream(stream.cuda_stream)
    for key, cfgno, n_int, leaf in (("config3", 3, 1024, 32), ("config5_build", 5, 2048, 32), ("config4", 4, 4096, 32)):
        op = dtn.discretize(dtn.baseline_problem(cfgno, n_int))
        tree = dtn.build_tree_uniform(n_int + 2, leaf)
        st = torch.from_numpy(op.stencil).to(dev)
        opt = dtn.AccelOptions(epsilon=1e-10, crossover=256, hbs_leaf=64)
        times = []
        sol = None
        for rep in range(4):  # first: plan + graph capture (untimed); then the best of three
            if sol is not None:
                sol.dense_op.free() if sol.dense_op is not None else None
                sol = None
            torch.cuda.synchronize(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            sol = dtn.build_root_accel(None, tree, opt, keep_dense=True, ctx=ctx, stencil_device_ptr=st.data_ptr())
            e1.record(stream)
            e1.synchronize()
            if rep:
                times.append((e0.elapsed_time(e1), sol.build_stats["build_ms"]))
        total_ms, dense_ms = min(times)
        nb = sol.boundary_size()
        g = torch.from_numpy(seeded_vectors(nb, 16)).to(dev).t().contiguous().t()
        Sg = dtn.apply_schur(sol.dense_op, g)
        Sg_h = dtn.apply_schur(sol, g)
        back = dtn.apply_dtn(sol, Sg)
        rel = lambda a, b: float(torch.linalg.norm(a - b) / torch.linalg.norm(b))
        r = {"workload": f"config{cfgno} operator n={n_int} interior, {leaf}x{leaf} leaves, compressed engine "
                         f"eps=1e-10 (dense merges -> compress root S -> invert_hbs)",
             "build_ms": total_ms, "dense_merges_ms": dense_ms, "compress_invert_ms": total_ms - dense_ms,
             "grid_points_per_s": n_int ** 2 / (total_ms * 1e-3),
             "boundary": nb, "S_max_rank": sol.S_hbs.max_rank(), "G_max_rank": sol.G_hbs.max_rank(),
             "S_hbs_bytes": sol.S_hbs.payload_bytes(), "G_hbs_bytes": sol.G_hbs.payload_bytes(),
             "dense_bytes": 8 * nb * nb, "cond_estimate": sol.cond_estimate,
             "Sg_rel_vs_dense": rel(Sg_h, Sg), "G_Sg_residual": rel(back, g), "tol": 1e-9}
        if cfgno == 5:  # configs[4]: the solve through G_hbs, 4096 vectors
            batch = 4096
            X = torch.from_numpy(seeded_vectors(nb, batch)).to(dev).t().contiguous().t()
            for _ in range(5):
                Y = dtn.apply_dtn(sol, X)
            torch.cuda.synchronize(dev)
            groups = []
            for _ in range(3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for _ in range(5):
                    Y = dtn.apply_dtn(sol, X)
                e1.record(stream)
                e1.synchronize()
                groups.append(e0.elapsed_time(e1) / 5)
            ms = sorted(groups)[1]
            P = sol.G_hbs.payload_bytes() / 8
            r["solve"] = {"workload": f"config5 solve: G_hbs applied to {batch} uniform[-1,1] vectors",
                          "vectors_per_s": batch / (ms * 1e-3), "ms_per_batch": ms,
                          "tflops": 2 * P * batch / (ms * 1e-3) / 1e12,
                          "frac_fp64_peak": 2 * P * batch / (ms * 1e-3) / 1e12 / peak_tf,
                          "flops_vs_dense": P / nb ** 2}
            del X, Y
        out[key] = r
        sol.dense_op.free()
        del sol, st, g, Sg, Sg_h, back
        torch.cuda.empty_cache()
    return out


def solve_cfg5(dtn, torch, ctx, dev, stream, rank, world, steps, warmup):
    """configs[4]: the DtN operator of the Helmholtz kappa=100, n=2048 build,
    compressed at 1e-10 (build_root_accel: G_hbs = invert_hbs(compress(S))),
    applied to 4096 seeded uniform[-1,1] Dirichlet vectors of length 4n-4,
    batch-sharded over the ranks (each rank holds the operator). Build
    untimed; the timed region is the batched apply from HBM-resident vectors.
    The same batch through the dense G (exact, 8188^2) is reported beside it."""
    n_int, batch = 2048, 4096
    n = n_int + 2
    op = dtn.discretize(dtn.baseline_problem(5, n_int))
    st = torch.from_numpy(op.stencil).to(dev)
    tree = dtn.build_tree_uniform(n, 32)
    acc = dtn.build_root_accel(None, tree, dtn.AccelOptions(epsilon=1e-10, crossover=256, hbs_leaf=64), ctx=ctx,
                               stencil_device_ptr=st.data_ptr())
    dense = dtn.build_root_gpu(None, tree, ctx=ctx, stencil_device_ptr=st.data_ptr())
    build_ms = dense.build_stats["build_ms"]
    nb = len(dense.boundary)
    mine = batch // world
    X = torch.from_numpy(seeded_vectors(nb, batch)[:, rank * mine:(rank + 1) * mine]).to(dev).t().contiguous().t()

    def timed(sol):
        for _ in range(warmup):
            dtn.apply_dtn(sol, X)
        torch.cuda.synchronize(dev)
        if world > 1:
            torch.distributed.barrier()
        # (the first batches after the untimed build run slow -- allocator / clock
        # ramp -- so the median of three timed groups after the warm-up is reported)
        groups = []
        with ClockSampler(torch.cuda.current_device()) as clk:
            for _ in range(3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for _ in range(steps):
                    Y = dtn.apply_dtn(sol, X)
                e1.record(stream)
                e1.synchronize()
                groups.append(e0.elapsed_time(e1) / steps)
        t = torch.tensor([sorted(groups)[1]], dtype=torch.float64, device=dev)
        if world > 1:
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item()), Y, clk.summary()

    ms_c, Yc, clk = timed(acc)
    ms_d, Yd, _ = timed(dense)
    rel = float(torch.linalg.norm(Yc - Yd) / torch.linalg.norm(Yd))
    P = acc.G_hbs.payload_bytes() / 8
    flops_c = 2.0 * P * batch
    flops_d = 2.0 * nb * nb * batch
    out = {"workload": f"config5: Helmholtz kappa=100 n={n_int}, operator compressed at 1e-10 (G_hbs = "
                       f"invert_hbs(S_hbs), max rank {acc.G_hbs.max_rank()}), applied to {batch} uniform[-1,1] "
                       f"vectors of length {nb}, batch-sharded x{world}",
           "vectors_per_s": batch / (ms_c * 1e-3), "ms_per_batch": ms_c, "tflops": flops_c / (ms_c * 1e-3) / 1e12,
           "G_hbs_vs_dense_G": rel, "clocks": clk,
           "hbm_GB_per_s": (8.0 * P + 16.0 * nb * mine) / (ms_c * 1e-3) / 1e9,
           "dense": {"workload": f"the same batch through the dense G ({nb}x{nb}, build {build_ms:.1f} ms untimed)",
                     "vectors_per_s": batch / (ms_d * 1e-3), "ms_per_batch": ms_d,
                     "tflops": flops_d / (ms_d * 1e-3) / 1e12}}
    dense.free()
    del acc, X
    return out


def run_b200(args, cfg, rank, world, local):
    import torch
    import paper_1302_5995_b200 as dtn

    if world > 1:
        import torch.distributed as tdist
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    ctx = dtn.Context(local)
    stream = torch.cuda.current_stream(dev)
    ctx.set_stream(stream.cuda_stream)

    n_int, nvec = cfg["n_int"], cfg["nvec"]
    n = n_int + 2
    spec = dtn.baseline_problem(args.config, n_int)
    op = dtn.discretize(spec)
    tree = dtn.build_tree_uniform(n, cfg["leaf"])
    nb = 4 * n_int - 4
    # inputs resident in HBM for the device-timed value
    stencil_d = torch.from_numpy(op.stencil).to(dev)
    X_h = seeded_vectors(nb, nvec)
    X_d = torch.from_numpy(X_h).to(dev).t().contiguous().t()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MB > 126 MB L2

    from paper_1302_5995_b200 import shard as SH
    eng_dev = SH.GpuShardEngine(None, tree, ctx=ctx, stencil_device_ptr=stencil_d.data_ptr(), device=dev)

    def device_step():
        if world == 1:
            sol = dtn.build_root_gpu(None, tree, ctx=ctx, stencil_device_ptr=stencil_d.data_ptr())
        else:  # subtree-sharded build: shards on every GPU, top merges + inverse on rank 0
            sol = SH.build_distributed(eng_dev, rank, world)
        Y = dtn.apply_dtn(sol, X_d) if sol is not None else None
        return sol, Y

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        sol, _ = device_step()
        if sol is not None:
            sol.free()
    barrier()
    events = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()  # L2 flush between timed steps (outside the events)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            sol, Y = device_step()
            e1.record(stream)
            if sol is not None:
                stats = sol.build_stats
                sol.free()
            events.append((e0, e1))
        barrier()
    dev_ms = sum(a.elapsed_time(b) for a, b in events)
    t_local = torch.tensor([dev_ms], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(t_local, op=torch.distributed.ReduceOp.MAX)
    total_ms = float(t_local.item())
    # world == 1: one build per step; world > 1: ONE sharded build of the same
    # problem per step over all GPUs (strong scaling)
    value = args.steps * n_int ** 2 / (total_ms * 1e-3)
    if rank != 0:
        stats = {"launches": 0}
    launches_per_step = stats["launches"] + (2 if nvec <= 32 else 1)  # + the apply (split-K: 2 kernels)

    # ---- e2e through the public API, host (pinned) buffers
    pin_st = torch.empty(op.stencil.shape, dtype=torch.float64, pin_memory=True).numpy()
    pin_st[...] = op.stencil
    op_h = dtn.DiscreteOperator(op.n, op.h, op.mode, pin_st)
    pin_x = torch.empty((nvec, nb), dtype=torch.float64, pin_memory=True).numpy().T
    pin_x[...] = X_h
    eng_host = SH.GpuShardEngine(op_h, tree, ctx=ctx, device=dev)

    def e2e_step():
        if world == 1:
            s = dtn.build_root_gpu(op_h, tree, ctx=ctx, export_S=True)
        else:
            s = SH.build_distributed(eng_host, rank, world)
        if s is not None:
            dtn.apply_dtn(s, pin_x)
            s.S_dense
            s.free()

    for _ in range(max(1, args.warmup // 2)):
        e2e_step()
    barrier()
    e2e_times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        e2e_step()
        torch.cuda.synchronize(dev)
        e2e_times.append(time.perf_counter() - t0)
    t_e2e = torch.tensor([sum(e2e_times)], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(t_e2e, op=torch.distributed.ReduceOp.MAX)
    e2e_value = args.steps * n_int ** 2 / float(t_e2e.item())

    # ---- per-kernel roofline from one profiled build (not timed above)
    prof = dtn.build_root_gpu(None, tree, ctx=ctx, stencil_device_ptr=stencil_d.data_ptr(), profile=True)
    ks = prof.kernel_stats
    pst = prof.build_stats  # per-phase split (leaf / merges / inverse) from the profiled, event-timed build
    prof.free()
    peak_tf, peak_src = fp64_peak()
    hbm, hbm_src = hbm_peak()
    dom_name, dom = max(ks.items(), key=lambda kv: kv[1]["ms"])
    total_prof_ms = sum(v["ms"] for v in ks.values())
    if dom["flops"] > 0:
        achieved = dom["flops"] / (dom["ms"] * 1e-3) / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s",
                "frac": achieved / peak_tf, "traffic": None, "kernel": dom_name,
                "share_of_build": dom["ms"] / total_prof_ms, "launches": dom["launches"],
                "avg_launch_ms": dom["ms"] / max(1, dom["launches"]), "peak_source": peak_src + " (FP64 DMMA)"}
    else:
        achieved = dom["bytes"] / (dom["ms"] * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "traffic": None, "kernel": dom_name, "share_of_build": dom["ms"] / total_prof_ms,
                "peak_source": hbm_src}
    try:
        with open(os.path.join(ROOT, "profiles", "r01_ncu_traffic.json")) as f:
            roof["traffic"] = json.load(f).get(dom_name)
    except Exception:
        pass
    if dom_name == "panel":
        roof["note"] = ("latency-bound pivot chain (32 sequential pivots per launch, a cluster exchange each on the "
                        "pivoted path); its FLOP/s fraction is small by construction -- see roofline_throughput")
    # the dominant throughput-bound (GEMM) class, for the tensor-pipe efficiency
    tname, tk = max(((k, v) for k, v in ks.items() if v["flops"] > 0 and "gemm" in k), key=lambda kv: kv[1]["flops"])
    t_ach = tk["flops"] / (tk["ms"] * 1e-3) / 1e12
    roof_t = {"bound": "tensor", "kernel": tname, "achieved": t_ach, "peak": peak_tf, "unit": "TFLOP/s",
              "frac": t_ach / peak_tf, "launches": tk["launches"], "share_of_build": tk["ms"] / total_prof_ms}

    merge_tf = pst["merge_flops"] / (pst["merge_ms"] * 1e-3) / 1e12 if pst["merge_ms"] > 0 else None
    line = {
        "metric": METRIC, "value": value, "unit": "grid-points/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE config shapes)",
        "config": {"workload": f"config{args.config}: {cfg['name']} n={n_int} interior (ref n={n}), "
                               f"{cfg['leaf']}x{cfg['leaf']} leaves, dense FP64 merges, G applied to "
                               f"{nvec} uniform[-1,1] vectors",
                   "parallelism": (f"subtree shards x{world} (NCCL gather of shard S to rank 0, top merges + "
                                   f"root inverse on rank 0)" if world > 1 else "single GPU"),
                   "l2": "flushed between timed steps (256 MB write)"},
        "e2e": {"value": e2e_value, "unit": "grid-points/s",
                "h2d_bytes_per_step": int(op.stencil.nbytes + X_h.nbytes),
                "d2h_bytes_per_step": int(nb * nb * 8 + nb * nvec * 8)},
        "gpu_launches": launches_per_step * args.steps,
        "roofline": roof,
        "roofline_throughput": roof_t,
        "clocks": clk.summary(),
        "build": {"build_ms": stats["build_ms"], "profiled_build_ms": pst["build_ms"], "leaf_ms": pst["leaf_ms"],
                  "merge_ms": pst["merge_ms"], "inverse_ms": pst["inverse_ms"],
                  "merge_gflop": pst["merge_flops"] / 1e9,
                  "merge_tflops": merge_tf,
                  "merge_frac_fp64_peak": merge_tf / peak_tf if merge_tf else None,
                  "build_tflops_algorithmic": (stats["merge_flops"] + stats["inverse_flops"]) /
                  (stats["build_ms"] * 1e-3) / 1e12,
                  "solve_vectors_per_s": None,
                  # leaf phase against HBM (coefficients in + S out per reference leaf)
                  "leaf_hbm": (lambda lb: {"bytes": lb, "GB_per_s": lb / (pst["leaf_ms"] * 1e-3) / 1e9,
                                           "frac_hbm": lb / (pst["leaf_ms"] * 1e-3) / 1e9 / hbm,
                                           "tflops": pst["leaf_flops"] / (pst["leaf_ms"] * 1e-3) / 1e12,
                                           "note": "latency-bound chain of in-leaf eliminations (6 waves)"})(
                      8.0 * (5 * cfg["leaf"] ** 2 + (4 * cfg["leaf"] - 4) ** 2) * (n_int // cfg["leaf"]) ** 2)
                  if pst["leaf_ms"] > 0 else None},
        "kernels": {k: {"ms": round(v["ms"], 4), "launches": v["launches"],
                        "tflops": (v["flops"] / (v["ms"] * 1e-3) / 1e12) if v["ms"] > 0 and v["flops"] else None}
                    for k, v in ks.items() if v["launches"]},
    }
    # solve throughput (device-resident, the configured batch)
    sol = dtn.build_root_gpu(None, tree, ctx=ctx, stencil_device_ptr=stencil_d.data_ptr())
    for _ in range(3):
        dtn.apply_dtn(sol, X_d)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    reps = 20
    for _ in range(reps):
        dtn.apply_dtn(sol, X_d)
    e1.record(stream)
    e1.synchronize()
    line["build"]["solve_vectors_per_s"] = reps * nvec / (e0.elapsed_time(e1) * 1e-3)
    # the small-batch solve is HBM-bound: G (8 nb^2 bytes) streamed once per batch
    sb = 8.0 * nb * nb + 16.0 * nb * nvec
    line["build"]["solve_hbm"] = {"bytes_per_batch": sb,
                                  "GB_per_s": sb / (e0.elapsed_time(e1) * 1e-3 / reps) / 1e9,
                                  "frac_hbm": sb / (e0.elapsed_time(e1) * 1e-3 / reps) / 1e9 / hbm}

    if not args.no_solve:
        try:
            peak_tf, _ = fp64_peak()
            sv = solve_cfg5(dtn, torch, ctx, dev, stream, rank, world, steps=max(3, args.steps // 2), warmup=5)
            sv["frac_fp64_peak"] = sv["tflops"] / peak_tf
            sv["dense"]["frac_fp64_peak"] = sv["dense"]["tflops"] / peak_tf
            line["solve"] = sv
        except Exception as e:  # pragma: no cover
            line["solve"] = {"error": str(e)}
    if rank == 0 and world == 1 and not args.no_cfg4:
        try:
            line["config3_dense"] = build_cfg3_dense(dtn, torch, dev)
        except Exception as e:  # pragma: no cover
            line["config3_dense"] = {"error": str(e)}
        try:
            line["config4_dense"] = build_cfg4_dense(dtn, torch, dev)
        except Exception as e:  # pragma: no cover
            line["config4_dense"] = {"error": str(e)}
        try:
            line["compressed"] = compressed_runs(dtn, torch, dev, stream)
        except Exception as e:  # pragma: no cover
            line["compressed"] = {"error": repr(e)}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            threads = os.cpu_count() or 1
            dts = [cpu_oracle_step(cfg, threads)[0] for _ in range(3)]
            dt = statistics.median(dts)
            line["cpu_baseline"] = {"value": n_int ** 2 / dt, "unit": "grid-points/s", "cores": threads,
                                    "kind": "port", "sample": f"median of 3 full config{args.config} builds + G*X, "
                                    "C++ restatement of dense_nd.cpp (OpenBLAS, all cores)"}
            # parity of this run's operator against the oracle (not timed)
            from oracle import oracle as O
            ref = O.build_root_dense(O.Problem(cfg["oracle"][0], n, cfg["oracle"][1]),
                                     O.Tree(n, uniform_side=cfg["leaf"]), threads=threads, mode=2)
            line["parity"] = {"S_rel_fro": O.rel_fro(sol.S_dense, ref.S),
                              "Sg_rel_fro": O.rel_fro(sol.S_dense @ X_h, ref.S @ X_h), "tol": 1e-10}
        except Exception as e:  # pragma: no cover
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    sol.free()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-solve", action="store_true", help="skip the config-5 solve measurement")
    ap.add_argument("--no-cfg4", action="store_true", help="skip the config-3/4 dense build measurements")
    args = ap.parse_args()
    rank, world, local = dist_env()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
    else:
        run_b200(args, cfg, rank, world, local)


if __name__ == "__main__":
    main()
