#!/usr/bin/env python
"""Benchmark of the build stage (leaf elimination + hierarchical merges + root
operator) and the solve stage on B200.

A step = one full build of the BASELINE workload from a stencil resident in HBM.
Default: configs[2] (BASELINE config 3, the largest single-GPU build config):
variable-coefficient convection-diffusion-reaction, kappa = 60, n = 1024 interior,
32 x 32 leaves, compressed (structured) merges above boundary 256 at eps = 1e-10 --
build_root_accel: structured merges, S_hbs = compress(root S), G_hbs = invert_hbs.
value = grid points/s over all ranks. e2e = the same metric through the public API
with host buffers (stencil H2D, the compressed operator's factors S_hbs and G_hbs
D2H as DTNHBS01 bytes -- what the reference adapter copies into SolutionOperator).
--config 2: the dense configuration (Helmholtz kappa=40, n=512, 16 vectors), e2e
with S and G D2H.

--impl reference: the reference's CPU path (restated C++ port of
proj/src/dense_nd.cpp with OpenBLAS; the reference itself needs Eigen, which is
not in this image) on all host cores, same metric and workload.

Multi-GPU (torchrun): one build per step, subtree-sharded over the GPUs
(paper_1302_5995_b200/shard.py) -- strong scaling.
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
    1: dict(name="laplace", n_int=256, leaf=16, nvec=1, oracle=("laplace", 0.0), compressed=False),
    2: dict(name="helmholtz_k40", n_int=512, leaf=16, nvec=16, oracle=("helmholtz", 40.0), compressed=False),
    3: dict(name="varcoef_k60", n_int=1024, leaf=32, nvec=0, oracle=("varcoef", 60.0), compressed=True),
}
EPS, CROSSOVER = 1e-10, 256
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
    r = O.build_root_dense(p, t, threads=threads, mode=2)  # S and G = S^{-1}, cond
    y = 0.0
    if cfg["nvec"]:
        X = seeded_vectors(len(r.boundary), cfg["nvec"])
        y = float(np.linalg.norm(r.G @ X))  # numpy/OpenBLAS DGEMM on the same cores
    dt = time.perf_counter() - t0
    return dt, y


def workload_text(args, cfg):
    if cfg["compressed"]:
        return (f"config{args.config}: {cfg['name']} n={cfg['n_int']} interior (ref n={cfg['n_int'] + 2}), "
                f"{cfg['leaf']}x{cfg['leaf']} leaves, compressed merges above boundary {CROSSOVER} at eps={EPS:g}: "
                f"root operator S_hbs and G_hbs = invert_hbs(S_hbs)")
    return (f"config{args.config}: {cfg['name']} n={cfg['n_int']} interior (ref n={cfg['n_int'] + 2}), "
            f"{cfg['leaf']}x{cfg['leaf']} leaves, dense FP64 merges, G applied to {cfg['nvec']} uniform[-1,1] vectors")


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
        "config": {"workload": workload_text(args, cfg)},
        "cpu_baseline": {"value": value, "unit": "grid-points/s", "cores": threads, "kind": "port",
                         "sample": f"{args.steps} full builds (S and G = S^-1"
                                   + (f", G*X for {cfg['nvec']} vectors" if cfg["nvec"] else "") +
                                   "), C++ restatement of dense_nd.cpp with OpenBLAS, all host threads (the "
                                   "reference needs Eigen, absent here; its compressed engine is not restated, so "
                                   "compressed configs are timed on the exact dense path)"},
        "e2e": {"value": value, "unit": "grid-points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ B200 arm
def build_cfg4_dense(dtn, torch, dev, reps=2):
    """configs[3]'s operator (Laplace, n=4096 interior, 32x32 leaves; 16.8M
    unknowns) on the DENSE engine on one GPU (the reference compresses these
    merges; dense is exact): S only, then one build with the dense G = S^{-1}
    (root LU of 16380 rows on the tall panel). Inputs resident in HBM; device
    time of the build from its events."""
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
    s = dtn.build_root_gpu(None, tree, want_G=True, stencil_device_ptr=st.data_ptr())
    g_ms = s.build_stats["build_ms"]
    s.free()
    peak_tf, _ = fp64_peak()
    del st
    torch.cuda.empty_cache()
    return {"workload": "config4 operator: laplace n=4096 interior, 32x32 leaves, dense FP64 merges (S only), 1 GPU",
            "build_ms": best["build_ms"], "grid_points_per_s": n_int ** 2 / (best["build_ms"] * 1e-3),
            "merge_tflops": best["merge_flops"] / (best["build_ms"] * 1e-3) / 1e12,
            "merge_frac_fp64_peak": best["merge_flops"] / (best["build_ms"] * 1e-3) / 1e12 / peak_tf,
            "merge_gflop": best["merge_flops"] / 1e9, "launches": best["launches"],
            "build_with_G_ms": g_ms}


def accel_opt(dtn):
    return dtn.AccelOptions(epsilon=EPS, crossover=CROSSOVER, hbs_leaf=64)


def compressed_build(dtn, torch, ctx, dev, stream, cfgno, n_int, leaf=32, reps=2, cpu=None):
    """build_root_accel (structured merges + compress + invert_hbs) of a BASELINE
    operator on one GPU from an HBM-resident stencil: device time of the whole call
    (CUDA events on the context stream), the structured build's own statistics, and
    the dense S-only build of the same operator beside it."""
    op = dtn.discretize(dtn.baseline_problem(cfgno, n_int))
    tree = dtn.build_tree_uniform(n_int + 2, leaf)
    st = torch.from_numpy(op.stencil).to(dev)
    opt = accel_opt(dtn)
    times, sol = [], None
    for rep in range(reps + 1):  # first: plans, graphs, learned factor ranks (untimed)
        sol = None
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        sol = dtn.build_root_accel(None, tree, opt, ctx=ctx, stencil_device_ptr=st.data_ptr())
        e1.record(stream)
        e1.synchronize()
        if rep:
            times.append(e0.elapsed_time(e1))
    ms = min(times)
    bs = sol.build_stats
    out = {"workload": f"config{cfgno} operator: n={n_int} interior, {leaf}x{leaf} leaves, compressed engine "
                       f"eps={EPS:g}, crossover {CROSSOVER} (structured merges -> compress root S -> invert_hbs), 1 GPU",
           "build_ms": ms, "grid_points_per_s": n_int ** 2 / (ms * 1e-3), "structured_build_ms": bs["build_ms"],
           "structured_merges": bs["structured_merges"], "max_rank": bs["max_rank"],
           "sketch_tail": bs["sketch_tail"], "arena_GB": bs["arena_bytes"] / 1e9,
           "arena_without_reuse_GB": bs["arena_sum_bytes"] / 1e9, "exec_tflop": bs["exec_flops"] / 1e12,
           "S_hbs_max_rank": sol.S_hbs.max_rank(), "G_hbs_max_rank": sol.G_hbs.max_rank(),
           "S_hbs_bytes": sol.S_hbs.payload_bytes(), "G_hbs_bytes": sol.G_hbs.payload_bytes(),
           "level_stats": [{"level": l.level, "max_rank": l.max_rank, "bytes": l.bytes} for l in sol.level_stats]}
    if cpu is not None:  # the oracle port on the host cores, one full build of the same operator (S and G):
        # a CPU figure and a parity check beside this configuration too (rank 0, N = 1 only)
        try:
            from oracle import oracle as O
            name, kappa = cpu
            threads = os.cpu_count() or 1
            t0 = time.perf_counter()
            ref = O.build_root_dense(O.Problem(name, n_int + 2, kappa), O.Tree(n_int + 2, uniform_side=leaf),
                                     threads=threads, mode=2)
            dt = time.perf_counter() - t0
            g = seeded_vectors(len(ref.boundary), 16)
            out["cpu_baseline"] = {"value": n_int ** 2 / dt, "unit": "grid-points/s", "cores": threads, "kind": "port",
                                   "sample": f"one full config{cfgno} build (S and G), C++ restatement of "
                                             "dense_nd.cpp (OpenBLAS, all host threads)", "seconds": dt}
            out["parity"] = {"Sg_hbs_rel_fro_vs_oracle": O.rel_fro(dtn.apply_schur(sol, g), ref.S @ g), "tol": 1e-9}
            del ref
        except Exception as e:  # pragma: no cover
            out["cpu_baseline"] = {"value": None, "error": repr(e)}
    del sol
    d = dtn.build_root_gpu(None, tree, want_G=False, ctx=ctx, stencil_device_ptr=st.data_ptr())
    d.free()
    d = dtn.build_root_gpu(None, tree, want_G=False, ctx=ctx, stencil_device_ptr=st.data_ptr())
    out["dense_S_only_build_ms"] = d.build_stats["build_ms"]
    d.free()
    del st
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
    ctx = dtn.collective_context(local) if world > 1 else dtn.Context(local)
    stream = torch.cuda.current_stream(dev)
    ctx.set_stream(stream.cuda_stream or 1)  # (torch legacy default stream = cudaStreamLegacy)

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

    def device_step():
        if world == 1:
            sol = dtn.build_root_gpu(None, tree, ctx=ctx, stencil_device_ptr=stencil_d.data_ptr())
        else:  # subtree-sharded build: shards on every GPU, top merges + inverse on rank 0
            sol = SH.build_collective(None, tree, ctx, stencil_device_ptr=stencil_d.data_ptr())
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

    def e2e_step():
        if world == 1:
            s = dtn.build_root_gpu(op_h, tree, ctx=ctx, export_S=True)
        else:
            s = SH.build_collective(op_h, tree, ctx)
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
                   "parallelism": (f"collective build x{world}: subtree shards, shard S all-gathered, top merges "
                                   f"and root inverse column-sharded (NCCL in the engine)" if world > 1
                                   else "single GPU"),
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
            line["config4_dense"] = build_cfg4_dense(dtn, torch, dev)
        except Exception as e:  # pragma: no cover
            line["config4_dense"] = {"error": str(e)}
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


def run_b200_compressed(args, cfg, rank, world, local):
    """The compressed configuration (default: BASELINE config 3): one step =
    build_root_accel -- leaf elimination, dense merges up to the crossover,
    structured merges above it (K5), S_hbs = compress(root S), G_hbs =
    invert_hbs(S_hbs) -- from an HBM-resident stencil."""
    import torch
    import paper_1302_5995_b200 as dtn
    from paper_1302_5995_b200 import hbs as H
    from paper_1302_5995_b200 import _lib as LB

    if world > 1:
        import torch.distributed as tdist
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    ctx = dtn.collective_context(local) if world > 1 else dtn.Context(local)
    stream = torch.cuda.current_stream(dev)
    ctx.set_stream(stream.cuda_stream or 1)
    n_int = cfg["n_int"]
    n = n_int + 2
    cfgno = args.config
    op = dtn.discretize(dtn.baseline_problem(cfgno, n_int))
    tree = dtn.build_tree_uniform(n, cfg["leaf"])
    opt = accel_opt(dtn)
    stencil_d = torch.from_numpy(op.stencil).to(dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MB > 126 MB L2
    from paper_1302_5995_b200 import shard as SH

    def device_step():
        if world == 1:
            return dtn.build_root_accel(None, tree, opt, ctx=ctx, stencil_device_ptr=stencil_d.data_ptr())
        return SH.build_collective(None, tree, ctx, stencil_device_ptr=stencil_d.data_ptr(), accel=opt)

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        device_step()
    barrier()
    events, hbs_launches, stats = [], 0, {"launches": 0}
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()  # L2 flush between timed steps (outside the events)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            h0 = LB.lib().dtn_gpu_hbs_launch_count()
            e0.record(stream)
            sol = device_step()
            e1.record(stream)
            hbs_launches += LB.lib().dtn_gpu_hbs_launch_count() - h0
            if sol is not None:
                stats = sol.build_stats
            events.append((e0, e1))
            del sol
        barrier()
    dev_ms = sum(a.elapsed_time(b) for a, b in events)
    t_local = torch.tensor([dev_ms], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(t_local, op=torch.distributed.ReduceOp.MAX)
    total_ms = float(t_local.item())
    value = args.steps * n_int ** 2 / (total_ms * 1e-3)

    # ---- e2e through the public API: host stencil in, S_hbs and G_hbs out (DTNHBS01 bytes)
    pin_st = torch.empty(op.stencil.shape, dtype=torch.float64, pin_memory=True).numpy()
    pin_st[...] = op.stencil
    op_h = dtn.DiscreteOperator(op.n, op.h, op.mode, pin_st)
    d2h = [0]

    def e2e_step():
        s_ = SH.build_collective(op_h, tree, ctx, accel=opt)
        if s_ is not None:
            d2h[0] = len(H.serialize(s_.S_hbs)) + len(H.serialize(s_.G_hbs))

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

    # ---- per-kernel roofline of the structured build (one profiled build, untimed above)
    peak_tf, peak_src = fp64_peak()
    hbm, hbm_src = hbm_peak()
    prof = dtn.build_root_gpu(None, tree, want_G=False, ctx=ctx, stencil_device_ptr=stencil_d.data_ptr(),
                              accel=opt, profile=True)
    ks = prof.kernel_stats
    pst = prof.build_stats
    prof.free()
    dom_name, dom = max(ks.items(), key=lambda kv: kv[1]["ms"])
    total_prof_ms = sum(v["ms"] for v in ks.values())
    achieved = dom["flops"] / (dom["ms"] * 1e-3) / 1e12 if dom["flops"] > 0 else 0.0
    roof = {"bound": "tensor", "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s", "frac": achieved / peak_tf,
            "traffic": None, "kernel": dom_name, "share_of_build": dom["ms"] / total_prof_ms,
            "launches": dom["launches"], "avg_launch_ms": dom["ms"] / max(1, dom["launches"]),
            "peak_source": peak_src + " (FP64; DMMA and DFMA share the FP64 peak on B200)"}
    try:
        with open(os.path.join(ROOT, "profiles", "r02c_ncu_traffic.json")) as f:
            roof["traffic"] = json.load(f).get(dom_name)
    except Exception:
        pass
    gemms = [(k, v) for k, v in ks.items() if v["flops"] > 0 and "gemm" in k]
    tname, tk = max(gemms, key=lambda kv: kv[1]["flops"])
    t_ach = tk["flops"] / (tk["ms"] * 1e-3) / 1e12
    line = {
        "metric": METRIC, "value": value, "unit": "grid-points/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, BASELINE config shapes)",
        "config": {"workload": workload_text(args, cfg),
                   "parallelism": (f"collective build x{world}: structured shard subtrees, shard S all-gathered, "
                                   f"top merges column-sharded (NCCL in the engine), root compressed on every rank"
                                   if world > 1 else "single GPU"),
                   "l2": "flushed between timed steps (256 MB write)"},
        "e2e": {"value": e2e_value, "unit": "grid-points/s", "h2d_bytes_per_step": int(op.stencil.nbytes),
                "d2h_bytes_per_step": int(d2h[0])},
        "gpu_launches": int(args.steps * stats["launches"] + hbs_launches),
        "roofline": roof,
        "roofline_throughput": {"bound": "tensor", "kernel": tname, "achieved": t_ach, "peak": peak_tf,
                                "unit": "TFLOP/s", "frac": t_ach / peak_tf, "launches": tk["launches"],
                                "share_of_build": tk["ms"] / total_prof_ms},
        "clocks": clk.summary(),
        "build": {"structured_build_ms": stats.get("build_ms"), "structured_merges": stats.get("structured_merges"),
                  "max_rank": stats.get("max_rank"), "sketch_tail": stats.get("sketch_tail"),
                  "arena_GB": stats.get("arena_bytes", 0) / 1e9,
                  "arena_without_reuse_GB": stats.get("arena_sum_bytes", 0) / 1e9,
                  "exec_tflop": stats.get("exec_flops", 0) / 1e12,
                  "dense_equivalent_merge_tflop": stats.get("merge_flops", 0) / 1e12,
                  "hbs_launches_per_step": hbs_launches / max(1, args.steps),
                  "profiled_ms": total_prof_ms, "profiled_build_ms": pst["build_ms"]},
        "kernels": {k: {"ms": round(v["ms"], 4), "launches": v["launches"],
                        "tflops": (v["flops"] / (v["ms"] * 1e-3) / 1e12) if v["ms"] > 0 and v["flops"] else None}
                    for k, v in ks.items() if v["launches"]},
    }
    if rank == 0 and world == 1:
        acc = device_step()
        line["build"]["level_stats"] = [{"level": l.level, "max_rank": l.max_rank, "bytes": l.bytes}
                                        for l in acc.level_stats]
        line["build"]["S_hbs_max_rank"] = acc.S_hbs.max_rank()
        line["build"]["G_hbs_max_rank"] = acc.G_hbs.max_rank()
        if not args.no_cpu_baseline:
            try:
                threads = os.cpu_count() or 1
                dts = [cpu_oracle_step(cfg, threads)[0] for _ in range(3)]
                dt = statistics.median(dts)
                line["cpu_baseline"] = {"value": n_int ** 2 / dt, "unit": "grid-points/s", "cores": threads,
                                        "kind": "port", "sample": f"median of 3 full config{cfgno} builds (S and G), "
                                        "C++ restatement of dense_nd.cpp (OpenBLAS, all host threads); the "
                                        "reference's compressed engine is not restated"}
                from oracle import oracle as O
                ref = O.build_root_dense(O.Problem(cfg["oracle"][0], n, cfg["oracle"][1]),
                                         O.Tree(n, uniform_side=cfg["leaf"]), threads=threads, mode=2)
                g = seeded_vectors(len(ref.boundary), 16)
                Sg = dtn.apply_schur(acc, g)
                line["parity"] = {"Sg_hbs_rel_fro_vs_oracle": O.rel_fro(Sg, ref.S @ g),
                                  "tol": 1e-7, "tol_note": "config 3's operator is near-resonant (cond(S) = 9e7): two exact "
                                  "FP64 eliminations differ by 3e-9..8e-9; bound 5 cond eps (tests/test_gpu_structured.py COND_TOL)"}
            except Exception as e:  # pragma: no cover
                line["cpu_baseline"] = {"value": None, "error": repr(e)}
        del acc
        if not args.no_cfg4:
            for key, cno, ni_ in (("config4_compressed", 4, 4096), ("config5_compressed_build", 5, 2048)):
                try:
                    cpu = ("helmholtz", 100.0) if (cno == 5 and not args.no_cpu_baseline) else None
                    line[key] = compressed_build(dtn, torch, ctx, dev, stream, cno, ni_, cpu=cpu)
                except Exception as e:  # pragma: no cover
                    line[key] = {"error": repr(e)}
            try:
                line["config4_dense"] = build_cfg4_dense(dtn, torch, dev)
            except Exception as e:  # pragma: no cover
                line["config4_dense"] = {"error": repr(e)}
    if not args.no_solve:
        try:
            sv = solve_cfg5(dtn, torch, ctx, dev, stream, rank, world, steps=max(3, args.steps // 2), warmup=5)
            sv["frac_fp64_peak"] = sv["tflops"] / peak_tf
            sv["dense"]["frac_fp64_peak"] = sv["dense"]["tflops"] / peak_tf
            line["solve"] = sv
        except Exception as e:  # pragma: no cover
            line["solve"] = {"error": repr(e)}
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
    ap.add_argument("--config", type=int, default=3, choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-solve", action="store_true", help="skip the config-5 solve measurement")
    ap.add_argument("--no-cfg4", action="store_true", help="skip the config-3/4 dense build measurements")
    args = ap.parse_args()
    rank, world, local = dist_env()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
    elif cfg["compressed"]:
        run_b200_compressed(args, cfg, rank, world, local)
    else:
        run_b200(args, cfg, rank, world, local)


if __name__ == "__main__":
    main()
