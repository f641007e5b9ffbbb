"""Key metrics of a one-kernel `ncu --set full` report: python tools/ncu_kernel_summary.py rep.ncu-rep"""
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, u, v = r[0], r[1], r[2]
want = ["Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.avg.per_cycle_active"]
print("| metric | value |\n|---|---|")
for k in want:
    if k in h:
        i = h.index(k)
        print(f"| {k} | {v[i]} {u[i]} |")
st = sorted(((float(v[i].replace(',', '')), h[i]) for i in range(len(h))
             if h[i].startswith("smsp__pcsamp_warps_issue_stalled") and not h[i].endswith("not_issued")
             and v[i].replace(',', '').replace('.', '').isdigit()), reverse=True)
tot = sum(x for x, _ in st) or 1
print("\nstall samples (top 6): " + ", ".join(f"{n.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * x / tot:.0f}%"
                                           for x, n in st[:6]))
