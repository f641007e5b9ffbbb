"""Markdown table of key metrics for every kernel in an `ncu --set full` report:
python tools/ncu_table.py rep.ncu-rep"""
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, u = r[0], r[1]
cols = [("Kernel Name", "kernel"), ("launch__grid_size", "grid"), ("gpu__time_duration.sum", "time"),
        ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "DMMA %"),
        ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
        ("dram__bytes_read.sum", "DRAM rd"), ("dram__bytes_write.sum", "DRAM wr"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM thr %")]
print("| " + " | ".join(c[1] for c in cols) + " | top stalls |")
print("|" + "---|" * (len(cols) + 1))
for v in r[2:]:
    cells = []
    for k, _ in cols:
        i = h.index(k)
        val = v[i]
        if k == "Kernel Name":
            val = val.split("(")[0].replace("void ", "")
        elif u[i]:
            val = f"{val} {u[i]}"
        cells.append(val)
    st = sorted(((float(v[i].replace(',', '')), h[i]) for i in range(len(h))
                 if h[i].startswith("smsp__pcsamp_warps_issue_stalled") and not h[i].endswith("not_issued")
                 and v[i].replace(',', '').replace('.', '').isdigit()), reverse=True)
    tot = sum(x for x, _ in st) or 1
    cells.append(", ".join(f"{n.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * x / tot:.0f}%"
                           for x, n in st[:3]))
    print("| " + " | ".join(cells) + " |")
