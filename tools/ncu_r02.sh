#!/bin/bash
# ncu evidence for the round-2 headline (config 3 compressed build) and config 4:
# (1) the launch list of the headline bench command (per-launch gpu__time_duration,
#     no clock control -- cold-cache, serialised: shares, not absolutes);
# (2) full captures of the dominant kernels (sketch QR, panel, the big DMMA GEMMs).
set -x
out=gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $out/r02_ncu_launches_cfg3.csv \
    python bench.py --steps 2 --warmup 1 --no-cfg4 --no-solve --no-cpu-baseline > $out/r02_ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"hqr|panel_kernel|gemm_big|gemm_desc_kernel|trailing" \
    --launch-skip 300 -c 12 -o $out/r02_cfg3_full python tools/k5_one.py 3 2 > $out/r02_ncu_full3.log 2>&1
ncu --set full --clock-control none -k regex:"gemm_big" --launch-skip 20 -c 4 -o $out/r02_cfg4_gemm \
    python tools/k5_one.py 4 1 > $out/r02_ncu_full4.log 2>&1
