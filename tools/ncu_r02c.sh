#!/bin/bash
# ncu evidence for the round-2 headline after the third session's kernel work (TMA-staged
# GEMM, fused one-CTA merges): (1) launch list of the headline bench command with per-launch
# duration and DRAM bytes (cold cache, serialised: shares, not absolutes); (2) full captures
# of the TMA GEMM (config-5 structured build and the dense solve) and of the fused merge kernel.
set -x
out=gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 6000 --csv \
    --log-file $out/r02c_ncu_launches_cfg3.csv \
    python bench.py --steps 1 --warmup 1 --no-cfg4 --no-solve --no-cpu-baseline > $out/r02c_ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"gemm_tma_kernel" --launch-skip 6 -c 5 \
    -o $out/r02c_tma_full python tools/k5_one.py 5 1 > $out/r02c_ncu_tma.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"fused_merge_kernel" -c 3 \
    -o $out/r02c_fused_full python tools/k5_one.py 3 1 > $out/r02c_ncu_fused.log 2>&1
