#!/bin/bash
# ncu evidence for the round-2 headline after the kernel work of this session
# (config-3 compressed build): (1) launch list of the headline bench command with
# per-launch duration and DRAM bytes (cold cache, serialised: shares, not absolutes);
# (2) full captures of the dominant kernels of the structured build.
set -x
out=gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 6000 --csv \
    --log-file $out/r02b_ncu_launches_cfg3.csv \
    python bench.py --steps 1 --warmup 1 --no-cfg4 --no-solve --no-cpu-baseline > $out/r02b_ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"panel2_kernel|hqrb_kernel|trailing_update|rowpanel|small_elim|gemm_big|gemm_desc_kernel" \
    --launch-skip 400 -c 14 -o $out/r02b_cfg3_full python tools/k5_one.py 3 2 > $out/r02b_ncu_full3.log 2>&1
