#!/bin/bash
# ncu --set full (source-level stall samples) of the column kernel and the lazy panels at n = 3840
mkdir -p gpurun_out
O=gpurun_out/r02s5g
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sytrd$|k_sytrd_lazy" -s 12 -c 2 -o ${O}_big_full python scripts/bench_eig.py 1 3840x960 > ${O}_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i ${O}_big_full.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active 2>&1 | tail -3 | cut -c1-600
