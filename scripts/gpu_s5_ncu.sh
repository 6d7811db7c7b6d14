#!/bin/bash
# ncu --set full of the shared-memory tridiagonalisation at n = 1920 (256-thread blocks, 4 register columns) and of the tail
mkdir -p gpurun_out
O=gpurun_out/r02s5b
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sytrd_smem|sytrd_tail2|bisect_tw" -s 3 -c 3 -o ${O}_sytrd1920_full python scripts/bench_eig.py 1 1920x480 > ${O}_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i ${O}_sytrd1920_full.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,sm__warps_active.avg.pct_of_peak_sustained_active > ${O}_sytrd1920_raw.csv 2>&1
cat ${O}_sytrd1920_raw.csv | cut -c1-600
