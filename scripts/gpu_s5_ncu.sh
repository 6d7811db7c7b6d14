#!/bin/bash
# ncu --set full (source-level stall samples) of the Ozaki tcgen05 GEMM on the C2 mode-1 full pass
mkdir -p gpurun_out
O=gpurun_out/r02s5e
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_oz_gemm" -s 1 -c 1 -o ${O}_oz_full python scripts/check_ozaki.py > ${O}_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i ${O}_oz_full.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active,lts__t_bytes.sum,lts__t_sectors_srcunit_tex.sum,l1tex__m_xbar2l1tex_read_bytes.sum,dram__bytes_read.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_uniform.sum 2>&1 | tail -3 | cut -c1-900
