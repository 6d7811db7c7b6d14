#!/bin/bash
# ncu --set full (source-level stall samples) of the shared-memory tridiagonalisation at n = 1080 and n = 1920
mkdir -p gpurun_out
O=gpurun_out/r02s5f
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sytrd_smem" -s 2 -c 2 -o ${O}_sytrd_full python scripts/bench_eig.py 1 1080x270 1920x480 > ${O}_ncu.log 2>&1; echo "ncu rc=$?"
