#!/bin/bash
# Ozaki tcgen05 GEMM after the elect.sync issue path: accuracy + time, the N = 128 variant, Ozaki tests, C2 bench
mkdir -p gpurun_out
O=gpurun_out/s5_oz
timeout 600 python scripts/check_ozaki.py > ${O}_check.txt 2>&1; cat ${O}_check.txt
TMB_OZ_N128=1 timeout 600 python scripts/check_ozaki.py > ${O}_check128.txt 2>&1; cat ${O}_check128.txt
timeout 1500 python -m pytest tests -q -x -m gpu -k "ozaki or ttm or golden or c2" 2>&1 | tail -3
timeout 900 python bench.py --no-cpu-baseline > ${O}_bench.log 2>&1; echo "bench rc=$?"; tail -1 ${O}_bench.log | cut -c1-330
