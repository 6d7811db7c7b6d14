#!/bin/bash
# Round profiling bundle (run under gpurun): full bench with clocks, the ncu
# launch list of exactly one timed bench step, and ncu --set full captures of
# the dominant kernels (tridiagonalisation at both C2 sizes, the TTM GEMM).
# Launch accounting: bench.py issues LPS launches per step (its gpu_launches /
# steps); warm-up = 3 steps precede the timed step.
set -x
LPS=${LPS:-1938}
# bench.py samples nvidia-smi clocks itself during the timed region (its "clocks" key)
python bench.py > gpurun_out/bench_full.log 2>&1
python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -s $((3 * LPS)) -c $LPS --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu1.log 2>&1
python scripts/bench_eig.py 1 1080x270 1920x480 > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:sytrd_smem -c 4 -o gpurun_out/sytrd_smem_full python scripts/bench_eig.py 1 1080x270 1920x480 > gpurun_out/ncu2.log 2>&1
python scripts/bench_gemm.py 1 ttm1 > gpurun_out/plain3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_gemm -c 1 -o gpurun_out/gemm_ttm1_full python scripts/bench_gemm.py 1 ttm1 > gpurun_out/ncu3.log 2>&1
python scripts/check_ozaki.py > gpurun_out/plain4.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_oz_gemm -c 1 -o gpurun_out/oz_gemm_full python scripts/check_ozaki.py > gpurun_out/ncu4.log 2>&1
tail -1 gpurun_out/bench_full.log
