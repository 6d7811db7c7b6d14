# Round profiling bundle (run under gpurun): full bench (clocks, cpu baseline),
# the ncu launch list of exactly one timed bench step, and ncu --set full
# captures of the kernels changed this session (cluster WY back-transform,
# Y'CbCr colour at C5 size, the DMMA TTM GEMM).
set -x
python bench.py > gpurun_out/bench_full.log 2>&1
LPS=$(python -c "import json;d=json.loads(open('gpurun_out/bench_full.log').read().strip().splitlines()[-1]);print(d['gpu_launches']//d['steps'])")
echo LPS=$LPS
python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -s $((3 * LPS)) -c $LPS --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu1.log 2>&1
python scripts/bench_eig.py 1 1920x480 > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_apply_wy_cl -c 1 -o gpurun_out/wy_cl_full python scripts/bench_eig.py 1 1920x480 > gpurun_out/ncu2.log 2>&1
python scripts/bench_elementwise.py 1 "c5 ycbcr" > gpurun_out/plain3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_color_u8 -c 1 -o gpurun_out/color_c5_full python scripts/bench_elementwise.py 1 "c5 ycbcr" > gpurun_out/ncu3.log 2>&1
python scripts/bench_elementwise.py 10 > gpurun_out/elem_full.log 2>&1
tail -1 gpurun_out/bench_full.log
