python -m pytest tests/test_gpu_api.py -x -q -k eig > gpurun_out/t18.log 2>&1; tail -2 gpurun_out/t18.log
python scripts/bench_eig.py 5 1080x270 1920x480 > gpurun_out/eig18.log 2>&1; cat gpurun_out/eig18.log
for t in 96 160; do TMB_SYTRD_TAIL1=$t python scripts/bench_eig.py 3 1080x270 1920x480 2>&1 | sed "s/^/tail1=$t /"; done
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench18.log 2>&1; tail -1 gpurun_out/bench18.log | cut -c1-300
