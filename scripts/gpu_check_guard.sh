python -m pytest tests/test_gpu_api.py tests/test_gpu_parity.py -x -q > gpurun_out/t20.log 2>&1; tail -2 gpurun_out/t20.log
python scripts/bench_eig.py 5 1080x270 1920x480 > gpurun_out/eig20.log 2>&1; cat gpurun_out/eig20.log
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench20.log 2>&1; tail -1 gpurun_out/bench20.log | cut -c1-300
