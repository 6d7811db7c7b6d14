# cluster row-split WY back-transform: tests + A/B; colour kernel timing
python -m pytest tests -m gpu -x -q > gpurun_out/t7.log 2>&1; tail -3 gpurun_out/t7.log
python scripts/bench_eig.py 5 1080x270 1920x480 1080x135 1920x240 601x150 > gpurun_out/eig7.log 2>&1
TMB_WY_NOCLUSTER=1 python scripts/bench_eig.py 5 1080x270 1920x480 1080x135 1920x240 601x150 > gpurun_out/eig7s.log 2>&1
cat gpurun_out/eig7.log gpurun_out/eig7s.log
python scripts/bench_elementwise.py 10 ycbcr > gpurun_out/elem7.log 2>&1; cat gpurun_out/elem7.log
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench7.log 2>&1; tail -1 gpurun_out/bench7.log | cut -c1-330
