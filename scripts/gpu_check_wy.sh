# A/B of the side-stream WY preparation + eig tests + ncu captures (colour C5 Y'CbCr, HOOI Grams)
set -x
python -m pytest tests/test_gpu_api.py -q -k "eig" > gpurun_out/t6.log 2>&1; tail -2 gpurun_out/t6.log
python scripts/bench_eig.py 5 1080x270 1920x480 > gpurun_out/eig6.log 2>&1
TMB_WY_SERIAL=1 python scripts/bench_eig.py 5 1080x270 1920x480 > gpurun_out/eig6s.log 2>&1
cat gpurun_out/eig6.log gpurun_out/eig6s.log
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench6.log 2>&1; tail -1 gpurun_out/bench6.log | cut -c1-400
ncu --set full --clock-control none --import-source on -k regex:k_color_u8 -c 1 -o gpurun_out/color_c5 python scripts/bench_elementwise.py 1 "c5 ycbcr" > gpurun_out/ncu6a.log 2>&1
python scripts/bench_gemm.py 2 gram_y1 > gpurun_out/gram6.log 2>&1; cat gpurun_out/gram6.log
ncu --set full --clock-control none --import-source on -k regex:k_gemm -c 3 -o gpurun_out/gram_y1 python scripts/bench_gemm.py 1 gram_y1 > gpurun_out/ncu6b.log 2>&1
