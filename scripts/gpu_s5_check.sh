#!/bin/bash
# eigen-solver tests + C2 bench after the tridiagonalisation change
mkdir -p gpurun_out
O=gpurun_out/s5_check
timeout 1500 python -m pytest tests/test_gpu_api.py -q -x -k "eig or lapack or two_stage or hosvd" > ${O}_tests.log 2>&1; echo "tests rc=$?"; tail -3 ${O}_tests.log
timeout 600 python scripts/bench_eig.py 3 601x100 700x175 1000x250 1080x270 1300x300 1500x300 1700x300 1920x480 2040x300 > ${O}_eig.txt 2>&1; cat ${O}_eig.txt
timeout 900 python bench.py --no-cpu-baseline > ${O}_bench.log 2>&1; echo "bench rc=$?"; tail -1 ${O}_bench.log | cut -c1-330
