#!/bin/bash
# after the incremental slot counters: eigen tests, sizes incl. the hand-off path, C2 bench
mkdir -p gpurun_out
O=gpurun_out/s5_idiv.txt
timeout 600 python scripts/bench_eig.py 3 601x100 700x175 1080x270 1500x300 1920x480 2040x300 2160x540 3840x960 > $O 2>&1; cat $O
timeout 1500 python -m pytest tests/test_gpu_api.py -q -x -k "eig or lapack or two_stage or hosvd" 2>&1 | tail -3
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/s5_idiv_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/s5_idiv_bench.log | cut -c1-330
