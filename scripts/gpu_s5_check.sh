#!/bin/bash
# full GPU suite + C2 bench (driver command) + C3 bench after a kernel change
mkdir -p gpurun_out
O=gpurun_out/s5_check
timeout 600 python scripts/bench_eig.py 3 601x100 1080x270 1920x480 2160x540 > ${O}_eig.txt 2>&1; cat ${O}_eig.txt
timeout 2400 python -m pytest tests -q -x -m gpu > ${O}_tests.log 2>&1; echo "tests rc=$?"; tail -3 ${O}_tests.log
timeout 900 python bench.py --steps 20 --warmup 5 > ${O}_bench.log 2>&1; echo "bench rc=$?"; tail -1 ${O}_bench.log | cut -c1-330
