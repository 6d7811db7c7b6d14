#!/bin/bash
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -x -m gpu > gpurun_out/s5_check2_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s5_check2_tests.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/s5_check2_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/s5_check2_bench.log | cut -c1-330
