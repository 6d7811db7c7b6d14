#!/bin/bash
# Session-3 state check: GPU test suite, default bench, eigen timings at C2/C4/C5 sizes.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/s3_tests.log 2>&1; echo "tests rc=$?"
timeout 600 python bench.py > gpurun_out/s3_bench.log 2>&1; echo "bench rc=$?"
timeout 600 python scripts/bench_eig.py 3 1080x270 1920x480 2160x540 3840x960 4320x540 > gpurun_out/s3_eig.log 2>&1; echo "eig rc=$?"
tail -3 gpurun_out/s3_tests.log; tail -1 gpurun_out/s3_bench.log | cut -c1-400; cat gpurun_out/s3_eig.log
