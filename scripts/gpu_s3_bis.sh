#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TMB_BISECT_3T=0 timeout 300 python scripts/bench_eig.py 5 1080x270 1920x480 > gpurun_out/b0.log 2>&1; echo "b0 rc=$?"
timeout 300 python scripts/bench_eig.py 5 1080x270 1920x480 > gpurun_out/b1.log 2>&1; echo "b1 rc=$?"
cat gpurun_out/b0.log gpurun_out/b1.log
timeout 900 python -m pytest tests/test_gpu_api.py -q -x -k "eig or two_stage" 2>&1 | tail -2
