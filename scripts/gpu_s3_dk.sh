#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TMB_SYTRD_DK=0 timeout 300 python scripts/bench_eig.py 5 1080x270 1920x480 > gpurun_out/dk0.log 2>&1; echo "dk0 rc=$?"
timeout 300 python scripts/bench_eig.py 5 1080x270 1920x480 > gpurun_out/dk1.log 2>&1; echo "dk1 rc=$?"
cat gpurun_out/dk0.log gpurun_out/dk1.log
timeout 900 python -m pytest tests/test_gpu_api.py -q -x -k "eig" 2>&1 | tail -2
