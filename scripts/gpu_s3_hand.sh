#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
SZ=${SZ:-"2160x270 2160x540 2160x1080 2500x97 3840x480 3840x960 3840x1920"}
TMB_SYTRD_HANDOFF=0 timeout 600 python scripts/bench_eig.py 2 $SZ > gpurun_out/h0.log 2>&1; echo "h0 rc=$?"
timeout 600 python scripts/bench_eig.py 2 $SZ > gpurun_out/h1.log 2>&1; echo "h1 rc=$?"
echo "--- no hand-off"; cat gpurun_out/h0.log; echo "--- hand-off"; cat gpurun_out/h1.log
timeout 900 python -m pytest tests/test_gpu_api.py -q -x -k "eig" 2>&1 | tail -2
