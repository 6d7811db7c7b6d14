#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_api.py -q -m gpu -x -k "lazy or large_n or kernel_paths" > gpurun_out/r02_t_lazy.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/r02_t_lazy.log
timeout 600 python scripts/bench_eig.py 2 4320x540 7680x960 > gpurun_out/r02_eig_lazy.txt 2>&1; cat gpurun_out/r02_eig_lazy.txt
TMB_LAZY=0 timeout 600 python scripts/bench_eig.py 2 4320x540 7680x960 > gpurun_out/r02_eig_nolazy.txt 2>&1; cat gpurun_out/r02_eig_nolazy.txt
