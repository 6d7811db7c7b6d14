#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_stream.py -x -q -m gpu > gpurun_out/r02_t_stream.log 2>&1; echo "stream rc=$?"
timeout 900 python -m pytest tests/test_gpu_configs.py -q -m gpu -k "not c5" --durations=5 > gpurun_out/r02_t_configs.log 2>&1; echo "configs rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k golden_parity > gpurun_out/r02_t_parity.log 2>&1; echo "parity rc=$?"
timeout 900 python -m pytest tests/test_gpu_api.py -q -m gpu -k large_n --durations=5 > gpurun_out/r02_t_eiglarge.log 2>&1; echo "eig rc=$?"
tail -3 gpurun_out/r02_t_*.log
