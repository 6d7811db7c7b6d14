#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_api.py -q -m gpu -x -k "colour" > gpurun_out/r02_t_ipt2.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/r02_t_ipt2.log
timeout 600 python scripts/bench_elementwise.py 10 color_u8 > gpurun_out/r02_elementwise2.txt 2>&1; cat gpurun_out/r02_elementwise2.txt
