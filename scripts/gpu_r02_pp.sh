#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_reference_suite.py tests/test_pp_parity.py tests/test_gpu_api.py -q -m gpu -x -s > gpurun_out/r02_t_pp_refsuite.log 2>&1; echo "rc=$?"
tail -45 gpurun_out/r02_t_pp_refsuite.log
