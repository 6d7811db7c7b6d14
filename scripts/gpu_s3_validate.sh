#!/bin/bash
# full GPU suite + C4/C5 stack timings after the eigen-solver changes
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/v_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/v_tests.log
timeout 900 python scripts/config_families.py c4_2 c5 > gpurun_out/v_families.log 2>&1; echo "families rc=$?"
cat gpurun_out/v_families.log | tail -4
