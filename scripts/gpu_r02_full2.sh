#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu --durations=10 > gpurun_out/r02_pytest_gpu_full2.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/r02_pytest_gpu_full2.log
timeout 1500 python scripts/run_configs.py c4_8 c4_4 c4_2 c5 > gpurun_out/r02_configs2.txt 2>&1; echo "configs rc=$?"; cat gpurun_out/r02_configs2.txt
timeout 900 python scripts/config_families.py c5 > gpurun_out/r02_families2.txt 2>&1; cat gpurun_out/r02_families2.txt
timeout 1500 python scripts/parity_report.py > gpurun_out/r02_parity.txt 2>&1; echo "parity rc=$?"; cat gpurun_out/r02_parity.txt
