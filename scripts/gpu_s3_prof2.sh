#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 120 python scripts/prof_twostage.py 2160 > gpurun_out/p2_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p2_launches.csv python scripts/prof_twostage.py 2160 > gpurun_out/p2_ncu.log 2>&1
echo rc=$?
python scripts/launch_summary.py gpurun_out/p2_launches.csv 2>&1 | head -40
