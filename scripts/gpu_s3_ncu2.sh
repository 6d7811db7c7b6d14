#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 120 python scripts/prof_twostage.py 1000 > gpurun_out/n2_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_panel_qr|k_sb2st" -s 10 -c 2 -o gpurun_out/s3_twostage_full python scripts/prof_twostage.py 1000 > gpurun_out/n2_ncu.log 2>&1
echo rc=$?
tail -3 gpurun_out/n2_ncu.log
