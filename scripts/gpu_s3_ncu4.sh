#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 120 python scripts/prof_twostage.py 1000 250 > gpurun_out/n4_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_band_invit" -c 1 -o gpurun_out/s3_invit_full python scripts/prof_twostage.py 1000 250 > gpurun_out/n4_ncu.log 2>&1
echo rc=$?
