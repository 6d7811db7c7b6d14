#!/bin/bash
# ncu of the two-stage's stage-1 group update GEMM and X GEMM at n = 7680 (C5 mode-1 Gram)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 300 python scripts/prof_twostage.py 7680 960 > gpurun_out/n5_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_gemm_dmma -s 25 -c 1 -o gpurun_out/s3_sbr_update python scripts/prof_twostage.py 7680 960 > gpurun_out/n5_ncu.log 2>&1
echo rc=$?
timeout 1200 ncu --set full --clock-control none -k regex:k_gemm_dmma -s 2 -c 1 -o gpurun_out/s3_sbr_x python scripts/prof_twostage.py 7680 960 > gpurun_out/n5b_ncu.log 2>&1
echo rc=$?
