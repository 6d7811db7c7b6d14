#!/bin/bash
# A/B: one-stage vs two-stage leading_eigvecs at the C4/C5 Gram sizes
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
SZ=${SZ:-"2160x540 3840x960 4320x540 7680x960"}
TMB_EIG_2STAGE=0 timeout 600 python scripts/bench_eig.py 2 $SZ > gpurun_out/ab_1stage.log 2>&1; echo "1stage rc=$?"
TMB_EIG_2STAGE=1 timeout 600 python scripts/bench_eig.py 2 $SZ > gpurun_out/ab_2stage.log 2>&1; echo "2stage rc=$?"
echo "--- one-stage"; cat gpurun_out/ab_1stage.log; echo "--- two-stage"; cat gpurun_out/ab_2stage.log
