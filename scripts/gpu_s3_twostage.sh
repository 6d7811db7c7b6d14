#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TMB_EIG_2STAGE=1 timeout 300 python scripts/check_twostage.py ${SIZES:-100 257 700 1000 2160} > gpurun_out/s3_2stage.log 2>&1; echo "rc=$?"
cat gpurun_out/s3_2stage.log | tail -30
