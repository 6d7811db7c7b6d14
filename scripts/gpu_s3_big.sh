#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TMB_EIG_2STAGE=1 timeout 900 python scripts/check_twostage.py 3840 4320 7680 > gpurun_out/big2.log 2>&1; echo "2stage rc=$?"
cat gpurun_out/big2.log
