#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TMB_EIG_2STAGE=1 timeout 900 python scripts/check_twostage.py 3840 5000 7680 > gpurun_out/mir_check.log 2>&1; echo "check rc=$?"
cat gpurun_out/mir_check.log
TMB_S2_MIRROR=0 timeout 600 python scripts/bench_eig.py 2 4700x600 7680x960 > gpurun_out/mir0.log 2>&1; echo "m0 rc=$?"
timeout 600 python scripts/bench_eig.py 2 4700x600 7680x960 > gpurun_out/mir1.log 2>&1; echo "m1 rc=$?"
cat gpurun_out/mir0.log gpurun_out/mir1.log
