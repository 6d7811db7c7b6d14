#!/bin/bash
# iterate on the two-stage path: correctness (LAPACK) + launch list at one size
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TMB_S2_PROF=${S2PROF:-} TMB_EIG_2STAGE=1 timeout 300 python scripts/check_twostage.py ${SIZES:-257 1000 2160} > gpurun_out/it_check.log 2>&1; echo "check rc=$?"
cat gpurun_out/it_check.log | tail -12
timeout 120 python scripts/prof_twostage.py ${PN:-2160} > gpurun_out/it_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/it_launches.csv python scripts/prof_twostage.py ${PN:-2160} > gpurun_out/it_ncu.log 2>&1
echo "ncu rc=$?"
python scripts/launch_summary.py gpurun_out/it_launches.csv 2>&1 | head -24
