#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python scripts/config_families.py c2 c5 > gpurun_out/oz0_off.log 2>&1; echo "off rc=$?"
TMB_OZ_MODE0=1 timeout 900 python scripts/config_families.py c2 c5 > gpurun_out/oz0_on.log 2>&1; echo "on rc=$?"
tail -2 gpurun_out/oz0_off.log; tail -2 gpurun_out/oz0_on.log
