#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for sw in 1000 1500 2000 2500 3000 3500; do
  echo "switch $sw"; TMB_LAZY_SWITCH=$sw timeout 600 python scripts/bench_eig.py 2 2160x270 3840x480 4320x540 7680x960 2>&1 | grep "n="
done
