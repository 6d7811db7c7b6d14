#!/bin/bash
# A/B: shifts per round in the two-sided multisection (32 / 64) at the larger sizes; default = adaptive
mkdir -p gpurun_out
O=gpurun_out/s5_bis3.txt
: > $O
for cfg in "TMB_BISECT_WARPS=1" "TMB_BISECT_WARPS=2" ""; do
  echo "cfg=[$cfg]" >> $O
  env $cfg timeout 600 python scripts/bench_eig.py 2 1920x480 2160x270 2160x540 3840x480 3840x960 4320x540 7680x960 >> $O 2>&1
done
cat $O
