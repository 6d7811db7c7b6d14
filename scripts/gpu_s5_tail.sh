#!/bin/bash
# A/B: single-CTA tail: shared-memory matrix (shape 2 = 512 x 4) vs the register-tiled tail (shape 9)
mkdir -p gpurun_out
O=gpurun_out/s5_tail2.txt
: > $O
for cfg in "TMB_T1_SHAPE=2" "TMB_T1_SHAPE=9" "TMB_T1_SHAPE=9 TMB_TRD_PROFILE=1"; do
  echo "cfg=[$cfg]" >> $O
  env $cfg timeout 600 python scripts/bench_eig.py 2 130x30 500x100 700x175 1080x270 1920x480 2>&1 | grep -v "sytrd_smem\|block-slot" >> $O
done
cat $O
