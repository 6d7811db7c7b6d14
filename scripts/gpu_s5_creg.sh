#!/bin/bash
# A/B: scribe block (block 0 owns no columns) x thread-count / register-column variants
mkdir -p gpurun_out
O=gpurun_out/s5_creg4.txt
: > $O
for cfg in "" "TMB_SMEM_SCRIBE=1" "TMB_SMEM_NT=256 TMB_SMEM_CREG=4" "TMB_SMEM_NT=256 TMB_SMEM_CREG=4 TMB_SMEM_SCRIBE=1" "TMB_SMEM_NT=384 TMB_SMEM_CREG=0 TMB_SMEM_SCRIBE=1" "TMB_SMEM_NT=384 TMB_SMEM_CREG=4 TMB_SMEM_SCRIBE=1"; do
  echo "cfg=[$cfg]" >> $O
  env $cfg timeout 600 python scripts/bench_eig.py 3 700x175 1080x270 1500x300 1920x480 >> $O 2>&1
done
cat $O
