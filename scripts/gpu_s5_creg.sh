#!/bin/bash
# A/B: software-pipelined shared-memory pass x register columns
mkdir -p gpurun_out
O=gpurun_out/s5_pipe.txt
: > $O
for cfg in "" "TMB_SMEM_PIPE=1" "TMB_SMEM_PIPE=1 TMB_SMEM_CREG=0" "TMB_SMEM_CREG=0"; do
  echo "cfg=[$cfg]" >> $O
  env $cfg timeout 600 python scripts/bench_eig.py 3 700x175 1080x270 1500x300 1920x480 >> $O 2>&1
done
cat $O
