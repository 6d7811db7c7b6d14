#!/bin/bash
# A/B: pass specialised on the block-uniform dead row-group count (no per-row predicates)
mkdir -p gpurun_out
O=gpurun_out/s5_ubs.txt
: > $O
for cfg in "TMB_SMEM_UBS=0" "" "TMB_SMEM_CREG=0"; do
  echo "cfg=[$cfg]" >> $O
  env $cfg timeout 600 python scripts/bench_eig.py 3 601x100 700x175 1080x270 1500x300 1920x480 2160x540 >> $O 2>&1
done
cat $O
timeout 1500 python -m pytest tests/test_gpu_api.py -q -x -k "eig or lapack or two_stage or hosvd" 2>&1 | tail -3
