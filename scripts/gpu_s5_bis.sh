#!/bin/bash
# A/B: two-sided Sturm counts in the multisection
mkdir -p gpurun_out
O=gpurun_out/s5_bis.txt
: > $O
for cfg in "TMB_BISECT_TWOSIDED=0" "" "TMB_BISECT_WARPS=4"; do
  echo "cfg=[$cfg]" >> $O
  env $cfg timeout 600 python scripts/bench_eig.py 3 100x30 700x175 1080x270 1920x480 4320x540 >> $O 2>&1
done
cat $O
timeout 1500 python -m pytest tests/test_gpu_api.py -q -x -k "eig or lapack or two_stage or hosvd" 2>&1 | tail -3
