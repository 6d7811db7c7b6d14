#!/bin/bash
# A/B of the tridiagonalisation variants: shared-memory-resident 512-thread
# blocks (default), with the trailing 128/256 columns on the cluster kernel,
# 256-thread blocks, and the L2-streaming row kernel.
for cfg in "" "TMB_SYTRD_TAIL=128" "TMB_SYTRD_TAIL=256" "TMB_SMEM_NT=256" "TMB_SYTRD_L2=1"; do echo "cfg=[$cfg]"; env $cfg python scripts/bench_eig.py 3 500x100 1080x270 1920x480; done
