#!/bin/bash
# Grid-size A/B of the shared-memory tridiagonalisation (fewer blocks: cheaper
# grid barrier, longer pass).
for nb in 148 128 112 96 74; do echo "NB=$nb"; TMB_SMEM_NB=$nb python scripts/bench_eig.py 3 1080x270 1920x480 2>&1 | grep -v "^sytrd"; done
