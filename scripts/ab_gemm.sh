#!/bin/bash
# A/B the DMMA GEMM tile variants built into scripts/ab_libs/ (see _build.py env hooks).
for lib in scripts/ab_libs/libtmb_*.so; do
  echo "== $lib"
  TMB_LIB=$lib python scripts/bench_gemm.py 3
done
