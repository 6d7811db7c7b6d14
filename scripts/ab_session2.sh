#!/bin/bash
# A/B switches behind this session's kernel changes (run under gpurun; each line
# prints the default build's numbers and the variant's):
#   TMB_WY_NOCLUSTER=1   one CTA per 4 eigenvector columns instead of the cluster row-split WY kernel
#   TMB_NO_TTM2=1        the two trailing small-mode contractions as separate passes
#   TMB_SMEM_RPT4=1      4 rows per thread in the shared-memory tridiagonalisation for n <= 1536
#   TMB_BISECT_WARPS=w   64 (w=2, default) / 32 / 128 shifts per multisection round
#   TMB_SYTRD_TAIL1=m    trailing block handed to the single-CTA kernel (default 128)
set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python scripts/bench_eig.py 5 1080x270 1920x480
TMB_WY_NOCLUSTER=1 python scripts/bench_eig.py 5 1080x270 1920x480
TMB_SMEM_RPT4=1 python scripts/bench_eig.py 5 1080x270
for w in 1 4; do TMB_BISECT_WARPS=$w python scripts/bench_eig.py 5 1080x270 1920x480; done
for t in 96 160; do TMB_SYTRD_TAIL1=$t python scripts/bench_eig.py 3 1080x270 1920x480; done
python bench.py --steps 3 --warmup 3 --no-cpu-baseline | cut -c1-300
TMB_NO_TTM2=1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline | cut -c1-300
