for w in 2 4 1; do TMB_BISECT_WARPS=$w python scripts/bench_eig.py 5 1080x270 1920x480 2>&1 | sed "s/^/warps=$w /"; done
