for nb in 64 32; do echo "TMB_WY_NB=$nb"; TMB_WY_NB=$nb python scripts/bench_eig.py 3 1080x270 1920x480; done
