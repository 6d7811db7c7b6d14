for cb in "" 1 2 4; do echo "TMB_ROWS_CB=$cb"; env ${cb:+TMB_ROWS_CB=$cb} python scripts/bench_eig.py 3 500x100 1080x270 1920x480; done
TMB_SYTRD_COLS=1 python scripts/bench_eig.py 3 500x100 1080x270 1920x480
