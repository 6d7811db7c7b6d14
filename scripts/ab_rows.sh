for cfg in "" "TMB_ROWS_NT=512" "TMB_ROWS_NT=512 TMB_ROWS_CB=1"; do echo "cfg=[$cfg]"; env $cfg python scripts/bench_eig.py 3 500x100 1080x270 1920x480; done
