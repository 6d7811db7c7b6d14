for t in 0 -1 ""; do echo "TMB_SYTRD_TAIL=$t"; env ${t:+TMB_SYTRD_TAIL=$t} python scripts/bench_eig.py 3 300x60 600x120 1080x270 1920x480; done
python -m pytest tests/test_gpu_api.py tests/test_gpu_parity.py tests/test_pp_parity.py -q -x -m gpu 2>&1 | tail -3
