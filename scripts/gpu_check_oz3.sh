timeout 120 python scripts/oz_sha.py; TMB_OZ_BK=32 timeout 120 python scripts/oz_sha.py
timeout 120 python scripts/check_ozaki.py; TMB_OZ_BK=32 timeout 120 python scripts/check_ozaki.py
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "ozaki or c2_full" 2>&1 | tail -2
