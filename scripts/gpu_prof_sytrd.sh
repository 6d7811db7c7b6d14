# small-n (C1) eigen-solve timings and the ncu capture of the current shared-memory tridiagonalisation
python scripts/bench_eig.py 5 384x48 512x64 300x60 600x120
TMB_SYTRD_TAIL=0 python scripts/bench_eig.py 5 384x48 300x60
python scripts/bench_eig.py 1 1080x270 1920x480 > gpurun_out/p32.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_sytrd_smem -c 2 -o gpurun_out/sytrd_smem_s2 python scripts/bench_eig.py 1 1080x270 1920x480 > gpurun_out/ncu32.log 2>&1
tail -1 gpurun_out/ncu32.log
