python scripts/bench_eig.py 1 1920x480 > gpurun_out/p9.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_sytrd_tail1 -c 1 -o gpurun_out/tail1 python scripts/bench_eig.py 1 1920x480 > gpurun_out/ncu9.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_bisect_mw -c 1 -o gpurun_out/bisect python scripts/bench_eig.py 1 1920x480 > gpurun_out/ncu9b.log 2>&1
tail -2 gpurun_out/ncu9.log
