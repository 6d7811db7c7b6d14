# every BASELINE config end to end on one B200 + the row-sharded C5 emulation (session-2 build)
python scripts/run_configs.py c1 c3 c4_8 c4_4 c4_2 c5 > gpurun_out/configs.log 2>&1
python scripts/run_sharded_emulated.py c5 2 3 > gpurun_out/sharded.log 2>&1
cat gpurun_out/configs.log gpurun_out/sharded.log
