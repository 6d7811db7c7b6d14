#!/bin/bash
# session-3 refresh: full GPU suite, driver-command bench, launch list of one C2 step, configs
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
O=gpurun_out/s3f
timeout 2400 python -m pytest tests -q -m gpu -x > ${O}_tests.log 2>&1; echo "tests rc=$?"; tail -2 ${O}_tests.log
timeout 1200 python bench.py --steps 20 --warmup 5 > ${O}_bench_c2.log 2>&1; echo "bench rc=$?"
LPS=$(python -c "import json;d=json.loads([x for x in open('${O}_bench_c2.log') if x.startswith('{')][-1]);print(int(d['gpu_launches']/d['steps']))")
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s $((3 * LPS)) -c $LPS --csv --log-file ${O}_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > ${O}_ncu.log 2>&1; echo "ncu rc=$?"
python scripts/launch_summary.py ${O}_launches.csv 25 > ${O}_launches_summary.txt 2>&1
timeout 1500 python scripts/run_configs.py c1 c3 c4_8 c4_4 c4_2 c5 > ${O}_configs.txt 2>&1; echo "configs rc=$?"
timeout 1200 python bench.py --workload c3 --steps 2 --warmup 3 --no-cpu-baseline > ${O}_bench_c3.log 2>&1; echo "c3 rc=$?"
tail -1 ${O}_bench_c2.log | cut -c1-300
