set -x
python bench.py > gpurun_out/bench5.log 2>&1
LPS=$(python -c "import json;d=json.loads(open('gpurun_out/bench5.log').read().strip().splitlines()[-1]);print(d['gpu_launches']//d['steps'])")
echo LPS=$LPS
python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/plain5.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -s $((3 * LPS)) -c $LPS --csv --log-file gpurun_out/launches5.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_color_u8 -s 4 -c 1 -o gpurun_out/color_c5 python scripts/bench_elementwise.py 1 c5 > gpurun_out/ncu5b.log 2>&1
tail -1 gpurun_out/bench5.log
