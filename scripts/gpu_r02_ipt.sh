#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_api.py -q -m gpu -x -k "colour or eig" > gpurun_out/r02_t_ipt.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r02_t_ipt.log
timeout 600 python scripts/bench_elementwise.py 10 color_u8 > gpurun_out/r02_elementwise.txt 2>&1; cat gpurun_out/r02_elementwise.txt
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_c2_ipt.log 2>&1; echo "bench rc=$?"
python -c "
import json
d=json.loads([x for x in open('gpurun_out/r02_bench_c2_ipt.log') if x.startswith('{')][-1])
print(d['value'], d['ms_per_step'], d['e2e']['value'], d['hooi_sweep_ms'], d['roofline_elementwise'], d['kernel_families'])
"
