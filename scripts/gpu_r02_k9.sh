#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_stream.py -q -m gpu -x -k "not c5" > gpurun_out/r02_t_k9.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r02_t_k9.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02_bench_c2_k9.log 2>&1; echo "bench rc=$?"
python -c "
import json
d=json.loads([x for x in open('gpurun_out/r02_bench_c2_k9.log') if x.startswith('{')][-1])
print(d['value'], d['ms_per_step'], d['e2e']['value'], d['hooi_sweep_ms'], d['rel_err'], d['cpu_baseline'])
"
