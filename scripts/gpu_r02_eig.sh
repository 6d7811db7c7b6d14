#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_api.py -q -m gpu -x > gpurun_out/r02_t_api.log 2>&1; echo "api rc=$?"
TMB_EIG_STATS=1 timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_eigstats.log 2> gpurun_out/r02_eigstats.err; echo "bench rc=$?"
sort gpurun_out/r02_eigstats.err | uniq -c | sort -rn | head -5 > gpurun_out/r02_eigstats_summary.txt
python - <<'PY' >> gpurun_out/r02_eigstats_summary.txt
import re
v=[float(m.group(1)) for m in re.finditer(r"= ([0-9.e+-]+)", open("gpurun_out/r02_eigstats.err").read())]
print("count", len(v), "max", max(v) if v else None)
PY
tail -3 gpurun_out/r02_t_api.log; cat gpurun_out/r02_eigstats_summary.txt
