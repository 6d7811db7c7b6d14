#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_api.py -q -m gpu -x -k "eig or hosvd" > gpurun_out/r02_t_eigfix.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/r02_t_eigfix.log
TMB_EIG_STATS=1 timeout 900 python scripts/run_configs.py c4_2 > gpurun_out/r02_c4_2.txt 2> gpurun_out/r02_c4_2_eig.err; echo "c4_2 rc=$?"
cat gpurun_out/r02_c4_2.txt
python - <<'PY'
import re
v=[(int(m.group(1)), float(m.group(3))) for m in re.finditer(r"n=(\d+) k=(\d+) max\|X\^T X - I\| = ([0-9.e+-]+)", open("gpurun_out/r02_c4_2_eig.err").read())]
for n in sorted(set(a for a,_ in v)):
    xs=[b for a,b in v if a==n]; print("n", n, "solves", len(xs), "max e0", max(xs))
PY
timeout 900 python scripts/config_families.py c4_2 c5 > gpurun_out/r02_families.txt 2>&1; echo "families rc=$?"; cat gpurun_out/r02_families.txt
