#!/bin/bash
# session-5 state check after the container was re-created: full GPU suite, smoke, driver-command bench (both arms)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
O=gpurun_out/s5
timeout 2400 python -m pytest tests -q -m gpu -x > ${O}_tests.log 2>&1; echo "tests rc=$?"; tail -3 ${O}_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > ${O}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 ${O}_smoke.log
timeout 1200 python bench.py > ${O}_bench_c2.log 2>&1; echo "bench rc=$?"
tail -1 ${O}_bench_c2.log | cut -c1-400
timeout 1200 python bench.py --impl reference --steps 2 --warmup 1 > ${O}_bench_ref.log 2>&1; echo "ref rc=$?"
tail -1 ${O}_bench_ref.log | cut -c1-600
