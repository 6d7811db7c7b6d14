#!/bin/bash
# full GPU suite + smoke + C2 bench (driver command)
mkdir -p gpurun_out
O=gpurun_out/s5_check
timeout 2400 python -m pytest tests -q -x -m gpu > ${O}_tests.log 2>&1; echo "tests rc=$?"; tail -3 ${O}_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > ${O}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 ${O}_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > ${O}_bench.log 2>&1; echo "bench rc=$?"; tail -1 ${O}_bench.log | cut -c1-330
